#!/bin/bash
# Polish timing vs SPK_POLISH_MINB (CTAs per SM the ring kernel is register-budgeted for).
# usage: bash scripts/polish_minb.sh "3 4"
for M in $1; do
  rm -rf /tmp/pm$M && mkdir -p /tmp/pm$M && cp -r paper_2108_02991_b200 include oracle tests scripts bench.py __graft_entry__.py /tmp/pm$M/
  (cd /tmp/pm$M && SPK_NVCC_EXTRA="-DSPK_POLISH_MINB=$M" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1) || echo "build M=$M failed"
  echo "== MINB=$M"
  (cd /tmp/pm$M && cuobjdump -res-usage paper_2108_02991_b200/_lib/project.o 2>&1 | grep -A1 "polish_kernelILi3ELi256" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - -
   timeout 300 python scripts/polish_c2.py 2>&1 | tail -2
   timeout 600 python scripts/profile_step.py --iters 8 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('project', [round(x,1) for x in d['project']['ms']], 'mean', round(d['project']['mean_ms'],1))")
done
