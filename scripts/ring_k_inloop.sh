#!/bin/bash
# In-loop projection time per optimizer iteration (C2, scripts/profile_step.py) vs RING_K.
# usage: bash scripts/ring_k_inloop.sh "1 4" [iters]
IT=${2:-8}
for K in $1; do
  rm -rf /tmp/rk$K && mkdir -p /tmp/rk$K && cp -r paper_2108_02991_b200 include oracle tests scripts bench.py __graft_entry__.py /tmp/rk$K/
  (cd /tmp/rk$K && SPK_NVCC_EXTRA="-DSPK_RING_K=$K" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1) || echo "build K=$K failed"
  echo "== RING_K=$K"
  (cd /tmp/rk$K && timeout 600 python scripts/profile_step.py --iters $IT 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
print('project', [round(x,1) for x in d['project']['ms']], 'mean', round(d['project']['mean_ms'],1))
print('sweeps', d.get('sweeps'))")
done
