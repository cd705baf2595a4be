#!/bin/bash
# (historical: the HEAD copies it compared against were removed after the A/B: working tree 3837-3854 ms vs HEAD 3863-3952 ms)
# A/B of the polish kernel: working tree vs HEAD's project.cu (C4 in-loop polish, alternating).
mkdir -p gpurun_out
for v in wt hd; do
  rm -rf /tmp/ab_$v && mkdir -p /tmp/ab_$v
  cp -r paper_2108_02991_b200 include oracle tests scripts bench.py bench_data __graft_entry__.py /tmp/ab_$v/
  rm -f /tmp/ab_$v/paper_2108_02991_b200/_lib/*.o /tmp/ab_$v/paper_2108_02991_b200/_lib/*.so
  if [ $v = hd ]; then cp scripts/variants/project_head.cu /tmp/ab_$v/paper_2108_02991_b200/csrc/project.cu; cp scripts/variants/sparkling_b200_head.h /tmp/ab_$v/include/sparkling_b200.h; fi
  (cd /tmp/ab_$v && python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /tmp/ab_$v.log 2>&1) || { echo "build $v failed"; tail /tmp/ab_$v.log; }
done
for r in 1 2 3; do for v in wt hd; do echo -n "$v: "; (cd /tmp/ab_$v && timeout 600 python scripts/polish_inloop_once.py 4096 1 c4 | tail -1); done; done
