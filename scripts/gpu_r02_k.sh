#!/bin/bash
# Round-2 GPU session K: N-body with 4 lattice tiles per TMA stage (one CTA barrier per
# 2048 cells) vs the previous tree (git HEAD), and the lattice-only launch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_optimize.py tests/test_gpu_trajectory.py -q -x -m gpu > gpurun_out/tests_k.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_k.log
rm -rf /tmp/ab_prev && mkdir -p /tmp/ab_prev && cp -r paper_2108_02991_b200 include scripts bench.py bench_data /tmp/ab_prev/ && cp scripts/variants/nbody_prev.cu /tmp/ab_prev/paper_2108_02991_b200/csrc/nbody.cu && rm -f /tmp/ab_prev/paper_2108_02991_b200/_lib/*
(cd /tmp/ab_prev && python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1)
for v in new prev new prev; do
  if [ $v = new ]; then d=.; else d=/tmp/ab_prev; fi
  echo "== $v"; (cd $d && timeout 600 python scripts/ab_r02.py nbody)
done > gpurun_out/ab_nbody_k.txt 2>&1
cat gpurun_out/ab_nbody_k.txt
