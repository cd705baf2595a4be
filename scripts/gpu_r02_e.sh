#!/bin/bash
# Round-2 GPU session E: polish box fast path (A/B), K2-under-polish overlap probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py tests/test_gpu_optimize.py -q -x -m gpu > gpurun_out/tests_e.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_e.log
bash scripts/ab_build.sh nobox "-DSPK_BOX_FAST=0"
for v in base nobox base nobox; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v" >> gpurun_out/ab_polish_e.txt
  (cd $d && timeout 300 python scripts/polish_inloop_once.py 128 2 && timeout 300 python scripts/polish_inloop_once.py 1024 2) >> gpurun_out/ab_polish_e.txt 2>&1
done
cat gpurun_out/ab_polish_e.txt
timeout 600 python scripts/overlap_probe.py 8 > gpurun_out/overlap8.txt 2>&1; cat gpurun_out/overlap8.txt
timeout 600 python scripts/overlap_probe.py 4 > gpurun_out/overlap4.txt 2>&1; cat gpurun_out/overlap4.txt
