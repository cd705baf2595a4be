#!/bin/bash
# Round-2 GPU session T: branch-free unpinned speed pairs / accel triples in the polish
# (bitwise tests on the variant build, in-loop A/B).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
bash scripts/ab_build.sh bf "-DSPK_POLISH_BRANCHFREE=1"
(cd /tmp/ab_bf && timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py tests/test_gpu_optimize.py -q -x -m gpu > /root/repo/gpurun_out/bf_tests.log 2>&1; echo "bf tests rc=$?"; tail -2 /root/repo/gpurun_out/bf_tests.log)
for v in base bf base bf; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v"; (cd $d && timeout 300 python scripts/polish_inloop_once.py 128 2 && timeout 300 python scripts/polish_inloop_once.py 1024 2 && timeout 300 python scripts/polish_fixed.py 16 3200)
done > gpurun_out/ab_bf.txt 2>&1
cat gpurun_out/ab_bf.txt
