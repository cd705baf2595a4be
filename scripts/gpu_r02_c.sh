#!/bin/bash
# Round-2 GPU session C: polish ring loop, 4x unrolled (static window) vs one step per
# iteration (register-move window, a quarter of the code).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
bash scripts/ab_build.sh u1 "-DSPK_RING_UNROLL=1"
bash scripts/ab_build.sh u1k8 "-DSPK_RING_UNROLL=1 -DSPK_RING_K=8"
(cd /tmp/ab_u1 && timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py -q -x -m gpu > /root/repo/gpurun_out/u1_tests.log 2>&1; echo "u1 tests rc=$?")
for v in base u1 u1k8 base u1; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v" >> gpurun_out/ab_polish_c.txt
  (cd $d && timeout 600 python scripts/ab_r02.py polish) >> gpurun_out/ab_polish_c.txt 2>&1
done
