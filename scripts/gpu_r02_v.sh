#!/bin/bash
# Round-2 GPU session V: neighbour-pair barriers + 3 wrap buffers in the polish ring
# (SPK_PAIR_BAR): bitwise tests on both builds, in-loop A/B.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/base_tests_v.log 2>&1; echo "base tests rc=$?"; tail -2 gpurun_out/base_tests_v.log
bash scripts/ab_build.sh pb "-DSPK_PAIR_BAR=1"
(cd /tmp/ab_pb && timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_fuzz.py tests/test_gpu_optimize.py -q -x -m gpu > /root/repo/gpurun_out/pb_tests.log 2>&1; echo "pb tests rc=$?"; tail -2 /root/repo/gpurun_out/pb_tests.log)
for v in base pb base pb; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v"; (cd $d && timeout 300 python scripts/polish_inloop_once.py 128 2 && timeout 300 python scripts/polish_inloop_once.py 1024 2 && timeout 300 python scripts/polish_fixed.py 16 3200 && timeout 300 python scripts/polish_inloop_once.py 4096 1 c4)
done > gpurun_out/ab_pb.txt 2>&1
cat gpurun_out/ab_pb.txt
