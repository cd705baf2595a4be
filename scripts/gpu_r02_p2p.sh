#!/bin/bash
# Fused position all-gather (polish epilogue writes into the peers' buffers over CUDA IPC):
# device tests (2 processes sharing cuda:0), and the polish timing of the changed kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_projection.py tests/test_gpu_abi_errors.py tests/test_gpu_optimize.py -q -x > gpurun_out/gputest_p2p.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest_p2p.log
for n in 4096; do timeout 600 python scripts/polish_inloop_once.py $n 2 c4 | tail -1; done
timeout 600 python scripts/polish_inloop_once.py 1024 3 c2 | tail -1
