#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_projection.py -q -x -m gpu > gpurun_out/tests_u.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_u.log
