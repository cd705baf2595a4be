#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_analysis.py tests/test_analysis_host.py -x -q 2>&1 | tail -25
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_optimize.py -q 2>&1 | tail -3
