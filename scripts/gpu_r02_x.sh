#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -x -m gpu -k schedules > gpurun_out/tests_x.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/tests_x.log
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; echo "c3 rc=$?"
