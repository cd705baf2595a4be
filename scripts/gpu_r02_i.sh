#!/bin/bash
# Round-2 GPU session I: full GPU tests, the driver's bench command, the reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_i.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.log 2>&1; echo "smoke rc=$?"
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_i.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_i.json 2> gpurun_out/bench_ref_i.err; echo "ref rc=$?"
