#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --config c2t --steps 5 --warmup 3 > gpurun_out/bench_c2t.json 2> gpurun_out/bench_c2t.err; tail -3 gpurun_out/bench_c2t.err
timeout 1500 python bench.py --config c4t --steps 3 --warmup 3 > gpurun_out/bench_c4t.json 2> gpurun_out/bench_c4t.err; tail -3 gpurun_out/bench_c4t.err
cat gpurun_out/bench_c2t.json gpurun_out/bench_c4t.json
