#!/bin/bash
# e2e through the public step API (bench default line) + the 2-rank bench test.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --steps 20 --warmup 5 --no-sub > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_e2e.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_e2e.json").read().strip().splitlines()[-1])
print("step", d["ms_per_step"], "e2e", d["e2e"]["s_per_iteration"], d["e2e"]["h2d_bytes_per_step"], d["e2e"]["d2h_bytes_per_step"], "numpy", d["e2e_numpy_api"]["s_per_iteration"], "cpu", d["cpu_baseline"]["value"], d["clocks"])
PY
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_bench_cli.py -q -x > gpurun_out/gputest_e2e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_e2e.log
