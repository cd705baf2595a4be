#!/bin/bash
# Round-2 GPU session W: stack (C3) with K2 under the polish: tests + C3 bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_optimize.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/tests_w.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_w.log
for o in 0 1; do SPK_OVERLAP=$o timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_ovl$o.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_c3_ovl$o.json').read().strip().splitlines()[-1]); print('overlap $o', d['ms_per_step'])"; done
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1]); print('default', d['ms_per_step'])"
