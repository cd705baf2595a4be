#!/bin/bash
# Refresh the other workloads' bench lines (C1 = configs[0], C3 stack, C2 treecodes).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for c in c1 c3 c2t; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d.get('e2e', {}).get('s_per_iteration'), (d.get('roofline') or {}).get('frac'))"; done
