#!/bin/bash
# round-end refresh: tests, smoke, every bench workload, C5 projection levels, full3d
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
tail -1 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>/dev/null
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c2t --steps 5 --warmup 3 > gpurun_out/bench_c2t.json 2>/dev/null
timeout 1200 python bench.py --config c4t --steps 3 --warmup 3 > gpurun_out/bench_c4t.json 2>/dev/null
for f in c2 c1 c3 c2t c4t; do python -c "import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', d['metric'], d['value'], d.get('ms_per_step'))"; done
timeout 2400 python scripts/full3d_run.py --n-git 100 --trace gpurun_out/full3d_trace.csv > gpurun_out/full3d.json 2> gpurun_out/full3d.err
python -c "import json; d=json.load(open('gpurun_out/full3d.json')); print('full3d', d['total_wall_s'], [round(l['wall_s'],1) for l in d['levels']], d['final_feasibility']['max'])"
timeout 2400 python scripts/c5_projection_levels.py > gpurun_out/c5_levels.jsonl 2> gpurun_out/c5_levels.err; tail -2 gpurun_out/c5_levels.err; wc -l gpurun_out/c5_levels.jsonl
