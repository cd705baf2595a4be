#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c2t --steps 5 --warmup 3 > gpurun_out/bench_c2t.json 2>/dev/null
timeout 1200 python bench.py --config c4t --steps 3 --warmup 3 > gpurun_out/bench_c4t.json 2>/dev/null
python -c "import json; [print(f, json.load(open(f))['value']) for f in ('gpurun_out/bench_c2t.json','gpurun_out/bench_c4t.json')]"
timeout 2400 python scripts/full3d_run.py --n-git 100 --trace gpurun_out/full3d_trace.csv > gpurun_out/full3d.json 2> gpurun_out/full3d.err; tail -2 gpurun_out/full3d.err
python -c "
import json; d=json.load(open('gpurun_out/full3d.json')); print(d['total_wall_s'], [round(l['wall_s'],1) for l in d['levels']], d['final_feasibility']['max'])
for k,v in d['phases_by_samples_per_shot'].items(): print(k, {n:(round(x['mean_ms'],1), round(x['total_s'],1)) for n,x in v.items()})"
