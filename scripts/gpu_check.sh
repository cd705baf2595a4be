#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
tail -1 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2', d['ms_per_step'], d['roofline']['launch_ms'], d['e2e']['s_per_iteration'], d['cpu_baseline']['s_per_iteration_extrapolated'])"
timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/profile_step.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/profile_step.json')); [print(k, v['mean_ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
timeout 1200 python bench.py --config c4t --steps 3 --warmup 3 > gpurun_out/bench_c4t.json 2>/dev/null; python -c "import json; print('c4t', json.load(open('gpurun_out/bench_c4t.json'))['value'])"
timeout 900 python bench.py --config c2t --steps 5 --warmup 3 > gpurun_out/bench_c2t.json 2>/dev/null; python -c "import json; print('c2t', json.load(open('gpurun_out/bench_c2t.json'))['value'])"
timeout 2400 python scripts/full3d_run.py --n-git 100 --trace gpurun_out/full3d_trace.csv > gpurun_out/full3d.json 2> gpurun_out/full3d.err
python -c "
import json; d=json.load(open('gpurun_out/full3d.json')); print(d['total_wall_s'], [round(l['wall_s'],1) for l in d['levels']], d['final_feasibility']['max'])
for k,v in d['phases_by_samples_per_shot'].items(): print(k, {n:(round(x['mean_ms'],1), round(x['total_s'],1)) for n,x in v.items()})"
