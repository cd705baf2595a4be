#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_optimize.py -x -q 2>&1 | tail -3
timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/profile_step.json 2> gpurun_out/profile_step.err
python -c "import json; d=json.load(open('gpurun_out/profile_step.json')); [print(k, v['mean_ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
timeout 900 python scripts/profile_step.py --config c4t --iters 3 > gpurun_out/prof_c4t_b.json 2> gpurun_out/prof_c4t_b.err
python -c "import json; d=json.load(open('gpurun_out/prof_c4t_b.json')); [print(k, v['ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
