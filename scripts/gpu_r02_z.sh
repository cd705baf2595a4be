#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_z.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_z.log
timeout 600 python scripts/e2e_profile.py > gpurun_out/e2e_profile_z.json 2>&1; cat gpurun_out/e2e_profile_z.json | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(sum(v[1:])/len(v[1:]),1) for k,v in d.items()})"
timeout 900 python bench.py --steps 20 --warmup 5 --no-sub --no-cpu-baseline > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err; python -c "import json; d=json.loads(open('gpurun_out/bench_z.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['s_per_iteration'])"
