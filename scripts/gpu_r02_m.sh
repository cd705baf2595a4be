#!/bin/bash
# Round-2 GPU session M: K1 co-running with the tail of the per-group K2 launches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_m.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_m.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-sub --no-cpu-baseline > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['s_per_iteration'], d['schedule']['timed_steps_with_k2_under_polish'])"
timeout 1200 python scripts/rank_share.py --config c2 > gpurun_out/rank_share_c2_m.jsonl 2> gpurun_out/rank_share_c2_m.err; echo "rank_share rc=$?"
