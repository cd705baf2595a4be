#!/bin/bash
# Round-2 GPU session O: ncu launch list of the bench's C2 step (the same command without
# the C4 sub-records), full ncu set of the fused N-body for profiles/, projected full3d
# scaling (probe warmed).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > gpurun_out/b_o.json 2>/dev/null; echo "bench rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > gpurun_out/ncu_launch_o.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nbody_kernel -s 1 -c 1 -o gpurun_out/nbody_c2_full python scripts/nbody_once.py 2 > /dev/null 2>&1; echo "ncu nbody rc=$?"
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d.json 2> gpurun_out/rank_share_full3d.err; echo "schedule rc=$?"
