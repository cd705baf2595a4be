#!/bin/bash
# Round-2 GPU session R: spatial target layout for the treecodes (test + projected C5).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_optimize.py tests/test_gpu_tree.py -q -x -m gpu > gpurun_out/tests_r.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_r.log
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d_sp.json 2> gpurun_out/rank_share_full3d_sp.err; echo "schedule rc=$?"; tail -2 gpurun_out/rank_share_full3d_sp.err
