#!/bin/bash
# Round-2 GPU session N: new ABI tests; projected scaling of the full3d (C5) schedule.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_projection.py -q -x -m gpu > gpurun_out/tests_n.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_n.log
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d.json 2> gpurun_out/rank_share_full3d.err; echo "schedule rc=$?"; tail -2 gpurun_out/rank_share_full3d.err
