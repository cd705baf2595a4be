#!/bin/bash
# Sub-walk traversal: the whole GPU suite, then the full3d per-rank-share projection.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_sw2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_sw2.log
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d_sw.json 2> gpurun_out/rank_share_full3d_sw.err; echo "schedule rc=$?"; tail -2 gpurun_out/rank_share_full3d_sw.err
