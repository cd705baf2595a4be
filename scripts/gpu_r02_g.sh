#!/bin/bash
# Round-2 GPU session G: K2-under-polish overlap (tests + projected per-rank shares).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_g.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_g.log
timeout 1200 python scripts/rank_share.py --config c2 > gpurun_out/rank_share_c2_g.jsonl 2> gpurun_out/rank_share_c2_g.err; echo "rank_share rc=$?"; tail -3 gpurun_out/rank_share_c2_g.err
