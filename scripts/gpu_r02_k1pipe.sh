#!/bin/bash
# K1 pipelined under the polish: device tests, 2-rank functional test, rank-share projection.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_optimize.py tests/test_gpu_multirank.py -q -x > gpurun_out/gputest_k1pipe.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_k1pipe.log
timeout 1500 python scripts/rank_share.py --ranks 1,2,4,8 > gpurun_out/rank_share_k1pipe.jsonl 2> gpurun_out/rank_share_k1pipe.err; echo "rank_share rc=$?"; tail -3 gpurun_out/rank_share_k1pipe.err
python - <<'PY'
import json
for l in open("gpurun_out/rank_share_k1pipe.jsonl"):
    d = json.loads(l)
    print(d["n_ranks"], "polite", round(d["polite_step_ms"], 1), round(d["polite_efficiency"] or 0, 3), "plain", round(d["step_ms"], 1), round(d["efficiency"] or 0, 3), "overlap", round(d["overlap_step_ms"], 1), round(d["overlap_efficiency"] or 0, 3), "pipelined", d["pipelined_step_ms"] and round(d["pipelined_step_ms"], 1), d["pipelined_efficiency"] and round(d["pipelined_efficiency"], 3))
PY
