#!/bin/bash
# Overlap schedule at a rank's N = 4 / 8 share of C2: number of polish groups.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for g in 8 16 32; do
  timeout 900 python scripts/rank_share.py --ranks 1,4,8 --groups $g > gpurun_out/rank_share_g$g.jsonl 2> gpurun_out/rank_share_g$g.err; echo "groups $g rc=$?"
  python - $g <<'PY'
import json, sys
for l in open(f"gpurun_out/rank_share_g{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    its = d["iterations"][1:]
    k1 = [max(r["overlap_k1_ms"] for r in it["ranks"]) for it in its]
    pk = [max(r["overlap_project_k2_ms"] for r in it["ranks"]) for it in its]
    print(d["n_ranks"], d["groups"], round(d["overlap_step_ms"], 1), round(d["overlap_efficiency"], 3), "proj", [round(x, 1) for x in pk], "k1", [round(x, 1) for x in k1])
PY
done
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d_med.json 2> gpurun_out/rank_share_full3d_med.err; echo "schedule rc=$?"; tail -2 gpurun_out/rank_share_full3d_med.err
