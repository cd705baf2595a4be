#!/bin/bash
# Sub-walk tree traversal: tree tests, fuzz, and the per-phase timing of one rank's block.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fuzz.py -q -x > gpurun_out/gputest_sw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_sw.log
timeout 600 python scripts/spatial_block_phases.py > gpurun_out/phases_sw.jsonl 2> gpurun_out/phases_sw.err; echo "phases rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/phases_sw.jsonl"):
    d = json.loads(l)
    print(d["n_s"], d["ranks"], d["subwalk"], d["segments"], {k: round(v, 2) for k, v in d["phases_ms"].items()})
PY
