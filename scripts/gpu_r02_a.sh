#!/bin/bash
# Round-2 GPU session A: tests (incl. trajectory drift), in-loop fixtures, bench with
# sub-records, per-rank shares.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
SPK_DRIFT_REPORT=gpurun_out/drift.jsonl timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest.log
timeout 900 python scripts/make_inloop_shots.py c2 c4 > gpurun_out/inloop.log 2>&1; echo "inloop rc=$?"; cp bench_data/*.npz gpurun_out/ 2>/dev/null
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 900 python scripts/rank_share.py --config c2 > gpurun_out/rank_share_c2.jsonl 2> gpurun_out/rank_share_c2.err; echo "rank_share rc=$?"
