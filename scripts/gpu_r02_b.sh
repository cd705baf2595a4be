#!/bin/bash
# Round-2 GPU session B: correctness of the FMA-rsqrt lattice and the certified fast
# sqrt/div polish, then A/B timings against the IEEE-only polish build.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_b.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest_b.log
timeout 600 python scripts/ab_r02.py nbody > gpurun_out/ab_nbody.txt 2>&1; echo "nbody rc=$?"
echo "== fastdiv" > gpurun_out/ab_polish.txt
timeout 600 python scripts/ab_r02.py polish >> gpurun_out/ab_polish.txt 2>&1; echo "polish rc=$?"
rm -rf /tmp/variant && mkdir -p /tmp/variant && cp -r paper_2108_02991_b200 include oracle tests scripts bench.py bench_data __graft_entry__.py /tmp/variant/
(cd /tmp/variant && SPK_NVCC_EXTRA="-DSPK_POLISH_FASTDIV=0" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1)
echo "== ieee only" >> gpurun_out/ab_polish.txt
(cd /tmp/variant && timeout 600 python scripts/ab_r02.py polish) >> gpurun_out/ab_polish.txt 2>&1; echo "polish-ieee rc=$?"
timeout 900 python scripts/rank_share.py --config c2 > gpurun_out/rank_share_c2_b.jsonl 2> gpurun_out/rank_share_c2_b.err; echo "rank_share rc=$?"
