#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
make -C oracle > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_tree_host.py -x -q 2>&1 | tail -30
timeout 1500 python scripts/tree_att_calibrate.py --cases c1,c2,c4 --out gpurun_out/tree_att_cal.jsonl > gpurun_out/tree_att_cal.log 2>&1
tail -5 gpurun_out/tree_att_cal.log
