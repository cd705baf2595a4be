#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
make -C oracle > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_tree_host.py -x -q 2>&1 | tail -30
timeout 1500 python scripts/tree_calibrate.py --clouds c2,u3,c1,s3 --orders 3,4,5,6 --thetas 0.5,0.6,0.7,0.8,0.9 --out gpurun_out/tree_cal3.jsonl > gpurun_out/tree_cal3.log 2>&1
tail -3 gpurun_out/tree_cal3.log
