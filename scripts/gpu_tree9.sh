#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tree.py -q 2>&1 | tail -6
timeout 600 python scripts/tree_small_p.py 2>&1 | tail -4
timeout 1200 python scripts/tree_calibrate.py --clouds c2,u3,c1,s3 --pairs 3:0.8,4:0.8,5:0.8,6:0.7,6:0.5,4:0.7,5:0.7,3:0.7 --out gpurun_out/tree_cal_w.jsonl > /dev/null 2>&1
timeout 1200 python scripts/tree_att_calibrate.py --cases c1,c2 --pairs 3:0.8,4:0.8,5:0.8,6:0.7,6:0.5,4:0.7,5:0.7 --out gpurun_out/tree_att_cal_w.jsonl > /dev/null 2>&1
ls -la gpurun_out/*_w.jsonl
