#!/bin/bash
# full GPU validation + default bench + ncu capture of the treecode eval kernel
set -x
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
timeout 900 python bench.py --config c2t --steps 3 --warmup 3 > gpurun_out/bench_c2t_b.json 2>/dev/null && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tree_eval_kernel -s 2 -c 1 -o gpurun_out/tree_eval python bench.py --config c2t --steps 1 --warmup 1 > gpurun_out/ncu_tree.log 2>&1; tail -3 gpurun_out/ncu_tree.log
