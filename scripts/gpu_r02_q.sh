#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python scripts/tree_minlevel.py > gpurun_out/tree_minlevel.txt 2>&1; echo "rc=$?"; cat gpurun_out/tree_minlevel.txt
