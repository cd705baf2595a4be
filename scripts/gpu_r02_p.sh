#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python scripts/lattice_tree_phases.py > gpurun_out/lattice_tree_phases.jsonl 2> gpurun_out/ltp.err; echo "rc=$?"; tail -3 gpurun_out/ltp.err
