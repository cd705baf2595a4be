#!/bin/bash
# ncu of the DMMA fp64 NUDFT adjoint (C2 pattern, 64^3 grid).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python scripts/nudft_once.py > /dev/null 2>&1 || { echo "run failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nudft_adjoint_dmma -c 1 -o gpurun_out/dmma_ncu python scripts/nudft_once.py > gpurun_out/dmma_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/dmma_ncu.log
