#!/bin/bash
# Round-2 GPU session H: source-level ncu captures of the fused N-body (C2) and FISTA (C4).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nbody_kernel -s 1 -c 1 -o gpurun_out/nbody_c2_src python scripts/nbody_once.py 2 > gpurun_out/ncu_nb.log 2>&1; echo "ncu nbody $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fista_kernel -c 1 -o gpurun_out/fista_c4_src python scripts/fista_once.py c4 > gpurun_out/ncu_fi.log 2>&1; echo "ncu fista $?"
