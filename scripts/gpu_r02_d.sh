#!/bin/bash
# Round-2 GPU session D: in-loop polish timing + ncu source-level profile of the polish.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for n in 16 128 1024; do timeout 300 python scripts/polish_inloop_once.py $n 2; done > gpurun_out/polish_inloop.txt 2>&1
cat gpurun_out/polish_inloop.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:polish_kernel -c 1 -o gpurun_out/polish_inloop128 python scripts/polish_inloop_once.py 128 1 > gpurun_out/ncu_pi.log 2>&1
echo "ncu exit $?"
