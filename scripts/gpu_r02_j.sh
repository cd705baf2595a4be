#!/bin/bash
# Round-2 GPU session J: polish ring width (warps per shot) vs throughput, in-loop shots.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for w in 16 12 8 6; do echo "== C4 warps $w"; SPK_POLISH_WARPS=$w timeout 600 python scripts/polish_inloop_once.py 4096 2 c4; done > gpurun_out/ring_width_c4.txt 2>&1
for w in 8 6 4; do echo "== C2 warps $w"; SPK_POLISH_WARPS=$w timeout 600 python scripts/polish_inloop_once.py 1024 2 c2; echo "== C2 128 shots warps $w"; SPK_POLISH_WARPS=$w timeout 600 python scripts/polish_inloop_once.py 128 2 c2; done > gpurun_out/ring_width_c2.txt 2>&1
cat gpurun_out/ring_width_c4.txt gpurun_out/ring_width_c2.txt
