#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python scripts/full3d_run.py --n-git 3 > gpurun_out/full3d_short.json 2> gpurun_out/full3d_short.err; tail -2 gpurun_out/full3d_short.err; cat gpurun_out/full3d_short.json
timeout 2400 python scripts/full3d_run.py --n-git 100 --trace gpurun_out/full3d_trace.csv > gpurun_out/full3d.json 2> gpurun_out/full3d.err; tail -2 gpurun_out/full3d.err; cat gpurun_out/full3d.json
