#!/bin/bash
# ncu evidence for profiles/: launch list of the bench step + full sets of the K3 and
# analysis kernels (each command first runs without ncu)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>/dev/null && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/polish_once.py > /dev/null && timeout 900 ncu --set full --import-source on --clock-control none -k regex:polish_kernel -c 1 -o gpurun_out/polish python scripts/polish_once.py > /dev/null 2>&1
python scripts/fista_once.py c4 > /dev/null && timeout 900 ncu --set full --import-source on --clock-control none -k regex:fista_kernel -c 1 -o gpurun_out/fista python scripts/fista_once.py c4 > /dev/null 2>&1
python scripts/nudft_once.py > /dev/null && timeout 900 ncu --set full --import-source on --clock-control none -k regex:nudft_ -c 2 -o gpurun_out/nudft python scripts/nudft_once.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches.csv
