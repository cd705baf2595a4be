#!/bin/bash
# Round-2 GPU session L: C1 / C3 bench lines, per-workload N-body DRAM traffic (ncu).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for c in c1 c3 c2t; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
for c in c1 c2 c3 c4; do
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:nbody_kernel -c 1 --csv python scripts/nbody_traffic_once.py $c > gpurun_out/traffic_$c.csv 2> gpurun_out/traffic_$c.err; echo "ncu $c rc=$?"
done
