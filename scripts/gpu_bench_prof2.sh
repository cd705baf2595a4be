# bench (plain) + launch list of the same command + ncu --set full of the N-body kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?"; cat gpurun_out/bench.json
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_small.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
timeout 300 python scripts/nbody_once.py 2 > gpurun_out/nbody_once.log 2>&1 && cat gpurun_out/nbody_once.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nbody_kernel -s 1 -c 1 -o gpurun_out/nbody_full3 python scripts/nbody_once.py 2 > gpurun_out/ncu_full3.log 2>&1
echo "ncu full exit $?"
