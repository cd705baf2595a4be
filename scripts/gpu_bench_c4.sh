mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "bench c4 exit $?"; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
