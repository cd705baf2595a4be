mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-rows 1024 > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?"
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.log
