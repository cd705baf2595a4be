mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/polish_latency.py 1600 2>&1 | tee gpurun_out/polish_latency.log
