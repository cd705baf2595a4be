mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/polish_latency.py 800 1 > gpurun_out/pl1.log 2>&1 && cat gpurun_out/pl1.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:polish_kernel -s 1 -c 1 -o gpurun_out/polish_single python scripts/polish_latency.py 800 1 > gpurun_out/ncu_ps.log 2>&1
echo "ncu exit $?"
