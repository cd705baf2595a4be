mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/profile_step.py --iters 1 > gpurun_out/ps1.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:polish_kernel -s 2 -c 1 -o gpurun_out/polish_full python scripts/profile_step.py --iters 1 > gpurun_out/ncu_polish.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_polish.log
