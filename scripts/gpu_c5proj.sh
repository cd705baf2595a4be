mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python scripts/c5_projection_levels.py 8 > gpurun_out/c5_proj.jsonl 2> gpurun_out/c5_proj.err; echo "exit $?"; cat gpurun_out/c5_proj.jsonl; tail -3 gpurun_out/c5_proj.err
