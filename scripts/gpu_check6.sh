mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/polish_latency.py 1600 1,592,1024 2>&1 | tail -3
timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/profile_step.json 2> gpurun_out/profile_step.err
python -c "import json; d=json.load(open('gpurun_out/profile_step.json')); [print(k, v['mean_ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
