mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/nbody_once.py 3 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -5 gpurun_out/pytest_gpu.log; grep drift gpurun_out/pytest_gpu.log
timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/profile_step.json 2> gpurun_out/profile_step.err
echo "profile exit $?"
python -c "import json; d=json.load(open('gpurun_out/profile_step.json')); [print(k, v['mean_ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
