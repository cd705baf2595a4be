mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
for w in 8 4 2 1; do
  SPK_POLISH_WARPS=$w timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/ps_w$w.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ps_w$w.json')); print('W=$w', 'project', round(d['project']['mean_ms'],1), 'nbody', round(d['nbody']['mean_ms'],1))"
done
