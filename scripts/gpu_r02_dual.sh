#!/bin/bash
# (historical: the dual-kind kernel and SPK_NB_DUAL / ND_*_CFG were removed after this A/B; see profiles/r02_ab_nbody_dual.txt)
# Dual-kind persistent N-body kernel: A/B against the unit-per-CTA kernel, parity tests, bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o gpurun_out/nbv scripts/micro/nbody_variants_main.cu > /dev/null 2>&1 || echo "micro build failed"
for r in 1 2; do for d in 0 1; do echo -n "dual=$d "; SPK_NB_DUAL=$d timeout 120 gpurun_out/nbv; done; done
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_optimize.py tests/test_gpu_stack.py tests/test_gpu_fuzz.py -q -x > gpurun_out/gputest_dual.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_dual.log
for d in 0 1; do SPK_NB_DUAL=$d timeout 900 python bench.py --steps 10 --warmup 3 --no-sub --no-cpu-baseline > gpurun_out/bench_dual$d.json 2> gpurun_out/bench_dual$d.err; python -c "import json; d=json.loads(open('gpurun_out/bench_dual$d.json').read().strip().splitlines()[-1]); print('dual=$d', d['ms_per_step'], d['roofline']['achieved'], d['roofline'].get('frac'), d['e2e']['s_per_iteration'])"; done
