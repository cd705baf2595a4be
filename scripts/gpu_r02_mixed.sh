#!/bin/bash
# (historical: the mixed-kind kernel and SPK_NB_MIXED were removed after this A/B)
# Mixed-kind N-body kernel (both kinds in one warp's instruction stream): A/B vs the
# unit-per-CTA kernel (SPK_NB_MIXED=0) at the C2 and C4 mixes, then the parity tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -o gpurun_out/nbv scripts/micro/nbody_variants_main.cu || exit 1
for m in 0 1; do echo "== C2 mixed=$m"; SPK_NB_MIXED=$m timeout 120 gpurun_out/nbv; done
for m in 0 1; do echo "== C4 mix (1M targets) mixed=$m"; SPK_NB_MIXED=$m NBV_P=8388608 NBV_T=1048576 NBV_SIDES=385,385,209 timeout 300 gpurun_out/nbv; done
timeout 900 python -m pytest tests/test_gpu_nbody.py tests/test_gpu_optimize.py tests/test_gpu_stack.py tests/test_gpu_fuzz.py tests/test_gpu_abi_errors.py -q -x > gpurun_out/gputest_mixed.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_mixed.log
