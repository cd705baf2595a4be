#!/bin/bash
# (historical: the dual-kind kernel and SPK_NB_DUAL / ND_*_CFG were removed after this A/B; see profiles/r02_ab_nbody_dual.txt)
# ncu of the dual-kind N-body kernel (micro driver, C2-sized uniform workload).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -o gpurun_out/nbv scripts/micro/nbody_variants_main.cu > /dev/null 2>&1 || echo "micro build failed"
SPK_NB_DUAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:nbody_dual -c 1 -o gpurun_out/dual_ncu gpurun_out/nbv > gpurun_out/dual_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/dual_ncu.log
