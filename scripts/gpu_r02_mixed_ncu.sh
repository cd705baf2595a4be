#!/bin/bash
# (historical: the mixed-kind kernel and SPK_NB_MIXED were removed after this A/B)
# ncu of the mixed-kind N-body kernel (micro driver, C2 mix).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -o gpurun_out/nbv scripts/micro/nbody_variants_main.cu || exit 1
SPK_NB_MIXED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:nbody_mixed -c 1 -o gpurun_out/mixed_ncu gpurun_out/nbv > gpurun_out/mixed_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/mixed_ncu.log
