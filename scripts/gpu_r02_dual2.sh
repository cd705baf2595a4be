#!/bin/bash
# (historical: the dual-kind kernel and SPK_NB_DUAL / ND_*_CFG were removed after this A/B; see profiles/r02_ab_nbody_dual.txt)
# Dual-kind N-body kernel: targets per thread x TMA stages (micro driver, C2-sized workload).
mkdir -p gpurun_out/dual
echo -n "unit-per-CTA: "; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o gpurun_out/dual/nb_ref scripts/micro/nbody_variants_main.cu && SPK_NB_DUAL=0 timeout 120 gpurun_out/dual/nb_ref
for cfg in "8 2" "6 2" "6 3" "4 2" "4 4"; do
  set -- $cfg
  out=gpurun_out/dual/nb_$1_$2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -DND_TPT_CFG=$1 -DND_STAGES_CFG=$2 -o $out scripts/micro/nbody_variants_main.cu || { echo "build failed $cfg"; continue; }
  echo -n "dual TPT=$1 STAGES=$2: "; SPK_NB_DUAL=1 timeout 120 $out || echo "run failed $cfg"
done
