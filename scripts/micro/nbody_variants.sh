# Build and time N-body tuning variants (run from the repo root on a GPU box).
set -e
mkdir -p gpurun_out/variants
for cfg in "8 256 2 2 4" "8 256 4 2 4" "8 256 1 2 4" "12 256 2 1 4" "6 256 2 2 4" "4 256 4 3 4" "8 128 2 4 4" "16 128 2 2 4"; do
  set -- $cfg
  out=gpurun_out/variants/nb_$1_$2_$3_$4_$5
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
      -DNB_TPT_CFG=$1 -DNB_THREADS_CFG=$2 -DNB_UNROLL_CFG=$3 -DNB_MINBLOCKS_CFG=$4 -DNB_STAGES_CFG=$5 \
      -Xptxas -v -o $out scripts/micro/nbody_variants_main.cu 2> $out.ptxas || { echo "build failed $cfg"; continue; }
  grep -A1 "nbody_kernelILi3" $out.ptxas | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '
  timeout 120 $out || echo "run failed $cfg"
done
