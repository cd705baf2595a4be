mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o gpurun_out/fp64_latency scripts/micro/fp64_latency.cu && ./gpurun_out/fp64_latency | tee gpurun_out/fp64_latency.log
