#!/bin/bash
# FMA-pipe + SFU co-issue ceiling (scripts/micro/mix_peak.cu).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mix_peak scripts/micro/mix_peak.cu || exit 1
timeout 300 gpurun_out/mix_peak | tee gpurun_out/mix_peak.txt
