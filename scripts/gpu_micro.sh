mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/fp32_peak scripts/micro/fp32_peak.cu
./gpurun_out/fp32_peak > gpurun_out/fp32_peak.log 2>&1 && cat gpurun_out/fp32_peak.log && \
ncu --metrics sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -s 0 -c 4 ./gpurun_out/fp32_peak > gpurun_out/fp32_ncu.log 2>&1
grep -E "k_|fma|xu" gpurun_out/fp32_ncu.log | head -40
