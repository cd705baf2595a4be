// DFMA / FFMA2 throughput microbenchmark (roofline denominators for the fp64 NUDFT).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 20000;
    for (int threads : {128, 256, 512}) {
        for (int per_sm : {2, 4, 8}) {
            int blocks = sms * per_sm;
            dfma_kernel<<<blocks, threads>>>(out, 100, 0.999, 1e-3);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double n = (double)blocks * threads * iters * 16;
            printf("{\"threads\": %d, \"blocks_per_sm\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.2f}\n",
                   threads, per_sm, n / (ms * 1e-3), 2 * n / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
