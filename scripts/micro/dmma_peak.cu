// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) throughput on B200 next to the DFMA pipe
// (scripts/micro/dfma_peak.cu): is the fp64 NUDFT adjoint's GEMM-shaped inner product
// worth moving from DFMA to DMMA?  Each warp runs NACC independent accumulator tiles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_kernel(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5 - threadIdx.x * 1e-6;
    double c[NACC][2];
#pragma unroll
    for (int k = 0; k < NACC; ++k) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
                "{%0, %1};"
                : "+d"(c[k][0]), "+d"(c[k][1])
                : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 20000;
    for (int threads : {128, 256}) {
        for (int per_sm : {2, 4, 8}) {
            const int blocks = sms * per_sm;
            dmma_kernel<8><<<blocks, threads>>>(out, 100);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            dmma_kernel<8><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // one m8n8k4 = 8 x 8 x 4 = 256 FMA per warp
            const double fma = (double)blocks * (threads / 32) * iters * 8 * 256;
            printf("{\"threads\": %d, \"blocks_per_sm\": %d, \"dmma_fma_per_s\": %.4e, "
                   "\"fp64_tc_tflops\": %.2f}\n",
                   threads, per_sm, fma / (ms * 1e-3), 2 * fma / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
