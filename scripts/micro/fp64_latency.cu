// Dependent-chain latency of fp64 ops on B200 (single warp): DADD, DMUL, IEEE sqrt,
// IEEE div, and a warp shuffle of a double.  Prints cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
#define N 4096
__global__ void k(double* out, double a, double b, long long* cyc) {
    double x = threadIdx.x * 1e-3 + 1.5;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x + a;
    t1 = clock64(); cyc[0] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x * b;
    t1 = clock64(); cyc[1] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = sqrt(x + a);
    t1 = clock64(); cyc[2] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = b / (x + a);
    t1 = clock64(); cyc[3] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + a;
    t1 = clock64(); cyc[4] = t1 - t0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { x = x + a; __syncthreads(); }
    t1 = clock64(); cyc[5] = t1 - t0;
    out[threadIdx.x] = x;
}
int main() {
    double* out; long long* cyc; long long h[6];
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 6 * 8);
    const char* names[6] = {"dadd", "dmul", "sqrt+dadd", "div+dadd", "shfl.f64+dadd", "dadd+bar(256thr)"};
    k<<<1, 32>>>(out, 1e-9, 0.999999, cyc);
    cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 5; ++i) printf("%-18s %8.1f cycles/iter (1 warp)\n", names[i], (double)h[i] / N);
    k<<<1, 256>>>(out, 1e-9, 0.999999, cyc);
    cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
    printf("%-18s %8.1f cycles/iter (8 warps)\n", names[5], (double)h[5] / N);
    return 0;
}
