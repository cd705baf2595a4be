// Microbenchmark: FP32 pipe throughput on B200 for scalar FFMA, packed FFMA2 (f32x2),
// a 1:1 mix, and MUFU.RSQ.  Prints achieved lane-ops / clk / SM and TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_ffma(float* out, float a, float b) {
    float x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[CH];
    for (int i = 0; i < CH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = __ffma2_rn(x[i], A, B);
    float s = 0;
    for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_mix(float* out, float a, float b) {
    float2 x[CH / 2];
    float y[CH / 2];
    for (int i = 0; i < CH / 2; ++i) {
        x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        y[i] = i * 0.25f;
    }
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) {
            x[i] = __ffma2_rn(x[i], A, B);
            y[i] = fmaf(y[i], a, b);
        }
    float s = 0;
    for (int i = 0; i < CH / 2; ++i) s += x[i].x + x[i].y + y[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_rsq(float* out, float a) {
    float x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i + 1.0f;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            float r;
            asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
            x[i] = r + a;
        }
    float s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    auto run = [&](const char* name, auto launch, double lane_ops_per_inner) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(s);
        for (int r = 0; r < 10; ++r) launch();
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        double ops = 10.0 * blocks * threads * (double)ITERS * lane_ops_per_inner;
        double per_s = ops / (ms * 1e-3);
        printf("%-8s %10.3f ms  %8.2f Gops/s  %7.2f ops/clk/SM (at %d MHz)\n", name, ms,
               per_s / 1e9, per_s / sms / (clk * 1e3), clk / 1000);
    };
    run("ffma", [&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-4f); }, CH);
    run("ffma2", [&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-4f); }, 2 * CH);
    run("mix", [&] { k_mix<<<blocks, threads>>>(out, 0.999f, 1e-4f); }, 3 * CH / 2);
    run("rsqrt", [&] { k_rsq<<<blocks, threads>>>(out, 1e-6f); }, CH);
    printf("(ops = FP32 lane operations; an FFMA counts once; FLOP = 2x for FFMA)\n");
    return 0;
}
