// Microbenchmark: can the FMA pipe (packed FFMA2) and the SFU (MUFU.RSQ) run concurrently
// at full rate on B200?  Each thread runs NF independent FFMA2 chains and NM independent
// rsqrt chains per iteration, with no memory traffic.  The same loop with only the FFMA2
// part and with only the MUFU part gives T_F and T_M; a perfect overlap would run the mix
// in max(T_F, T_M).  The mixes are the N-body launch's executed instruction mixes:
// per 2 x 3 pairs at C2 (1 position : 2 lattice pairs) 22 FFMA2-class + 6 MUFU, at C4
// (1 : 3.66) ~32 + 9.3, and a pipe-balanced 24 + 6.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_peak mix_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 16384

__device__ __forceinline__ float rsq(float x) {
    float r;
    asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int NF, int NM>
__global__ void __launch_bounds__(256) k_mix(float* out, float a, float b) {
    float2 f[NF > 0 ? NF : 1];
    float m[NM > 0 ? NM : 1];
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
    for (int j = 0; j < NM; ++j) m[j] = threadIdx.x * 1e-3f + j + 1.5f;
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < (NF > NM ? NF : NM); ++k) {
            if (k < NF) f[k] = __ffma2_rn(f[k], A, B);
            if (k < NM) m[k] = rsq(m[k]);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NF; ++i) s += f[i].x + f[i].y;
#pragma unroll
    for (int j = 0; j < NM; ++j) s += m[j];
    if (s == 1234.5f) out[0] = s;
}

template <int NF, int NM>
float time_kernel(float* out, int blocks) {
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    for (int w = 0; w < 2; ++w) k_mix<NF, NM><<<blocks, 256>>>(out, 0.999f, 1e-3f);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(s);
        k_mix<NF, NM><<<blocks, 256>>>(out, 0.999f, 1e-3f);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        if (ms < best) best = ms;
    }
    return best;
}

template <int NF, int NM>
void run(const char* name, float* out, int blocks) {
    const float tf = time_kernel<NF, 0>(out, blocks);
    const float tm = time_kernel<0, NM>(out, blocks);
    const float tx = time_kernel<NF, NM>(out, blocks);
    const float bound = tf > tm ? tf : tm;
    printf("%-28s FFMA2 x%-2d alone %7.3f ms | MUFU x%-2d alone %7.3f ms | mix %7.3f ms | "
           "max(alone)/mix = %.3f\n",
           name, NF, tf, NM, tm, tx, bound / tx);
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {2, 4, 8}) {
        const int blocks = sms * occ;
        printf("-- %d CTAs x 256 threads per SM (%d warps / sub-partition)\n", occ, occ * 2);
        run<22, 6>("C2 mix (1:2)", out, blocks);
        run<32, 9>("C4 mix (1:3.66)", out, blocks);
        run<24, 6>("pipe-balanced", out, blocks);
        run<10, 2>("positions only (K1)", out, blocks);
        run<6, 2>("lattice only (K2)", out, blocks);
    }
    return 0;
}
