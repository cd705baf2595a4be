// Driver for N-body tuning variants: includes the production kernel source compiled with
// different NB_*_CFG macros and times the fused C2 workload (p = 2^20 targets vs
// 2^20 positions + 129^3 weighted grid nodes) with CUDA events.
#include "../../paper_2108_02991_b200/csrc/nbody.cu"

#include <cstdlib>
#include <vector>

int main() {
    const long long p = 1 << 20, g = 129LL * 129 * 129;
    std::vector<float4> hp(p), hg(g);
    srand(1);
    auto u = [] { return 2.f * rand() / (float)RAND_MAX - 1.f; };
    for (auto& v : hp) v = make_float4(u(), u(), u(), 1.f);
    for (long long c = 0; c < g; ++c) {
        const long long i = c / (129 * 129), j = (c / 129) % 129, k = c % 129;
        hg[c] = make_float4((i - 64) / 64.f, (j - 64) / 64.f, (k - 64) / 64.f, 1.f / g);
    }
    float4 *dp, *dg;
    double *va, *ga, *vr, *gr;
    cudaMalloc(&dp, p * 16);
    cudaMalloc(&dg, g * 16);
    cudaMemcpy(dp, hp.data(), p * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, hg.data(), g * 16, cudaMemcpyHostToDevice);
    cudaMalloc(&va, p * 8);
    cudaMalloc(&vr, p * 8);
    cudaMalloc(&ga, p * 24);
    cudaMalloc(&gr, p * 24);
    size_t wsb = spk_nbody_workspace_bytes(p, g, p);
    void* ws;
    cudaMalloc(&ws, wsb);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(s);
        int rc = spk_fused_sums(dp, p, 3, dg, g, 1.f / (128.f * 128.f), dp, p, 1e-6f, va, ga, vr,
                                gr, ws, wsb, nullptr);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        if (rc) {
            printf("error %s\n", spk_last_error());
            return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        if (ms < best) best = ms;
    }
    const double pairs = (double)p * p + (double)p * g;
    const double flops = (double)p * p * 17 + (double)p * g * 19;
    printf("TPT=%d THREADS=%d UNROLL=%d MINB=%d STAGES=%d slots=%d : %.1f ms  %.4g pairs/s  %.2f TFLOP/s\n",
           NB_TPT, NB_THREADS, NB_UNROLL_CFG, NB_MINBLOCKS_CFG, NB_STAGES, spk::nbody_slots(),
           best, pairs / (best * 1e-3), flops / (best * 1e-3) / 1e12);
    return 0;
}
