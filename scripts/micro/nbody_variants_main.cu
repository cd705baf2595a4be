// Driver for N-body tuning variants: includes the production kernel source compiled with
// different NB_*_CFG macros and times the fused C2 workload (p = 2^20 targets vs
// 2^20 positions + 129^3 weighted grid nodes) with CUDA events.  NBV_P (positions),
// NBV_T (targets: the first T positions) and NBV_SIDES ("s0,s1,s2") change the shape,
// e.g. the C4 mix: NBV_P=8388608 NBV_T=1048576 NBV_SIDES=385,385,209.
#include "../../paper_2108_02991_b200/csrc/nbody.cu"

#include <cstdlib>
#include <vector>

int main() {
    const long long p = getenv("NBV_P") ? atoll(getenv("NBV_P")) : (1 << 20);
    const long long nt = getenv("NBV_T") ? atoll(getenv("NBV_T")) : p;
    int64_t side[3] = {129, 129, 129};
    if (getenv("NBV_SIDES"))
        sscanf(getenv("NBV_SIDES"), "%ld,%ld,%ld", &side[0], &side[1], &side[2]);
    const long long g = side[0] * side[1] * side[2];
    std::vector<float4> hp(p);
    std::vector<float> hg((g + 3) / 4 * 4, 0.f);
    srand(1);
    auto u = [] { return 2.f * rand() / (float)RAND_MAX - 1.f; };
    for (auto& v : hp) {
        v = make_float4(u(), u(), u(), 0.f);
        v.w = v.x * v.x + v.y * v.y + v.z * v.z;
    }
    for (long long c = 0; c < g; ++c) hg[c] = 1.f / g;
    float4* dp;
    float* dg;
    double *va, *ga, *vr, *gr;
    cudaMalloc(&dp, p * 16);
    cudaMalloc(&dg, hg.size() * 4);
    cudaMemcpy(dp, hp.data(), p * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, hg.data(), hg.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&va, p * 8);
    cudaMalloc(&vr, p * 8);
    cudaMalloc(&ga, p * 24);
    cudaMalloc(&gr, p * 24);
    size_t wsb = spk_nbody_workspace_bytes(nt, g, p);
    void* ws;
    cudaMalloc(&ws, wsb);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(s);
        int rc = spk_fused_sums(dp, nt, 3, dg, side, 1.f / (128.f * 128.f), dp, p, 1e-6f, va, ga,
                                vr, gr, ws, wsb, nullptr);
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
    const double pairs = (double)nt * p + (double)nt * g;
    const double flops = (double)nt * p * 17 + (double)nt * g * 19;
    // checksum of the outputs (compare variants)
    std::vector<double> h(nt);
    cudaMemcpy(h.data(), va, nt * 8, cudaMemcpyDeviceToHost);
    double cs_a = 0, cs_r = 0;
    for (long long i = 0; i < nt; ++i) cs_a += h[i];
    cudaMemcpy(h.data(), vr, nt * 8, cudaMemcpyDeviceToHost);
    for (long long i = 0; i < nt; ++i) cs_r += h[i];
    printf("sum(val_att) %.12e sum(val_rep) %.12e\n", cs_a, cs_r);
    printf("TPT=%d THREADS=%d UNROLL=%d MINB=%d STAGES=%d slots=%d : %.1f ms  %.4g pairs/s  %.2f TFLOP/s\n",
           NB_TPT, NB_THREADS, NB_UNROLL_CFG, NB_MINBLOCKS_CFG, NB_STAGES, spk::nbody_slots(),
           best, pairs / (best * 1e-3), flops / (best * 1e-3) / 1e12);
    return 0;
}
