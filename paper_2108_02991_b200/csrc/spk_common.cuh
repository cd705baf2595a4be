// spk_common.cuh -- shared helpers for the sm_100a kernels behind the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "sparkling_b200.h"

namespace spk {

// Thread-local last error text for spk_last_error() (include/sparkling_b200.h).
void set_error(const char* fmt, ...);

#define SPK_CHECK_LAUNCH(what)                                                   \
    do {                                                                         \
        cudaError_t e__ = cudaGetLastError();                                    \
        if (e__ != cudaSuccess) {                                                \
            ::spk::set_error("%s: %s", what, cudaGetErrorString(e__));           \
            return SPK_ERR_LAUNCH;                                               \
        }                                                                        \
    } while (0)

#define SPK_REQUIRE(cond, code, ...)                                             \
    do {                                                                         \
        if (!(cond)) {                                                           \
            ::spk::set_error(__VA_ARGS__);                                       \
            return code;                                                         \
        }                                                                        \
    } while (0)

inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// The SM this thread runs on (%smid: < 256 on B200).
__device__ __forceinline__ int sm_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return (int)r;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Position record {x, y, z, |x|^2} consumed by the N-body kernels (fp32; the norm is
// computed from the rounded coordinates with explicit roundings, identical in every TU).
__device__ __forceinline__ float4 pos_record(double x, double y, double z) {
    const float fx = (float)x, fy = (float)y, fz = (float)z;
    return make_float4(fx, fy, fz, __fmaf_rn(fx, fx, __fmaf_rn(fy, fy, __fmul_rn(fz, fz))));
}

// ---- mbarrier + 1-D bulk TMA (cp.async.bulk) --------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}
// Global -> shared bulk copy completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src,
                                            uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace spk
