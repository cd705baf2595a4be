// nbody.cu -- K1 (repulsion) and K2 (attraction) all-pairs sums for sm_100a.
//
// Replaces the reference's O(p^2) numba loops: direct_sums / direct_sums_subset
// (/root/reference/pkg/src/vdtraj/_treecode.py:474-534) and, for the north-star exact
// attraction, the density-weighted sum that precompute_field evaluates by FFT
// (attraction.py:62-113).
//
// Design:
//  * Work unit = (target block of NB_TB targets) x (source chunk).  Units are sized on
//    the host so that their count fills 148 SMs evenly; every unit writes its fp64
//    partial sums to its own workspace slot and a second kernel adds the slots in a
//    fixed order => bitwise run-to-run determinism without float atomics.
//  * Source tiles (NB_TILE float4 records) are staged into shared memory with 1-D bulk
//    TMA (cp.async.bulk + mbarrier complete_tx), NB_STAGES deep.  Every thread reads
//    each source record with one broadcast LDS.128.
//  * Each thread owns NB_TPT targets as NB_TPT/2 packed f32x2 pairs: one FADD2/FFMA2/
//    FMUL2 instruction advances two pair-interactions; the reciprocal square root runs
//    on the SFU (MUFU.RSQ).  Per pair (3D, unweighted): 3 FADD + 3 FFMA (r^2) + 1 MUFU
//    + 1 FFMA (value) + 3 FFMA (gradient) = 17 flops, 10 FP32 lane-ops, 1 MUFU.
//  * fp32 accumulation inside a tile, folded into fp64 per tile (relative gradient
//    error vs the fp64 reference ~1e-6, well inside the 1e-4 north-star bound).
#include <algorithm>
#include <cfloat>
#include <cstdarg>
#include <cstring>

#include "spk_common.cuh"

namespace spk {

// Tuning knobs (overridable at compile time for scripts/micro/nbody_variants.sh).
#ifndef NB_THREADS_CFG
#define NB_THREADS_CFG 256
#endif
#ifndef NB_TPT_CFG
#define NB_TPT_CFG 8
#endif
#ifndef NB_UNROLL_CFG
#define NB_UNROLL_CFG 2
#endif
#ifndef NB_MINBLOCKS_CFG
#define NB_MINBLOCKS_CFG 2
#endif
#ifndef NB_STAGES_CFG
#define NB_STAGES_CFG 4
#endif
constexpr int NB_THREADS = NB_THREADS_CFG;
constexpr int NB_TPT = NB_TPT_CFG;          // targets per thread
constexpr int NB_PAIRS = NB_TPT / 2;        // f32x2 pairs per thread
constexpr int NB_TB = NB_THREADS * NB_TPT;  // targets per CTA
constexpr int NB_TILE = 512;                // sources per shared-memory stage
constexpr int NB_STAGES = NB_STAGES_CFG;
constexpr int NB_UNROLL = NB_UNROLL_CFG;
constexpr int NB_TILE_BYTES = NB_STAGES * NB_TILE * 16;
// fp64 per-target accumulators live in shared memory (per-thread slots) so that the
// kernel fits 128 registers and two CTAs (16 warps) share an SM.
constexpr int NB_ACC_BYTES = NB_TPT * 4 * NB_THREADS * 8;
constexpr int NB_AXES_BYTES = 3 * 1024 * 4;  // lattice node tables (NB_AXIS_MAX per axis)
constexpr int NB_SMEM = NB_TILE_BYTES + NB_ACC_BYTES + NB_AXES_BYTES;
constexpr int NB_MAX_CHUNKS = 64;

// Source segment.  kind 0: positions, float4 {x, y, z, |x|^2} records (unweighted,
// repulsion).  kind 1: the density lattice -- fp32 weights w[c] for the node grid
// s0 x s1 (x s2), node coordinates implicit ((i - N_a)/N_a, density.py:58-67).
struct SegDesc {
    const void* src;
    long long n;      // records (kind 0) or cells (kind 1)
    long long tiles;  // ceil(n / tile size)
    int n_chunks;     // chunks this segment is split into (0 if empty)
    int kind;
    float eps2;
    int s0, s1, s2;   // lattice sides (kind 1); s2 = 1 in 2D
};

struct NBParams {
    const float4* tgt;
    long long n_tgt;
    long long n_tb;
    SegDesc seg[2];
    double* part;  // [chunk][4][n_tgt]: value, gx, gy, gz
    // Independent problems batched in one launch (stack-of-SPARKLING, C3): targets are
    // n_groups contiguous groups of per_group; group q's position sources start at
    // record q * src_stride.  A single problem has n_groups = 1, src_stride = 0.
    long long per_group;
    long long tb_per_group;
    long long src_stride;
    // optional: CTAs wait until their SM holds no polish CTA (polish_kernel's count), so a
    // launch beside the polish takes only the SMs the polish has left
    const int* sm_busy;
};

constexpr int NB_TILE_W = NB_TILE;  // lattice cells per stage (fp32 partials span <= 512 cells)
constexpr int NB_AXIS_MAX = 1024;       // per-axis node table capacity (shared memory)

__device__ __forceinline__ float rsqrt_sfu(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// Positions tile against this thread's NB_TPT targets (difference form).
// G: guard r2 below the fp32 normal range (eps2 < FLT_MIN, incl. eps = 0 => coincident
// points contribute value 0, gradient 0, like the reference's `if h > 0` at
// _treecode.py:525; for 0 < eps < 1.1e-19 the dropped value is eps itself).
template <int D, bool G>
__device__ __forceinline__ void tile_positions(const float4* __restrict__ tile, int cnt,
                                               const float2 (&X)[NB_PAIRS],
                                               const float2 (&Y)[NB_PAIRS],
                                               const float2 (&Z)[NB_PAIRS], float2 e2,
                                               float2 (&av)[NB_PAIRS], float2 (&ax)[NB_PAIRS],
                                               float2 (&ay)[NB_PAIRS],
                                               float2 (&az)[NB_PAIRS]) {
#pragma unroll NB_UNROLL
    for (int j = 0; j < cnt; ++j) {
        const float4 s = tile[j];
        const float2 nsx = bc(-s.x);
        const float2 nsy = bc(-s.y);
        const float2 nsz = bc(-s.z);
#pragma unroll
        for (int k = 0; k < NB_PAIRS; ++k) {
            const float2 dx = __fadd2_rn(X[k], nsx);
            const float2 dy = __fadd2_rn(Y[k], nsy);
            float2 r2 = __ffma2_rn(dx, dx, e2);
            r2 = __ffma2_rn(dy, dy, r2);
            float2 dz;
            if (D == 3) {
                dz = __fadd2_rn(Z[k], nsz);
                r2 = __ffma2_rn(dz, dz, r2);
            }
            float2 inv;
            inv.x = rsqrt_sfu(r2.x);
            inv.y = rsqrt_sfu(r2.y);
            if (G) {
                inv.x = r2.x >= FLT_MIN ? inv.x : 0.0f;  // rsqrt.approx.ftz flushes subnormal r2
                inv.y = r2.y >= FLT_MIN ? inv.y : 0.0f;
            }
            av[k] = __ffma2_rn(r2, inv, av[k]);  // sum h = sum r2 / h
            ax[k] = __ffma2_rn(dx, inv, ax[k]);
            ay[k] = __ffma2_rn(dy, inv, ay[k]);
            if (D == 3) az[k] = __ffma2_rn(dz, inv, az[k]);
        }
    }
}

// Lattice tile: cells [c0, c0 + cnt) of the density grid.  Cells are walked row by row
// (a row = all nodes along the last axis with the other coordinates fixed), so along a
// row only the last-axis difference dl changes: per target and row
//     a = dx^2 (+ dy^2) + eps^2,  and per cell
//     r2 = dl^2 + a,  winv = w / h,  v += r2 winv,  S += winv,  g_last += dl winv
// then g_other += d_other * S at the end of the row.  6 FP32 lane-ops + 1 MUFU per pair
// (the reference's algorithmic count stays 19 flops per pair).
template <int D, bool G>
__device__ __forceinline__ void tile_lattice(const float* __restrict__ tile, long long c0, int cnt,
                                             const SegDesc& S, const float* __restrict__ axes,
                                             const float2 (&X)[NB_PAIRS],
                                             const float2 (&Y)[NB_PAIRS],
                                             const float2 (&Z)[NB_PAIRS], float2 e2,
                                             float2 (&av)[NB_PAIRS], float2 (&ax)[NB_PAIRS],
                                             float2 (&ay)[NB_PAIRS],
                                             float2 (&az)[NB_PAIRS]) {
    const int R = D == 3 ? S.s2 : S.s1;  // row length
    const float* AX = axes;
    const float* AY = axes + S.s0;
    const float* AL = D == 3 ? axes + S.s0 + S.s1 : AY;  // last-axis table
    long long row = c0 / R;
    int k = (int)(c0 - row * R);
    int done = 0;
    while (done < cnt) {
        const int n_run = min(R - k, cnt - done);
        // per-row constants
        float2 d0[NB_PAIRS], d1[NB_PAIRS], A[NB_PAIRS], Sw[NB_PAIRS];
        if (D == 3) {
            const int i = (int)(row / S.s1), j = (int)(row - (long long)(row / S.s1) * S.s1);
            const float2 nxi = bc(-AX[i]), nyj = bc(-AY[j]);
#pragma unroll
            for (int q = 0; q < NB_PAIRS; ++q) {
                d0[q] = __fadd2_rn(X[q], nxi);
                d1[q] = __fadd2_rn(Y[q], nyj);
                A[q] = __ffma2_rn(d1[q], d1[q], __ffma2_rn(d0[q], d0[q], e2));
                Sw[q] = bc(0.f);
            }
        } else {
            const float2 nxi = bc(-AX[(int)row]);
#pragma unroll
            for (int q = 0; q < NB_PAIRS; ++q) {
                d0[q] = __fadd2_rn(X[q], nxi);
                A[q] = __ffma2_rn(d0[q], d0[q], e2);
                Sw[q] = bc(0.f);
            }
        }
        const float* wrow = tile + done;
        const float* lrow = AL + k;
#pragma unroll 4
        for (int m = 0; m < n_run; ++m) {
            const float w = wrow[m];
            const float2 nl = bc(-lrow[m]);
#pragma unroll
            for (int q = 0; q < NB_PAIRS; ++q) {
                const float2 dl = __fadd2_rn(D == 3 ? Z[q] : Y[q], nl);
                const float2 r2 = __ffma2_rn(dl, dl, A[q]);
                float2 inv;
                inv.x = rsqrt_sfu(r2.x);
                inv.y = rsqrt_sfu(r2.y);
                if (G) {
                    inv.x = r2.x >= FLT_MIN ? inv.x : 0.0f;  // rsqrt.approx.ftz flushes subnormal r2
                    inv.y = r2.y >= FLT_MIN ? inv.y : 0.0f;
                }
                const float2 winv = __fmul2_rn(inv, bc(w));
                av[q] = __ffma2_rn(r2, winv, av[q]);
                Sw[q] = __fadd2_rn(Sw[q], winv);
                if (D == 3) az[q] = __ffma2_rn(dl, winv, az[q]);
                else ay[q] = __ffma2_rn(dl, winv, ay[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < NB_PAIRS; ++q) {
            ax[q] = __ffma2_rn(d0[q], Sw[q], ax[q]);
            if (D == 3) ay[q] = __ffma2_rn(d1[q], Sw[q], ay[q]);
        }
        done += n_run;
        k = 0;
        ++row;
    }
}

template <int D, int KIND, bool G>
__device__ __forceinline__ void run_chunk(const SegDesc& S, long long t_begin, long long t_end,
                                          char* stages, uint64_t* bars, const float* axes,
                                          const float2 (&X)[NB_PAIRS],
                                          const float2 (&Y)[NB_PAIRS],
                                          const float2 (&Z)[NB_PAIRS], double* acc) {
    const int tid = threadIdx.x;
    const float2 e2 = bc(S.eps2);
    constexpr int TILE = KIND == 0 ? NB_TILE : NB_TILE_W;
    constexpr int REC = KIND == 0 ? 16 : 4;
    constexpr int STAGE_BYTES = NB_TILE * 16;
    auto issue = [&](long long t, int stage) {
        const long long first = t * TILE;
        const long long cnt = min((long long)TILE, S.n - first);
        const uint32_t bytes = (uint32_t)(((cnt * REC) + 15) & ~15LL);  // weights padded
        mbar_expect_tx(&bars[stage], bytes);
        tma_load_1d(stages + stage * STAGE_BYTES,
                    static_cast<const char*>(S.src) + first * REC, bytes, &bars[stage]);
    };
    if (tid == 0) {
        for (int s = 0; s < NB_STAGES; ++s)
            if (t_begin + s < t_end) issue(t_begin + s, s);
    }
    for (long long t = t_begin; t < t_end; ++t) {
        const long long i = t - t_begin;
        const int stage = (int)(i % NB_STAGES);
        const uint32_t parity = (uint32_t)((i / NB_STAGES) & 1);
        const int cnt = (int)min((long long)TILE, S.n - t * TILE);
        float2 av[NB_PAIRS], ax[NB_PAIRS], ay[NB_PAIRS], az[NB_PAIRS];
#pragma unroll
        for (int k = 0; k < NB_PAIRS; ++k) {
            av[k] = ax[k] = ay[k] = az[k] = bc(0.f);
        }
        mbar_wait(&bars[stage], parity);
        if (KIND == 0)
            tile_positions<D, G>(reinterpret_cast<const float4*>(stages + stage * STAGE_BYTES),
                                 cnt, X, Y, Z, e2, av, ax, ay, az);
        else
            tile_lattice<D, G>(reinterpret_cast<const float*>(stages + stage * STAGE_BYTES),
                               t * TILE, cnt, S, axes, X, Y, Z, e2, av, ax, ay, az);
#define NB_ACC(k, c) acc[((k) * 4 + (c)) * NB_THREADS + tid]
#pragma unroll
        for (int k = 0; k < NB_PAIRS; ++k) {
            NB_ACC(2 * k, 0) += av[k].x;
            NB_ACC(2 * k + 1, 0) += av[k].y;
            NB_ACC(2 * k, 1) += ax[k].x;
            NB_ACC(2 * k + 1, 1) += ax[k].y;
            NB_ACC(2 * k, 2) += ay[k].x;
            NB_ACC(2 * k + 1, 2) += ay[k].y;
            if (D == 3) {
                NB_ACC(2 * k, 3) += az[k].x;
                NB_ACC(2 * k + 1, 3) += az[k].y;
            }
        }
        __syncthreads();  // every warp is done with this stage
        if (tid == 0 && t + NB_STAGES < t_end) issue(t + NB_STAGES, stage);
    }
}

template <int D>
__global__ void __launch_bounds__(NB_THREADS, NB_MINBLOCKS_CFG) nbody_kernel(const NBParams P) {
    extern __shared__ __align__(128) char stages[];
    double* acc = reinterpret_cast<double*>(stages + NB_TILE_BYTES);
    float* axes = reinterpret_cast<float*>(stages + NB_TILE_BYTES + NB_ACC_BYTES);
    __shared__ __align__(8) uint64_t bars[NB_STAGES];
    const int tid = threadIdx.x;
    if (P.sm_busy) {
        if (tid == 0) {
            const volatile int* busy = P.sm_busy + sm_id();
            while (*busy > 0) __nanosleep(20000);
        }
        __syncthreads();
    }
    // Interleave the lattice (SFU-bound) and position (FMA-bound) units in launch order,
    // in proportion to their counts (Bresenham), so that the CTAs resident on an SM mix
    // both kinds and the two pipes overlap instead of running one phase after the other.
    // Unit k of a segment is (tb = k % n_tb, chunk k / n_tb): slots and the fixed-order
    // finalize are unchanged.
    const long long u = blockIdx.x;
    const long long U0 = P.n_tb * P.seg[0].n_chunks;
    const long long U = U0 + P.n_tb * P.seg[1].n_chunks;
    const long long i0 = u * U0 / U;
    const bool first = (u + 1) * U0 / U > i0;
    const long long k = first ? i0 : u - i0;
    const long long tb = k % P.n_tb;
    const int chunk = (int)(k / P.n_tb) + (first ? 0 : P.seg[0].n_chunks);
    const SegDesc S = first ? P.seg[0] : P.seg[1];
    const long long lc = first ? chunk : chunk - P.seg[0].n_chunks;
    const long long t_begin = lc * S.tiles / S.n_chunks;
    const long long t_end = (lc + 1) * S.tiles / S.n_chunks;

    const long long grp = tb / P.tb_per_group;
    const long long gfirst = grp * P.per_group;  // first target of this problem
    const long long base = (tb - grp * P.tb_per_group) * NB_TB + tid;  // local index
    SegDesc Sg = S;
    if (S.kind == 0)
        Sg.src = static_cast<const float4*>(S.src) + grp * P.src_stride;
    float2 X[NB_PAIRS], Y[NB_PAIRS], Z[NB_PAIRS];
#pragma unroll
    for (int k = 0; k < NB_PAIRS; ++k) {
        const long long i0 = gfirst + min(base + (2 * k) * NB_THREADS, P.per_group - 1);
        const long long i1 = gfirst + min(base + (2 * k + 1) * NB_THREADS, P.per_group - 1);
        const float4 a = P.tgt[i0];
        const float4 b = P.tgt[i1];
        X[k] = make_float2(a.x, b.x);
        Y[k] = make_float2(a.y, b.y);
        Z[k] = make_float2(D == 3 ? a.z : 0.f, D == 3 ? b.z : 0.f);
    }
#pragma unroll
    for (int k = 0; k < NB_TPT * 4; ++k) acc[k * NB_THREADS + tid] = 0.0;
    if (S.kind == 1) {
        // node coordinate tables (i - N_a) / N_a, computed in fp64 then rounded
        const int sides[3] = {S.s0, S.s1, S.s2};
        int off = 0;
        for (int a = 0; a < D; ++a) {
            const int h = (sides[a] - 1) / 2;
            for (int i = tid; i < sides[a]; i += NB_THREADS)
                axes[off + i] = (float)((double)(i - h) / (double)h);
            off += sides[a];
        }
    }
    if (tid == 0) {
        for (int s = 0; s < NB_STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const bool guard = !(S.eps2 >= FLT_MIN);
    if (S.kind == 1) {
        if (guard) run_chunk<D, 1, true>(Sg, t_begin, t_end, stages, bars, axes, X, Y, Z, acc);
        else run_chunk<D, 1, false>(Sg, t_begin, t_end, stages, bars, axes, X, Y, Z, acc);
    } else {
        if (guard) run_chunk<D, 0, true>(Sg, t_begin, t_end, stages, bars, axes, X, Y, Z, acc);
        else run_chunk<D, 0, false>(Sg, t_begin, t_end, stages, bars, axes, X, Y, Z, acc);
    }

    double* slot = P.part + (size_t)chunk * 4 * P.n_tgt;
#pragma unroll
    for (int k = 0; k < NB_TPT; ++k) {
        const long long li = base + k * NB_THREADS;
        const long long i = gfirst + li;
        if (li < P.per_group) {
            slot[i] = NB_ACC(k, 0);
            slot[P.n_tgt + i] = NB_ACC(k, 1);
            slot[2 * P.n_tgt + i] = NB_ACC(k, 2);
            if (D == 3) slot[3 * P.n_tgt + i] = NB_ACC(k, 3);
        }
    }
}

// Fixed-order sum over the chunk slots of one segment.
__global__ void nbody_finalize(const double* __restrict__ part, long long n_tgt, int c_begin,
                               int c_end, int dims, double* __restrict__ val,
                               double* __restrict__ grad) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_tgt) return;
    double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int c = c_begin; c < c_end; ++c) {
        const double* slot = part + (size_t)c * 4 * n_tgt;
        v += slot[i];
        gx += slot[n_tgt + i];
        gy += slot[2 * n_tgt + i];
        if (dims == 3) gz += slot[3 * n_tgt + i];
    }
    if (val) val[i] = v;
    if (grad) {
        grad[i * dims] = gx;
        grad[i * dims + 1] = gy;
        if (dims == 3) grad[i * dims + 2] = gz;
    }
}

struct Plan {
    long long n_tb = 0;
    int nc0 = 0, nc1 = 0;
    size_t ws_bytes = 0;
};

static int nbody_slots() {
    static int slots = 0;
    if (slots == 0) {
        int occ = 0;
        cudaFuncSetAttribute(nbody_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             NB_SMEM);
        cudaFuncSetAttribute(nbody_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             NB_SMEM);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nbody_kernel<3>, NB_THREADS,
                                                          NB_SMEM) != cudaSuccess ||
            occ <= 0) {
            cudaGetLastError();
            occ = 1;
        }
        slots = num_sms() * occ;
    }
    return slots;
}

// Relative cost of one tile: a position tile is NB_TILE pairs per target at ~10 FP32
// lane-ops, a lattice tile NB_TILE_W pairs bounded by the SFU (16 / clk / SM).
constexpr double NB_COST_POS_TILE = NB_TILE / 12.8;
constexpr double NB_COST_LAT_TILE = NB_TILE_W / 16.0;

// Choose the chunk counts: minimise (waves x longest unit) + per-unit overhead, with the
// two segments split in proportion to their estimated cost.  seg0 is the lattice.
static Plan make_plan(long long n_tgt, long long n0, long long n1, long long n_groups = 1) {
    Plan pl;
    if (n_tgt <= 0) return pl;
    const long long per_group = n_tgt / n_groups;
    pl.n_tb = n_groups * ((per_group + NB_TB - 1) / NB_TB);
    const long long t0 = (n0 + NB_TILE_W - 1) / NB_TILE_W;
    const long long t1 = (n1 + NB_TILE - 1) / NB_TILE;
    const double w0 = t0 * NB_COST_LAT_TILE, w1 = t1 * NB_COST_POS_TILE;
    const long long slots = nbody_slots();
    double best = 1e300;
    const int cmin = (t0 > 0) + (t1 > 0);
    for (int c = std::max(cmin, 1); c <= NB_MAX_CHUNKS; ++c) {
        int c0 = 0, c1 = 0;
        if (t0 > 0 && t1 > 0) {
            c0 = (int)std::llround((double)c * w0 / (w0 + w1));
            c0 = std::max(1, std::min(c - 1, c0));
            c1 = c - c0;
        } else if (t0 > 0) {
            c0 = c;
        } else {
            c1 = c;
        }
        if ((t0 > 0 && c0 > t0) || (t1 > 0 && c1 > t1)) break;
        const double l0 = c0 ? (double)((t0 + c0 - 1) / c0) * NB_COST_LAT_TILE : 0.0;
        const double l1 = c1 ? (double)((t1 + c1 - 1) / c1) * NB_COST_POS_TILE : 0.0;
        const long long units = pl.n_tb * c;
        const long long waves = (units + slots - 1) / slots;
        // per-unit fixed cost ~ 0.25 position tile (prologue, pipeline fill, slot write)
        const double cost = (double)waves * (std::max(l0, l1) + 0.25 * NB_COST_POS_TILE);
        if (cost < best * 0.995) {
            best = cost;
            pl.nc0 = c0;
            pl.nc1 = c1;
        }
    }
    pl.ws_bytes = (size_t)(pl.nc0 + pl.nc1) * 4 * (size_t)n_tgt * sizeof(double);
    return pl;
}

// seg0 = lattice (weights w0 over `side`), seg1 = positions.
static int launch_sums(const float4* tgt, long long n_tgt, int dims, const float* w0,
                       const int64_t* side, float e0, const float4* s1, long long n1, float e1,
                       double* val0, double* grad0, double* val1, double* grad1, void* ws,
                       size_t ws_bytes, cudaStream_t stream, long long n_groups = 1,
                       const int* sm_busy = nullptr) {
    SPK_REQUIRE(n_groups >= 1 && n_tgt % n_groups == 0, SPK_ERR_ARG,
                "targets (%lld) must split evenly into %lld groups", n_tgt, n_groups);
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    long long n0 = 0;
    int sd[3] = {1, 1, 1};
    if (w0) {
        SPK_REQUIRE(side != nullptr, SPK_ERR_ARG, "lattice sides missing");
        n0 = 1;
        for (int a = 0; a < dims; ++a) {
            sd[a] = (int)side[a];
            SPK_REQUIRE(side[a] >= 3 && (side[a] & 1) && side[a] <= NB_AXIS_MAX, SPK_ERR_ARG,
                        "lattice sides must be odd, >= 3 and <= %d", NB_AXIS_MAX);
            n0 *= side[a];
        }
    }
    SPK_REQUIRE(n_tgt >= 0 && n1 >= 0, SPK_ERR_ARG, "negative size");
    if (n_tgt == 0 || (n0 == 0 && n1 == 0)) {
        // Empty sums: zero the outputs like a loop that never runs.
        if (n_tgt > 0) {
            if (val0) cudaMemsetAsync(val0, 0, n_tgt * 8, stream);
            if (grad0) cudaMemsetAsync(grad0, 0, n_tgt * dims * 8, stream);
            if (val1) cudaMemsetAsync(val1, 0, n_tgt * 8, stream);
            if (grad1) cudaMemsetAsync(grad1, 0, n_tgt * dims * 8, stream);
        }
        return SPK_OK;
    }
    SPK_REQUIRE(tgt != nullptr, SPK_ERR_ARG, "null target pointer");
    SPK_REQUIRE(((uintptr_t)w0 & 15) == 0 && ((uintptr_t)s1 & 15) == 0, SPK_ERR_ARG,
                "source arrays must be 16-byte aligned");
    const Plan pl = make_plan(n_tgt, n0, n1, n_groups);
    SPK_REQUIRE(ws != nullptr && ws_bytes >= pl.ws_bytes, SPK_ERR_WORKSPACE,
                "nbody workspace too small: need %zu bytes, got %zu", pl.ws_bytes, ws_bytes);
    NBParams P;
    P.tgt = tgt;
    P.n_tgt = n_tgt;
    P.n_tb = pl.n_tb;
    P.per_group = n_tgt / n_groups;
    P.tb_per_group = pl.n_tb / n_groups;
    P.src_stride = n_groups > 1 ? n1 : 0;
    P.sm_busy = sm_busy;
    P.seg[0] = SegDesc{w0, n0, (n0 + NB_TILE_W - 1) / NB_TILE_W, pl.nc0, 1, e0,
                       sd[0], sd[1], dims == 3 ? sd[2] : 1};
    P.seg[1] = SegDesc{s1, n1, (n1 + NB_TILE - 1) / NB_TILE, pl.nc1, 0, e1, 0, 0, 0};
    P.part = static_cast<double*>(ws);
    const long long grid = pl.n_tb * (pl.nc0 + pl.nc1);
    nbody_slots();  // sets the shared-memory attribute once
    if (dims == 3)
        nbody_kernel<3><<<(unsigned)grid, NB_THREADS, NB_SMEM, stream>>>(P);
    else
        nbody_kernel<2><<<(unsigned)grid, NB_THREADS, NB_SMEM, stream>>>(P);
    SPK_CHECK_LAUNCH("nbody_kernel");
    const unsigned fb = (unsigned)((n_tgt + 255) / 256);
    if (pl.nc0 > 0 && (val0 || grad0))
        nbody_finalize<<<fb, 256, 0, stream>>>(P.part, n_tgt, 0, pl.nc0, dims, val0, grad0);
    if (pl.nc1 > 0 && (val1 || grad1))
        nbody_finalize<<<fb, 256, 0, stream>>>(P.part, n_tgt, pl.nc0, pl.nc0 + pl.nc1, dims,
                                               val1, grad1);
    SPK_CHECK_LAUNCH("nbody_finalize");
    return SPK_OK;
}

// ------------------------------------------------------------------ packing kernels
__global__ void pack_positions_kernel(const double* __restrict__ c, long long p, int dims,
                                      float4* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= p) return;
    const double* r = c + i * dims;
    out[i] = pos_record(r[0], r[1], dims == 3 ? r[2] : 0.0);
}

// Lattice weights (fp32, zero-padded to a multiple of 4) and, optionally, the node
// position records {x, y, z, |x|^2} (targets for precompute_field).
__global__ void grid_sources_kernel(const double* __restrict__ rho, long long s0,
                                    long long s1, long long s2, int dims,
                                    float* __restrict__ w, float4* __restrict__ nodes) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long n = s0 * s1 * s2;
    const long long npad = (n + 3) & ~3LL;
    if (c >= npad) return;
    if (c >= n) {
        w[c] = 0.f;
        return;
    }
    w[c] = (float)rho[c];
    if (nodes) {
        const long long k = c % s2;
        const long long j = (c / s2) % s1;
        const long long i = c / (s1 * s2);
        const long long h0 = (s0 - 1) / 2, h1 = (s1 - 1) / 2, h2 = (s2 - 1) / 2;
        const double x = (double)(i - h0) / (double)h0;
        const double y = (double)(j - h1) / (double)h1;
        const double z = dims == 3 ? (double)(k - h2) / (double)h2 : 0.0;
        nodes[c] = pos_record(x, y, z);
    }
}

// ------------------------------------------------------------ gradient combination
constexpr int CB_THREADS = 256;

__global__ void combine_kernel(long long n, long long per_group, int dims,
                               const double* __restrict__ va,
                               const double* __restrict__ ga, double pa,
                               const double* __restrict__ vr, const double* __restrict__ gr,
                               double pr, const double* __restrict__ coords,
                               const double* __restrict__ prev_c,
                               const double* __restrict__ prev_g, double* __restrict__ grad,
                               double* __restrict__ block_out) {
    __shared__ double red[5][CB_THREADS];
    // blockIdx.y = group (problem); blocks never straddle two problems
    const long long li = blockIdx.x * (long long)CB_THREADS + threadIdx.x;
    const long long i = blockIdx.y * per_group + li;
    double s_va = 0, s_vr = 0, s_kg = 0, s_gg = 0, s_nf = 0;
    if (li < per_group && i < n) {
        if (va) s_va = va[i];
        if (vr) s_vr = vr[i];
        const double prr = pr * pr;
        for (int l = 0; l < dims; ++l) {
            const long long e = i * dims + l;
            double g = 0.0;
            if (ga) g = ga[e] / pa;
            if (gr) g = g - gr[e] / prr;
            grad[e] = g;
            if (!isfinite(g)) s_nf += 1.0;
            if (prev_c && prev_g) {
                const double dk = coords[e] - prev_c[e];
                const double dg = g - prev_g[e];
                s_kg += dk * dg;
                s_gg += dg * dg;
            }
        }
    }
    red[0][threadIdx.x] = s_va;
    red[1][threadIdx.x] = s_vr;
    red[2][threadIdx.x] = s_kg;
    red[3][threadIdx.x] = s_gg;
    red[4][threadIdx.x] = s_nf;
    __syncthreads();
    for (int w = CB_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 5; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 5)
        block_out[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 5 + threadIdx.x] =
            red[threadIdx.x][0];
}

__global__ void combine_final_kernel(const double* __restrict__ block_out, long long nb,
                                     double* __restrict__ out_all) {
    // one block per group: fixed-order sum of that group's nb block partials
    __shared__ double red[5][CB_THREADS];
    const double* bo = block_out + (long long)blockIdx.x * nb * 5;
    double* out = out_all + (long long)blockIdx.x * 6;
    double s[5] = {0, 0, 0, 0, 0};
    for (long long b = threadIdx.x; b < nb; b += CB_THREADS)
        for (int q = 0; q < 5; ++q) s[q] += bo[b * 5 + q];
    for (int q = 0; q < 5; ++q) red[q][threadIdx.x] = s[q];
    __syncthreads();
    for (int w = CB_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 5; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 5) out[threadIdx.x] = red[threadIdx.x][0];
    if (threadIdx.x == 5) out[5] = 0.0;
}

// --------------------------------------------------------------------- error text
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// Rows of a shot subset: gather the listed shots' target records into a contiguous
// buffer, and scatter per-target results back to their rows (val [n], grad [n][dims]).
__global__ void gather_shot_rows_kernel(const float4* __restrict__ src,
                                        const int32_t* __restrict__ ids, long long n_ids,
                                        int n_s, float4* __restrict__ dst) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_ids * n_s) return;
    const long long k = i / n_s;
    dst[i] = src[(long long)ids[k] * n_s + (i - k * n_s)];
}

__global__ void scatter_shot_rows_kernel(const double* __restrict__ v, const double* __restrict__ g,
                                         const int32_t* __restrict__ ids, long long n_ids,
                                         int n_s, int dims, double* __restrict__ val,
                                         double* __restrict__ grad) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_ids * n_s) return;
    const long long k = i / n_s;
    const long long r = (long long)ids[k] * n_s + (i - k * n_s);
    val[r] = v[i];
    for (int l = 0; l < dims; ++l) grad[r * dims + l] = g[i * dims + l];
}

}  // namespace spk

using namespace spk;

extern "C" {

int spk_version(void) { return 1; }

const char* spk_last_error(void) { return g_err; }

// CUDA IPC for the fused position all-gather (engine.ShardedRun._setup_peers): the other
// ranks' buffers are opened on the CALLER's current device, so peer access from this
// device to the owner's is enabled (cudaIpcMemLazyEnablePeerAccess).
int spk_ipc_handle(const void* base, void* handle_out) {
    SPK_REQUIRE(base != nullptr && handle_out != nullptr, SPK_ERR_ARG, "ipc: null pointer");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(base));
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle_out, &h, sizeof(h));
    return SPK_OK;
}

int spk_ipc_open(const void* handle, void** ptr_out) {
    SPK_REQUIRE(handle != nullptr && ptr_out != nullptr, SPK_ERR_ARG, "ipc: null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "cudaIpcOpenMemHandle: %s",
                cudaGetErrorString(e));
    return SPK_OK;
}

int spk_ipc_close(void* ptr) {
    const cudaError_t e = cudaIpcCloseMemHandle(ptr);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "cudaIpcCloseMemHandle: %s",
                cudaGetErrorString(e));
    return SPK_OK;
}

size_t spk_nbody_workspace_bytes(int64_t n_tgt, int64_t n_src0, int64_t n_src1) {
    return make_plan(n_tgt, n_src0, n_src1).ws_bytes + 256;
}

size_t spk_nbody_batched_workspace_bytes(int64_t n_groups, int64_t per_group, int64_t n_cells,
                                         int64_t n_pos) {
    return make_plan(n_groups * per_group, n_cells, n_pos, n_groups).ws_bytes + 256;
}

int spk_fused_sums_batched(const void* tgt, int64_t n_groups, int64_t per_group, int dims,
                           const float* grid_w, const int64_t* side, float eps2_att,
                           const void* pos_src, int64_t n_pos, float eps2_rep,
                           double* val_att, double* grad_att, double* val_rep,
                           double* grad_rep, void* ws, size_t ws_bytes, spk_stream_t stream) {
    return launch_sums((const float4*)tgt, n_groups * per_group, dims, grid_w, side, eps2_att,
                       (const float4*)pos_src, n_pos, eps2_rep, val_att, grad_att, val_rep,
                       grad_rep, ws, ws_bytes, (cudaStream_t)stream, n_groups);
}

int spk_direct_sums(const void* tgt, int64_t n_tgt, const void* src, int64_t n_src, int dims,
                    float eps2, double* val, double* grad, void* ws, size_t ws_bytes,
                    spk_stream_t stream) {
    return launch_sums((const float4*)tgt, n_tgt, dims, nullptr, nullptr, 0.f,
                       (const float4*)src, n_src, eps2, nullptr, nullptr, val, grad, ws,
                       ws_bytes, (cudaStream_t)stream);
}

int spk_grid_sums(const void* tgt, int64_t n_tgt, const float* grid_w, const int64_t* side,
                  int dims, float eps2, double* val, double* grad, void* ws, size_t ws_bytes,
                  spk_stream_t stream) {
    return launch_sums((const float4*)tgt, n_tgt, dims, grid_w, side, eps2, nullptr, 0, 0.f,
                       val, grad, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

static size_t shot_rows_scratch(int64_t n_rows) {
    return ((size_t)n_rows * (16 + 8 + 24) + 255) & ~(size_t)255;
}

size_t spk_grid_sums_shots_workspace_bytes(int64_t n_ids, int n_s, int64_t n_cells) {
    return shot_rows_scratch(n_ids * n_s) + spk_nbody_workspace_bytes(n_ids * n_s, n_cells, 0);
}

int spk_grid_sums_shots(const void* tgt, const int32_t* shot_ids, int64_t n_ids, int n_s,
                        const float* grid_w, const int64_t* side, int dims, float eps2,
                        double* val, double* grad, const int32_t* sm_busy, void* ws,
                        size_t ws_bytes, spk_stream_t stream_) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(n_ids >= 0 && n_s >= 1, SPK_ERR_ARG, "shot subset: bad sizes");
    if (n_ids == 0) return SPK_OK;
    SPK_REQUIRE(shot_ids != nullptr, SPK_ERR_ARG, "shot subset: null shot list");
    const long long n = n_ids * n_s;
    long long n_cells = 1;
    for (int a = 0; a < dims; ++a) n_cells *= side[a];
    SPK_REQUIRE(ws != nullptr && ws_bytes >= spk_grid_sums_shots_workspace_bytes(n_ids, n_s, n_cells),
                SPK_ERR_WORKSPACE, "grid sums (shot subset): workspace too small");
    cudaStream_t stream = (cudaStream_t)stream_;
    char* p = static_cast<char*>(ws);
    float4* t4 = reinterpret_cast<float4*>(p);
    double* v = reinterpret_cast<double*>(p + (size_t)n * 16);
    double* g = v + n;
    const size_t scratch = shot_rows_scratch(n);
    const unsigned nb = (unsigned)((n + 255) / 256);
    gather_shot_rows_kernel<<<nb, 256, 0, stream>>>((const float4*)tgt, shot_ids, n_ids, n_s, t4);
    SPK_CHECK_LAUNCH("grid_sums_shots(gather)");
    const int rc = launch_sums(t4, n, dims, grid_w, side, eps2, nullptr, 0, 0.f, v, g, nullptr,
                               nullptr, p + scratch, ws_bytes - scratch, stream, 1, sm_busy);
    if (rc != SPK_OK) return rc;
    scatter_shot_rows_kernel<<<nb, 256, 0, stream>>>(v, g, shot_ids, n_ids, n_s, dims, val, grad);
    SPK_CHECK_LAUNCH("grid_sums_shots(scatter)");
    return SPK_OK;
}

int spk_fused_sums(const void* tgt, int64_t n_tgt, int dims, const float* grid_w,
                   const int64_t* side, float eps2_att, const void* pos_src, int64_t n_pos,
                   float eps2_rep, double* val_att, double* grad_att, double* val_rep,
                   double* grad_rep, void* ws, size_t ws_bytes, spk_stream_t stream) {
    return launch_sums((const float4*)tgt, n_tgt, dims, grid_w, side, eps2_att,
                       (const float4*)pos_src, n_pos, eps2_rep, val_att, grad_att, val_rep,
                       grad_rep, ws, ws_bytes, (cudaStream_t)stream);
}

int spk_pack_positions(const double* coords, int64_t p, int dims, void* pos4,
                       spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    if (p <= 0) return SPK_OK;
    pack_positions_kernel<<<(unsigned)((p + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        coords, p, dims, (float4*)pos4);
    SPK_CHECK_LAUNCH("pack_positions");
    return SPK_OK;
}

int spk_build_grid_sources(const double* rho, int dims, const int64_t* side, float* weights,
                           void* nodes, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    const long long s0 = side[0], s1 = side[1], s2 = dims == 3 ? side[2] : 1;
    SPK_REQUIRE(s0 >= 3 && s1 >= 3 && s2 >= 1 && (s0 & 1) && (s1 & 1) && (s2 & 1),
                SPK_ERR_ARG, "grid sides must be odd (2N+1) and >= 3");
    const long long npad = (s0 * s1 * s2 + 3) & ~3LL;
    grid_sources_kernel<<<(unsigned)((npad + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        rho, s0, s1, s2, dims, weights, (float4*)nodes);
    SPK_CHECK_LAUNCH("grid_sources");
    return SPK_OK;
}

size_t spk_combine_workspace_bytes(int64_t n) {
    return (size_t)((n + CB_THREADS - 1) / CB_THREADS) * 5 * sizeof(double) + 256;
}

int spk_combine_gradient(int64_t n_tgt, int dims, const double* val_att,
                         const double* grad_att, double p_att, const double* val_rep,
                         const double* grad_rep, double p_rep, const double* coords,
                         const double* prev_coords, const double* prev_grad, double* grad,
                         double* out, void* ws, size_t ws_bytes, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    SPK_REQUIRE(n_tgt > 0, SPK_ERR_ARG, "n_tgt must be positive");
    SPK_REQUIRE(ws_bytes >= spk_combine_workspace_bytes(n_tgt), SPK_ERR_WORKSPACE,
                "combine workspace too small");
    const long long nb = (n_tgt + CB_THREADS - 1) / CB_THREADS;
    double* bo = static_cast<double*>(ws);
    combine_kernel<<<dim3((unsigned)nb, 1), CB_THREADS, 0, (cudaStream_t)stream>>>(
        n_tgt, n_tgt, dims, val_att, grad_att, p_att, val_rep, grad_rep, p_rep, coords,
        prev_coords, prev_grad, grad, bo);
    combine_final_kernel<<<1, CB_THREADS, 0, (cudaStream_t)stream>>>(bo, nb, out);
    SPK_CHECK_LAUNCH("combine_gradient");
    return SPK_OK;
}

size_t spk_combine_batched_workspace_bytes(int64_t n_groups, int64_t per_group) {
    return (size_t)n_groups * ((per_group + CB_THREADS - 1) / CB_THREADS) * 5 * sizeof(double) +
           256;
}

int spk_combine_gradient_batched(int64_t n_groups, int64_t per_group, int dims,
                                 const double* val_att, const double* grad_att, double p_att,
                                 const double* val_rep, const double* grad_rep, double p_rep,
                                 const double* coords, const double* prev_coords,
                                 const double* prev_grad, double* grad, double* out, void* ws,
                                 size_t ws_bytes, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    SPK_REQUIRE(n_groups >= 1 && per_group >= 1, SPK_ERR_ARG, "empty batch");
    SPK_REQUIRE(ws_bytes >= spk_combine_batched_workspace_bytes(n_groups, per_group),
                SPK_ERR_WORKSPACE, "combine workspace too small");
    const long long nb = (per_group + CB_THREADS - 1) / CB_THREADS;
    double* bo = static_cast<double*>(ws);
    combine_kernel<<<dim3((unsigned)nb, (unsigned)n_groups), CB_THREADS, 0,
                     (cudaStream_t)stream>>>(n_groups * per_group, per_group, dims, val_att,
                                             grad_att, p_att, val_rep, grad_rep, p_rep, coords,
                                             prev_coords, prev_grad, grad, bo);
    combine_final_kernel<<<(unsigned)n_groups, CB_THREADS, 0, (cudaStream_t)stream>>>(bo, nb,
                                                                                       out);
    SPK_CHECK_LAUNCH("combine_gradient_batched");
    return SPK_OK;
}

}  // extern "C"
