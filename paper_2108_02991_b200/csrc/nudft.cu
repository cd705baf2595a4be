// nudft.cu -- direct nonuniform DFT between trajectory samples and the image grid
// (density compensation and the PSF of a pattern).
//
// Replaces the reference's numpy phase-table products (analysis.py:25-69):
//   adjoint  out[r] = sum_i w_i exp(+i pi k_i . r)            (nudft_adjoint)
//   forward  f_i    = sum_r img[r] exp(-i pi k_i . r)          (nudft_forward)
// with r_a = 0..n_a-1 minus n_a/2 (integer voxel offsets) and k in [-1, 1]^d.
//
// Both are complex GEMM-shaped sums with generated operands.  The grid is split as
// U x V (3D: U = (a, b), V = c; 2D: U = a, V = b):
//   adjoint: out[u, v] = sum_i A_i[u] B_i[v],  A = e0 e1 (3D) or w e0 (2D),
//            B = w e2 (3D) or e1 (2D); one CTA owns a 64 (u) x 32 (v) output tile and
//            a slice of the samples, phase tables for 128 samples are generated in fp64
//            by recurrence from one sincospi per row (exact start, fp64 steps) and stored
//            as fp32 complex in shared memory; each thread accumulates 16 products per
//            sample with packed FFMA, folding into fp64 every 128 samples.
//   forward: one thread per sample; for every u the inner sum over v is a Horner
//            polynomial in zeta = exp(-i pi k_v) (4 FFMA per voxel, image rows broadcast
//            from shared memory), multiplied by conj(A_i[u]) kept by an fp32 recurrence
//            re-seeded from fp64 at every 8-row stage and row wrap.
// Deterministic: fixed sample slices per CTA and a fixed-order reduction of the slices.
#include <algorithm>
#include <cmath>
#include <cfloat>

#include "spk_common.cuh"

namespace spk {

constexpr int NU_THREADS = 128;
constexpr int NU_UT = 64;   // u per adjoint tile
constexpr int NU_VT = 32;   // v per adjoint tile
constexpr int NU_VPT = 16;  // v per thread
#ifndef NU_CH_CFG
#define NU_CH_CFG 64
#endif
constexpr int NU_CH = NU_CH_CFG;  // samples per shared-memory chunk (48 KB of tables)
constexpr int NF_UT = 8;    // image rows (u) per forward stage
constexpr int NF_VMAX = 1024;

struct C2 {
    float x, y;
};
// Table row strides (complex elements), padded so that the row-per-thread generation
// does not put a whole warp on one shared-memory bank; B rows stay 16-byte aligned for
// the float4 reads of the product loop.
constexpr int NU_AS = NU_UT + 1;
constexpr int NU_BS = NU_VT + 2;

// B rows are stored as (re_2k, re_2k+1, im_2k, im_2k+1) quadruples so that one float4
// load yields the packed real and imaginary pairs the FFMA2s consume.
__device__ __forceinline__ void put_b(C2* row, int q, double2 v) {
    float* f = reinterpret_cast<float*>(row) + (q >> 1) * 4 + (q & 1);
    f[0] = (float)v.x;
    f[2] = (float)v.y;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// exp(i pi t) in fp64 (sincospi is exact in its argument reduction).
__device__ __forceinline__ double2 cispi(double t) {
    double s, c;
    sincospi(t, &s, &c);
    return make_double2(c, s);
}

struct AdjParams {
    const double* pts;   // [p][dims]
    const double* w;     // [p][2] complex weights (re, im)
    long long p;
    int dims;
    int n0, n1, n2;      // grid (2D: n2 = 1)
    long long U, V;      // U x V split of the grid
    int slices;          // sample slices (split-K)
    double* part;        // [slices][U][V][2]
};

// Generated operand tables for one chunk of samples.
__global__ void __launch_bounds__(NU_THREADS, 4) nudft_adjoint_kernel(const AdjParams P) {
    extern __shared__ __align__(16) char sm[];
    C2* At = reinterpret_cast<C2*>(sm);                  // [NU_CH][NU_AS]
    C2* Bt = At + ((NU_CH * NU_AS + 1) & ~1);            // [NU_CH][NU_BS], 16-B aligned
    const int tid = threadIdx.x;
    const long long u0 = (long long)blockIdx.x * NU_UT;
    const long long v0 = (long long)blockIdx.y * NU_VT;
    const int slice = blockIdx.z;
    const long long i_begin = P.p * slice / P.slices;
    const long long i_end = P.p * (slice + 1) / P.slices;
    const int u_loc = tid % NU_UT;
    const int vg = tid / NU_UT;  // 0..1 -> v in [vg*16, vg*16+16)
    double acc[NU_VPT][2];
#pragma unroll
    for (int k = 0; k < NU_VPT; ++k) acc[k][0] = acc[k][1] = 0.0;
    const int h0 = P.n0 / 2, h1 = P.n1 / 2, h2 = P.n2 / 2;

    for (long long c0 = i_begin; c0 < i_end; c0 += NU_CH) {
        const int cnt = (int)min((long long)NU_CH, i_end - c0);
        // ---- tables: work item r < NU_CH builds A row r, r >= NU_CH builds B row r - NU_CH
        for (int r = tid; r < 2 * NU_CH; r += NU_THREADS) {
            const bool rowA = r < NU_CH;
            const int j = rowA ? r : r - NU_CH;
            const long long i = c0 + j;
            if (j >= cnt) {
                if (rowA)
                    for (int q = 0; q < NU_UT; ++q) At[j * NU_AS + q] = C2{0.f, 0.f};
                else
                    for (int q = 0; q < NU_VT; ++q) Bt[j * NU_BS + q] = C2{0.f, 0.f};  // any layout
                continue;
            }
            const double k0 = P.pts[i * P.dims];
            const double k1 = P.pts[i * P.dims + 1];
            const double2 wi = make_double2(P.w[2 * i], P.w[2 * i + 1]);
            if (P.dims == 3) {
                if (rowA) {
                    // A[u] = e0[a] e1[b], u = a * n1 + b, over this tile's u range
                    int a = (int)(u0 / P.n1), b = (int)(u0 - (long long)a * P.n1);
                    double2 e0 = cispi(k0 * (double)(a - h0));
                    double2 e1 = cispi(k1 * (double)(b - h1));
                    const double2 z1 = cispi(k1);
                    for (int q = 0; q < NU_UT; ++q) {
                        const double2 v = cmul(e0, e1);
                        At[j * NU_AS + q] = C2{(float)v.x, (float)v.y};
                        if (++b == P.n1) {
                            b = 0;
                            ++a;
                            e0 = cispi(k0 * (double)(a - h0));
                            e1 = cispi(k1 * (double)(b - h1));
                        } else {
                            e1 = cmul(e1, z1);
                        }
                    }
                } else {
                    // B[v] = w e2[c], v = c
                    const double k2 = P.pts[i * P.dims + 2];
                    double2 e2 = cmul(wi, cispi(k2 * (double)(v0 - h2)));
                    const double2 z2 = cispi(k2);
                    for (int q = 0; q < NU_VT; ++q) {
                        put_b(Bt + j * NU_BS, q, e2);
                        e2 = cmul(e2, z2);
                    }
                }
            } else if (rowA) {
                double2 e0 = cmul(wi, cispi(k0 * (double)(u0 - h0)));
                const double2 z0 = cispi(k0);
                for (int q = 0; q < NU_UT; ++q) {
                    At[j * NU_AS + q] = C2{(float)e0.x, (float)e0.y};
                    e0 = cmul(e0, z0);
                }
            } else {
                double2 e1 = cispi(k1 * (double)(v0 - h1));
                const double2 z1 = cispi(k1);
                for (int q = 0; q < NU_VT; ++q) {
                    put_b(Bt + j * NU_BS, q, e1);
                    e1 = cmul(e1, z1);
                }
            }
        }
        __syncthreads();
        // ---- products: out[u, v] += A[u] B[v]
        float2 re[NU_VPT / 2], im[NU_VPT / 2];  // packed over v pairs
#pragma unroll
        for (int k = 0; k < NU_VPT / 2; ++k) re[k] = im[k] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = 0; j < cnt; ++j) {
            const C2 a = At[j * NU_AS + u_loc];
            const float4* brow = reinterpret_cast<const float4*>(Bt + j * NU_BS + vg * NU_VPT);
            const float2 ax = make_float2(a.x, a.x), ay = make_float2(a.y, a.y);
            const float2 nay = make_float2(-a.y, -a.y);
#pragma unroll
            for (int k = 0; k < NU_VPT / 2; ++k) {
                const float4 b = brow[k];  // (re, re, im, im) of v = 2k, 2k + 1
                const float2 br = make_float2(b.x, b.y), bi = make_float2(b.z, b.w);
                re[k] = __ffma2_rn(ax, br, re[k]);
                re[k] = __ffma2_rn(nay, bi, re[k]);
                im[k] = __ffma2_rn(ax, bi, im[k]);
                im[k] = __ffma2_rn(ay, br, im[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < NU_VPT / 2; ++k) {
            acc[2 * k][0] += re[k].x;
            acc[2 * k + 1][0] += re[k].y;
            acc[2 * k][1] += im[k].x;
            acc[2 * k + 1][1] += im[k].y;
        }
        __syncthreads();
    }
    const long long u = u0 + u_loc;
    if (u >= P.U) return;
    double* out = P.part + ((size_t)slice * P.U + u) * P.V * 2;
#pragma unroll
    for (int k = 0; k < NU_VPT; ++k) {
        const long long v = v0 + vg * NU_VPT + k;
        if (v < P.V) {
            out[2 * v] = acc[k][0];
            out[2 * v + 1] = acc[k][1];
        }
    }
}

__global__ void nudft_reduce_kernel(const double* __restrict__ part, int slices, long long n,
                                    double* __restrict__ out) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= n) return;
    double s = 0.0;
    for (int q = 0; q < slices; ++q) s += part[(size_t)q * n + e];
    out[e] = s;
}

struct FwdParams {
    const double* pts;  // [p][dims]
    const double* img;  // [U][V][2]
    long long p;
    int dims;
    int n0, n1, n2;
    long long U, V;
    int slices;         // u slices (split-K)
    double* part;       // [slices][p][2]
};

__global__ void __launch_bounds__(NU_THREADS) nudft_forward_kernel(const FwdParams P) {
    extern __shared__ __align__(16) char sm[];
    float2* rows = reinterpret_cast<float2*>(sm);  // [NF_UT][V]
    const int tid = threadIdx.x;
    const long long i = (long long)blockIdx.x * NU_THREADS + tid;
    const int slice = blockIdx.y;
    const long long ub = P.U * slice / P.slices, ue = P.U * (slice + 1) / P.slices;
    const bool live = i < P.p;
    const long long ii = live ? i : P.p - 1;
    const double k0 = P.pts[ii * P.dims];
    const double k1 = P.pts[ii * P.dims + 1];
    const double kv = P.dims == 3 ? P.pts[ii * P.dims + 2] : k1;
    const int hv = (P.dims == 3 ? P.n2 : P.n1) / 2;
    // zeta = exp(-i pi k_v); the Horner sum over v is sum_v img[u, v] zeta^v, then times
    // zeta^(-hv) = exp(+i pi k_v hv)
    const double2 zd = cispi(-kv);
    const float zr = (float)zd.x, zi = (float)zd.y;
    const double2 shift = cispi(kv * (double)hv);
    // per-u step of conj(A): exp(-i pi k_b) along b (3D) or exp(-i pi k0) along a (2D)
    const double2 wd = cispi(-(P.dims == 3 ? k1 : k0));
    const float wr = (float)wd.x, wi = (float)wd.y;
    double fr = 0.0, fi = 0.0;
    for (long long s0 = ub; s0 < ue; s0 += NF_UT) {
        const int nu = (int)min((long long)NF_UT, ue - s0);
        __syncthreads();
        for (long long e = tid; e < (long long)nu * P.V; e += NU_THREADS) {
            const double* src = P.img + ((size_t)s0 * P.V + e) * 2;
            rows[e] = make_float2((float)src[0], (float)src[1]);
        }
        __syncthreads();
        float cr = 0.f, ci = 0.f;  // sum over this stage's rows of conj(A[u]) P_u
        // conj(A[u]) = exp(-i pi (k0 (a - h0) [+ k1 (b - h1)])): exact fp64 seed at the
        // stage start and at row wraps, fp32 steps by exp(-i pi k_b) in between
        float ar = 0.f, ai = 0.f;
        int a = 0, b = 0;
        for (int q = 0; q < nu; ++q) {
            const long long u = s0 + q;
            bool seed = q == 0;
            if (P.dims == 3) {
                if (q == 0) {
                    a = (int)(u / P.n1);
                    b = (int)(u - (long long)a * P.n1);
                } else if (++b == P.n1) {
                    b = 0;
                    ++a;
                    seed = true;
                }
            }
            if (seed) {
                const double t = P.dims == 3
                                     ? k0 * (double)(a - P.n0 / 2) + k1 * (double)(b - P.n1 / 2)
                                     : k0 * (double)(u - P.n0 / 2);
                const double2 ad = cispi(-t);
                ar = (float)ad.x;
                ai = (float)ad.y;
            } else {
                const float nr = fmaf(ar, wr, -ai * wi);
                ai = fmaf(ar, wi, ai * wr);
                ar = nr;
            }
            const float2* row = rows + (size_t)q * P.V;
            float pr = 0.f, pi = 0.f;
            for (long long v = P.V - 1; v >= 0; --v) {  // Horner: p = p zeta + img[v]
                const float2 g = row[v];
                const float nr = fmaf(pr, zr, fmaf(-pi, zi, g.x));
                pi = fmaf(pr, zi, fmaf(pi, zr, g.y));
                pr = nr;
            }
            cr = fmaf(ar, pr, fmaf(-ai, pi, cr));
            ci = fmaf(ar, pi, fmaf(ai, pr, ci));
        }
        fr += (double)cr;
        fi += (double)ci;
    }
    if (live) {
        // times zeta^(-hv)
        const double2 f = cmul(make_double2(fr, fi), shift);
        double* out = P.part + ((size_t)slice * P.p + i) * 2;
        out[0] = f.x;
        out[1] = f.y;
    }
}

// ---------------------------------------------------------------------------------------
// fp64 kernels (the default, SPK_NUDFT_FP64).  Same decomposition as above with fp64
// tables and DFMA products.  density_compensation's fixed-point iteration amplifies
// relative noise in forward(adjoint(w)) by ~1e6 (a 1e-7 perturbation moves the weights by
// ~20% on a 3D radial pattern), so the reference's results are reproduced only with fp64
// products; the mixed kernels above are the opt-in fast mode.
constexpr int ND_CH = 64;            // samples per chunk
constexpr int ND_AS = NU_UT + 1;     // double2 row strides
constexpr int ND_BS = NU_VT + 1;  // odd row stride: the row-per-thread B generation
                                 // would otherwise put a quarter-warp on the same banks

__global__ void __launch_bounds__(NU_THREADS, 2) nudft_adjoint64_kernel(const AdjParams P) {
    extern __shared__ __align__(16) char sm[];
    double2* At = reinterpret_cast<double2*>(sm);        // [ND_CH][ND_AS]
    double2* Bt = At + ND_CH * ND_AS;                    // [ND_CH][ND_BS]
    const int tid = threadIdx.x;
    const long long u0 = (long long)blockIdx.x * NU_UT;
    const long long v0 = (long long)blockIdx.y * NU_VT;
    const int slice = blockIdx.z;
    const long long i_begin = P.p * slice / P.slices;
    const long long i_end = P.p * (slice + 1) / P.slices;
    const int u_loc = tid % NU_UT;
    const int vg = tid / NU_UT;
    double re[NU_VPT], im[NU_VPT];
#pragma unroll
    for (int k = 0; k < NU_VPT; ++k) re[k] = im[k] = 0.0;
    const int h0 = P.n0 / 2, h1 = P.n1 / 2, h2 = P.n2 / 2;

    for (long long c0 = i_begin; c0 < i_end; c0 += ND_CH) {
        const int cnt = (int)min((long long)ND_CH, i_end - c0);
        for (int r = tid; r < 2 * ND_CH; r += NU_THREADS) {
            const bool rowA = r < ND_CH;
            const int j = rowA ? r : r - ND_CH;
            if (j >= cnt) continue;  // rows past cnt are never read
            const long long i = c0 + j;
            const double k0 = P.pts[i * P.dims];
            const double k1 = P.pts[i * P.dims + 1];
            const double2 wi = make_double2(P.w[2 * i], P.w[2 * i + 1]);
            double2* row = rowA ? At + j * ND_AS : Bt + j * ND_BS;
            if (P.dims == 3) {
                if (rowA) {
                    int a = (int)(u0 / P.n1), b = (int)(u0 - (long long)a * P.n1);
                    double2 e0 = cispi(k0 * (double)(a - h0));
                    double2 e1 = cispi(k1 * (double)(b - h1));
                    const double2 z1 = cispi(k1);
                    for (int q = 0; q < NU_UT; ++q) {
                        row[q] = cmul(e0, e1);
                        if (++b == P.n1) {
                            b = 0;
                            ++a;
                            e0 = cispi(k0 * (double)(a - h0));
                            e1 = cispi(k1 * (double)(b - h1));
                        } else {
                            e1 = cmul(e1, z1);
                        }
                    }
                } else {
                    const double k2 = P.pts[i * P.dims + 2];
                    double2 e2 = cmul(wi, cispi(k2 * (double)(v0 - h2)));
                    const double2 z2 = cispi(k2);
                    for (int q = 0; q < NU_VT; ++q) {
                        row[q] = e2;
                        e2 = cmul(e2, z2);
                    }
                }
            } else if (rowA) {
                double2 e0 = cmul(wi, cispi(k0 * (double)(u0 - h0)));
                const double2 z0 = cispi(k0);
                for (int q = 0; q < NU_UT; ++q) {
                    row[q] = e0;
                    e0 = cmul(e0, z0);
                }
            } else {
                double2 e1 = cispi(k1 * (double)(v0 - h1));
                const double2 z1 = cispi(k1);
                for (int q = 0; q < NU_VT; ++q) {
                    row[q] = e1;
                    e1 = cmul(e1, z1);
                }
            }
        }
        __syncthreads();
#pragma unroll 2
        for (int j = 0; j < cnt; ++j) {
            const double2 a = At[j * ND_AS + u_loc];
            const double2* brow = Bt + j * ND_BS + vg * NU_VPT;
#pragma unroll
            for (int k = 0; k < NU_VPT; ++k) {
                const double2 b = brow[k];
                re[k] = fma(a.x, b.x, re[k]);
                re[k] = fma(-a.y, b.y, re[k]);
                im[k] = fma(a.x, b.y, im[k]);
                im[k] = fma(a.y, b.x, im[k]);
            }
        }
        __syncthreads();
    }
    const long long u = u0 + u_loc;
    if (u >= P.U) return;
    double* out = P.part + ((size_t)slice * P.U + u) * P.V * 2;
#pragma unroll
    for (int k = 0; k < NU_VPT; ++k) {
        const long long v = v0 + vg * NU_VPT + k;
        if (v < P.V) {
            out[2 * v] = re[k];
            out[2 * v + 1] = im[k];
        }
    }
}

// ---------------------------------------------------------------------------------------
// fp64 adjoint on the FP64 tensor cores (the default; SPK_NUDFT_DMMA=0 selects the DFMA
// kernel above).  Same tiles, chunks and fp64 generated tables; the products run as
// mma.sync.m8n8k4.f64 (DMMA: 256 fp64 FMA per warp instruction, measured 1.86e13 FMA/s
// vs 1.70e13 for DFMA, scripts/micro/dmma_peak.cu) with the complex product split into
// four real MMAs, Re += Ar Br + (-Ai) Bi and Im += Ar Bi + Ai Br.  Warp w owns the
// u-blocks 2w, 2w+1 (8 u each) against the four 8-wide v-blocks of the tile: 8 output
// tiles, 32 DMMA per 4 samples.  The tables are stored transposed, [u][sample] and
// [v][sample]: fragment lane = 4 r + c reads sample 4 ks + c of u (A) or v (B) = block
// base + r, so with a row stride = 4 (mod 8) double2 each quarter-warp of the 128-bit
// fragment loads hits 8 distinct bank groups, and the row-per-thread generation (one
// sample per thread) writes consecutive addresses across the warp.
#ifndef NM_CH_CFG
#define NM_CH_CFG 64
#endif
#ifndef NM_MINB_CFG
#define NM_MINB_CFG 2
#endif
constexpr int NM_CH = NM_CH_CFG;  // samples per table chunk
constexpr int NM_S = NM_CH + 4;   // table row stride (double2), = 4 (mod 8)
static_assert(2 * NM_CH == NU_THREADS, "one thread per (sample, half) of the table chunk");

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
                 "{%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NU_THREADS, NM_MINB_CFG)
    nudft_adjoint_dmma_kernel(const AdjParams P) {
    extern __shared__ __align__(16) char sm[];
    double2* At = reinterpret_cast<double2*>(sm);        // [NU_UT][NM_S]: u-major
    double2* Bt = At + NU_UT * NM_S;                     // [NU_VT][NM_S]: v-major
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int fr = lane >> 2, fc = lane & 3;  // fragment row (u / v offset), column (sample)
    const long long u0 = (long long)blockIdx.x * NU_UT;
    const long long v0 = (long long)blockIdx.y * NU_VT;
    const int slice = blockIdx.z;
    const long long i_begin = P.p * slice / P.slices;
    const long long i_end = P.p * (slice + 1) / P.slices;
    double cre[2][4][2], cim[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cre[a][b][0] = cre[a][b][1] = cim[a][b][0] = cim[a][b][1] = 0.0;
    const int h0 = P.n0 / 2, h1 = P.n1 / 2, h2 = P.n2 / 2;

    for (long long c0 = i_begin; c0 < i_end; c0 += NM_CH) {
        const int cnt = (int)min((long long)NM_CH, i_end - c0);
        // operand tables: thread (sample j = tid mod NM_CH, half h = tid / NM_CH) writes
        // half h of sample j's A column (32 u) and of its B column (16 v), the two fp64
        // recurrences interleaved; each half starts from its own sincospi seed
        {
            const int j = tid % NM_CH, h = tid / NM_CH;
            double2* colA = At + j;
            double2* colB = Bt + j;
            constexpr int QA = NU_UT / 2, QB = NU_VT / 2;
            if (j >= cnt) {
                // the MMAs read whole groups of 4 samples: zero columns past the chunk end
                for (int q = 0; q < QA; ++q) colA[(h * QA + q) * NM_S] = make_double2(0.0, 0.0);
                for (int q = 0; q < QB; ++q) colB[(h * QB + q) * NM_S] = make_double2(0.0, 0.0);
            } else {
                const long long i = c0 + j;
                const double k0 = P.pts[i * P.dims];
                const double k1 = P.pts[i * P.dims + 1];
                const double2 wi = make_double2(P.w[2 * i], P.w[2 * i + 1]);
                if (P.dims == 3) {
                    const long long ua = u0 + h * QA;
                    int a = (int)(ua / P.n1), b = (int)(ua - (long long)a * P.n1);
                    double2 e0 = cispi(k0 * (double)(a - h0));
                    double2 e1 = cispi(k1 * (double)(b - h1));
                    const double2 z1 = cispi(k1);
                    const double k2 = P.pts[i * P.dims + 2];
                    double2 e2 = cmul(wi, cispi(k2 * (double)(v0 + h * QB - h2)));
                    const double2 z2 = cispi(k2);
                    for (int q = 0; q < QA; ++q) {
                        colA[(h * QA + q) * NM_S] = cmul(e0, e1);
                        if (q < QB) {
                            colB[(h * QB + q) * NM_S] = e2;
                            e2 = cmul(e2, z2);
                        }
                        if (++b == P.n1) {
                            b = 0;
                            ++a;
                            e0 = cispi(k0 * (double)(a - h0));
                            e1 = cispi(k1 * (double)(b - h1));
                        } else {
                            e1 = cmul(e1, z1);
                        }
                    }
                } else {
                    double2 e0 = cmul(wi, cispi(k0 * (double)(u0 + h * QA - h0)));
                    const double2 z0 = cispi(k0);
                    double2 e1 = cispi(k1 * (double)(v0 + h * QB - h1));
                    const double2 z1 = cispi(k1);
                    for (int q = 0; q < QA; ++q) {
                        colA[(h * QA + q) * NM_S] = e0;
                        e0 = cmul(e0, z0);
                        if (q < QB) {
                            colB[(h * QB + q) * NM_S] = e1;
                            e1 = cmul(e1, z1);
                        }
                    }
                }
            }
        }
        __syncthreads();
        const int ksteps = (cnt + 3) >> 2;
#pragma unroll 2
        for (int ks = 0; ks < ksteps; ++ks) {
            const int j = 4 * ks + fc;
            double2 a[2], b[4];
#pragma unroll
            for (int ub = 0; ub < 2; ++ub) a[ub] = At[((2 * warp + ub) * 8 + fr) * NM_S + j];
#pragma unroll
            for (int vb = 0; vb < 4; ++vb) b[vb] = Bt[(vb * 8 + fr) * NM_S + j];
            // two passes over the 16 accumulators, so that the two MMAs into one
            // accumulator are 16 instructions apart (DMMA latency)
#pragma unroll
            for (int ub = 0; ub < 2; ++ub)
#pragma unroll
                for (int vb = 0; vb < 4; ++vb) {
                    dmma(cre[ub][vb][0], cre[ub][vb][1], a[ub].x, b[vb].x);
                    dmma(cim[ub][vb][0], cim[ub][vb][1], a[ub].x, b[vb].y);
                }
#pragma unroll
            for (int ub = 0; ub < 2; ++ub) {
                const double nai = -a[ub].y;
#pragma unroll
                for (int vb = 0; vb < 4; ++vb) {
                    dmma(cre[ub][vb][0], cre[ub][vb][1], nai, b[vb].y);
                    dmma(cim[ub][vb][0], cim[ub][vb][1], a[ub].y, b[vb].x);
                }
            }
        }
        __syncthreads();
    }
    // accumulator fragment: lane holds C[row fr][cols 2 fc, 2 fc + 1] of each 8 x 8 tile
#pragma unroll
    for (int ub = 0; ub < 2; ++ub) {
        const long long u = u0 + (2 * warp + ub) * 8 + fr;
        if (u >= P.U) continue;
        double* out = P.part + ((size_t)slice * P.U + u) * P.V * 2;
#pragma unroll
        for (int vb = 0; vb < 4; ++vb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long long v = v0 + vb * 8 + 2 * fc + e;
                if (v < P.V) {
                    out[2 * v] = cre[ub][vb][e];
                    out[2 * v + 1] = cim[ub][vb][e];
                }
            }
    }
}

__global__ void __launch_bounds__(NU_THREADS) nudft_forward64_kernel(const FwdParams P) {
    extern __shared__ __align__(16) char sm[];
    double2* rows = reinterpret_cast<double2*>(sm);  // [NF_UT][V]
    const int tid = threadIdx.x;
    const long long i = (long long)blockIdx.x * NU_THREADS + tid;
    const int slice = blockIdx.y;
    const long long ub = P.U * slice / P.slices, ue = P.U * (slice + 1) / P.slices;
    const bool live = i < P.p;
    const long long ii = live ? i : P.p - 1;
    const double k0 = P.pts[ii * P.dims];
    const double k1 = P.pts[ii * P.dims + 1];
    const double kv = P.dims == 3 ? P.pts[ii * P.dims + 2] : k1;
    const int hv = (P.dims == 3 ? P.n2 : P.n1) / 2;
    const double2 z = cispi(-kv);
    const double2 shift = cispi(kv * (double)hv);
    const double2 w = cispi(-(P.dims == 3 ? k1 : k0));
    double fr = 0.0, fi = 0.0;
    for (long long s0 = ub; s0 < ue; s0 += NF_UT) {
        const int nu = (int)min((long long)NF_UT, ue - s0);
        __syncthreads();
        const double2* src = reinterpret_cast<const double2*>(P.img) + (size_t)s0 * P.V;
        for (long long e = tid; e < (long long)nu * P.V; e += NU_THREADS) rows[e] = src[e];
        __syncthreads();
        double2 A = make_double2(0.0, 0.0);
        int a = 0, b = 0;
        for (int q = 0; q < nu; ++q) {
            const long long u = s0 + q;
            bool seed = q == 0;
            if (P.dims == 3) {
                if (q == 0) {
                    a = (int)(u / P.n1);
                    b = (int)(u - (long long)a * P.n1);
                } else if (++b == P.n1) {
                    b = 0;
                    ++a;
                    seed = true;
                }
            }
            if (seed) {
                const double t = P.dims == 3
                                     ? k0 * (double)(a - P.n0 / 2) + k1 * (double)(b - P.n1 / 2)
                                     : k0 * (double)(u - P.n0 / 2);
                A = cispi(-t);
            } else {
                A = cmul(A, w);
            }
            const double2* row = rows + (size_t)q * P.V;
            double pr = 0.0, pi = 0.0;
            for (long long v = P.V - 1; v >= 0; --v) {
                const double2 g = row[v];
                const double nr = fma(pr, z.x, fma(-pi, z.y, g.x));
                pi = fma(pr, z.y, fma(pi, z.x, g.y));
                pr = nr;
            }
            fr = fma(A.x, pr, fma(-A.y, pi, fr));
            fi = fma(A.x, pi, fma(A.y, pr, fi));
        }
    }
    if (live) {
        const double2 f = cmul(make_double2(fr, fi), shift);
        double* out = P.part + ((size_t)slice * P.p + i) * 2;
        out[0] = f.x;
        out[1] = f.y;
    }
}

// density_compensation update (analysis.py:90-96): w_i <- w_i / max(|back_i|, 1e-12)
__global__ void dcf_update_kernel(double* __restrict__ w, const double* __restrict__ back,
                                  long long p) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= p) return;
    const double m = fmax(hypot(back[2 * i], back[2 * i + 1]), 1e-12);
    w[2 * i] = w[2 * i] / m;
    w[2 * i + 1] = w[2 * i + 1] / m;
}

// compute_psf magnitudes (analysis.py:126-131): |vol / sum(w)|
__global__ void psf_magnitude_kernel(const double* __restrict__ vol, long long n, double total,
                                     double* __restrict__ mag) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= n) return;
    mag[e] = hypot(vol[2 * e] / total, vol[2 * e + 1] / total);
}

}  // namespace spk

using namespace spk;

extern "C" {

size_t spk_nudft_workspace_bytes(int64_t p, int dims, const int64_t* grid) {
    const long long U = dims == 3 ? grid[0] * grid[1] : grid[0];
    const long long V = dims == 3 ? grid[2] : grid[1];
    // adjoint: up to 16 slices of U x V complex; forward: up to 16 slices of p complex
    const size_t adj = (size_t)16 * U * V * 16;
    const size_t fwd = (size_t)16 * p * 16;
    return adj > fwd ? adj : fwd;
}

// Sample slices (split-K) of the adjoint: at least ~2 waves of resident CTAs, and among
// the candidates the one whose last wave is fullest (tiles x slices vs the resident slots).
static int adj_slices(long long U, long long V, long long p, int chunk, int slots) {
    const long long tiles = ((U + NU_UT - 1) / NU_UT) * ((V + NU_VT - 1) / NU_VT);
    const long long smax = std::max(1LL, std::min(16LL, (p + chunk - 1) / chunk));
    const long long smin = std::min(smax, std::max(1LL, (2LL * slots + tiles - 1) / tiles));
    long long best = smin;
    double best_eff = -1.0;
    for (long long s = smin; s <= smax; ++s) {
        const double waves = (double)(tiles * s) / slots;
        const double eff = waves / std::ceil(waves) - 0.002 * (double)s;
        if (eff > best_eff + 1e-12) {
            best_eff = eff;
            best = s;
        }
    }
    return (int)best;
}

int spk_nudft_adjoint(const double* pts, const double* weights, int64_t p, int dims,
                      const int64_t* grid, int mode, double* out, void* ws, size_t ws_bytes,
                      spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(mode == SPK_NUDFT_FP64 || mode == SPK_NUDFT_MIXED, SPK_ERR_ARG,
                "nudft: unknown mode %d", mode);
    SPK_REQUIRE(p >= 1, SPK_ERR_ARG, "nudft: empty sample set");
    AdjParams P{};
    P.pts = pts;
    P.w = weights;
    P.p = p;
    P.dims = dims;
    P.n0 = (int)grid[0];
    P.n1 = (int)grid[1];
    P.n2 = dims == 3 ? (int)grid[2] : 1;
    P.U = dims == 3 ? (long long)P.n0 * P.n1 : P.n0;
    P.V = dims == 3 ? P.n2 : P.n1;
    const bool f64 = mode == SPK_NUDFT_FP64;
    static int dmma_on = -1;
    if (dmma_on < 0) {
        const char* e = getenv("SPK_NUDFT_DMMA");
        dmma_on = (e && e[0] == '0') ? 0 : 1;
    }
    const bool tc = f64 && dmma_on;
    const void* kern = tc ? (const void*)nudft_adjoint_dmma_kernel
                          : f64 ? (const void*)nudft_adjoint64_kernel
                                : (const void*)nudft_adjoint_kernel;
    const size_t smem =
        tc    ? (size_t)(NU_UT + NU_VT) * NM_S * sizeof(double2)
        : f64 ? (size_t)ND_CH * (ND_AS + ND_BS) * sizeof(double2)
              : ((size_t)((NU_CH * NU_AS + 1) & ~1) + (size_t)NU_CH * NU_BS) * sizeof(C2);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NU_THREADS, smem);
    P.slices = adj_slices(P.U, P.V, p, tc ? NM_CH : f64 ? ND_CH : NU_CH,
                          std::max(1, per_sm) * num_sms());
    SPK_REQUIRE(ws_bytes >= (size_t)P.slices * P.U * P.V * 16, SPK_ERR_WORKSPACE,
                "nudft adjoint: workspace too small");
    P.part = static_cast<double*>(ws);
    dim3 grid3((unsigned)((P.U + NU_UT - 1) / NU_UT), (unsigned)((P.V + NU_VT - 1) / NU_VT),
               (unsigned)P.slices);
    cudaStream_t s = (cudaStream_t)stream;
    if (tc)
        nudft_adjoint_dmma_kernel<<<grid3, NU_THREADS, smem, s>>>(P);
    else if (f64)
        nudft_adjoint64_kernel<<<grid3, NU_THREADS, smem, s>>>(P);
    else
        nudft_adjoint_kernel<<<grid3, NU_THREADS, smem, s>>>(P);
    SPK_CHECK_LAUNCH("spk_nudft_adjoint");
    const long long n = P.U * P.V * 2;
    nudft_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P.part, P.slices, n, out);
    SPK_CHECK_LAUNCH("spk_nudft_adjoint(reduce)");
    return SPK_OK;
}

int spk_nudft_forward(const double* pts, const double* image, int64_t p, int dims,
                      const int64_t* grid, int mode, double* out, void* ws, size_t ws_bytes,
                      spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(mode == SPK_NUDFT_FP64 || mode == SPK_NUDFT_MIXED, SPK_ERR_ARG,
                "nudft: unknown mode %d", mode);
    SPK_REQUIRE(p >= 1, SPK_ERR_ARG, "nudft: empty sample set");
    FwdParams P{};
    P.pts = pts;
    P.img = image;
    P.p = p;
    P.dims = dims;
    P.n0 = (int)grid[0];
    P.n1 = (int)grid[1];
    P.n2 = dims == 3 ? (int)grid[2] : 1;
    P.U = dims == 3 ? (long long)P.n0 * P.n1 : P.n0;
    P.V = dims == 3 ? P.n2 : P.n1;
    SPK_REQUIRE(P.V <= NF_VMAX, SPK_ERR_ARG, "nudft forward: last grid axis %lld > %d",
                P.V, NF_VMAX);
    const long long blocks = (p + NU_THREADS - 1) / NU_THREADS;
    const long long want = 4LL * num_sms();
    long long sl = std::max(1LL, std::min(16LL, (want + blocks - 1) / blocks));
    sl = std::min(sl, P.U);
    P.slices = (int)sl;
    SPK_REQUIRE(ws_bytes >= (size_t)P.slices * p * 16, SPK_ERR_WORKSPACE,
                "nudft forward: workspace too small");
    P.part = static_cast<double*>(ws);
    dim3 grid2((unsigned)blocks, (unsigned)P.slices);
    cudaStream_t s = (cudaStream_t)stream;
    if (mode == SPK_NUDFT_FP64) {
        const size_t smem = (size_t)NF_UT * P.V * sizeof(double2);
        cudaFuncSetAttribute(nudft_forward64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)std::max(smem, (size_t)1));
        nudft_forward64_kernel<<<grid2, NU_THREADS, smem, s>>>(P);
    } else {
        const size_t smem = (size_t)NF_UT * P.V * sizeof(float2);
        cudaFuncSetAttribute(nudft_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)std::max(smem, (size_t)1));
        nudft_forward_kernel<<<grid2, NU_THREADS, smem, s>>>(P);
    }
    SPK_CHECK_LAUNCH("spk_nudft_forward");
    const long long n = p * 2;
    nudft_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P.part, P.slices, n, out);
    SPK_CHECK_LAUNCH("spk_nudft_forward(reduce)");
    return SPK_OK;
}

int spk_dcf_update(double* weights, const double* back, int64_t p, spk_stream_t stream) {
    if (p == 0) return SPK_OK;
    dcf_update_kernel<<<(unsigned)((p + 255) / 256), 256, 0, (cudaStream_t)stream>>>(weights,
                                                                                   back, p);
    SPK_CHECK_LAUNCH("spk_dcf_update");
    return SPK_OK;
}

int spk_psf_magnitude(const double* vol, int64_t n, double total, double* mag,
                      spk_stream_t stream) {
    if (n == 0) return SPK_OK;
    psf_magnitude_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        vol, n, total, mag);
    SPK_CHECK_LAUNCH("spk_psf_magnitude");
    return SPK_OK;
}

}  // extern "C"
