// project.cu -- K3 batched shot projection (fp64) and the per-shot helpers around it.
//
// Compiled with -fmad=false: every fp64 expression is evaluated with the reference's
// operation order and no FMA contraction, so results are bit-identical to the numba
// kernels of /root/reference/pkg/src/vdtraj/projection.py (IEEE div/sqrt on both sides).
//
//  * fista_kernel: one CTA per shot, one thread per sample (strided), n_pit iterations
//    of dual FISTA with gradient restart (_project_shot, projection.py:169-284).  s and
//    the first/second-difference duals live in shared memory (neighbour access); the
//    remaining per-sample state lives in an L2-resident workspace.  The restart test
//    sign(<y - z, z - q>) uses a block tree reduction plus a rounding-error bound; if the
//    bound cannot certify the sign, thread 0 re-sums the terms in the reference's
//    sequential order, so restart decisions are identical to the reference.
//  * polish_kernel: the relaxed cyclic projections (_feasibility_polish, :287-373),
//    a Gauss-Seidel recurrence.  One warp per shot, wavefront-pipelined: lane k runs
//    sweep (base + k) four samples behind lane k-1, so 32 sweeps advance together with
//    exactly the reference's per-element operation sequence; a checkpoint + replay
//    reproduces the reference's stopping sweep.
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "spk_common.cuh"

namespace spk {

constexpr int PJ_THREADS = 512;  // FISTA CTA size: 16 warps hide the state loads
constexpr int PJ_SMEM_LIMIT = 200 * 1024;

struct ProjArgs {
    const double* in;
    const double* grad;
    double eta;
    const double* eta_shot;  // per-shot step (batched problems); overrides eta when set
    double* out;
    long long n_shots;
    int ns;
    double a, b;
    int pin;
    double pv[3];
    int n_pit;
    double tau;
    int monotone;
    double* trace;
    int32_t* nonfinite;
    double* ws;         // per-shot state, stride = ws_stride doubles
    long long ws_stride;
    int smem_arrays;    // 1: s/y1/y2 in shared memory, 2: s/y1/y2/y0
};

// Workspace layout per shot (units of ns*D doubles): k, q0, q1, q2, y0, z0, z1, z2, s_obj,
// [s, y1, y2 when they do not fit in shared memory].
constexpr int PJ_WS_ARRAYS = 12;

__device__ __forceinline__ double clamp_unit(double z) {
    const double m = (z > -1.0) ? z : -1.0;  // max(z, -1.0)
    return (m < 1.0) ? m : 1.0;              // min(., 1.0)
}

// s = k - (A0^T q0 + A1^T q1 + A2^T q2) for one row n (_dual_to_primal,
// projection.py:103-123); the pinned row is handled by the caller.
template <int D>
__device__ __forceinline__ void primal_row(const double* k, const double* q0, const double* q1,
                                           const double* q2, int ns, int n, double* s) {
#pragma unroll
    for (int l = 0; l < D; ++l) {
        double r = q0[n * D + l];
        if (n <= ns - 2) r -= q1[n * D + l];
        if (n >= 1) r += q1[(n - 1) * D + l];
        if (n <= ns - 3) r += q2[n * D + l];
        if (1 <= n && n <= ns - 2) r -= 2.0 * q2[(n - 1) * D + l];
        if (n >= 2) r += q2[(n - 2) * D + l];
        s[n * D + l] = k[n * D + l] - r;
    }
}

// Dual objective of (q0, q1, q2) in the reference's sequential order (_dual_objective,
// projection.py:126-166).  Requires s = primal(q) already written for all rows; run by
// a single thread.
template <int D>
__device__ double dual_objective_serial(const double* s, const double* q0, const double* q1,
                                        const double* q2, int ns, int pin, const double* pv,
                                        double a, double b) {
    double obj = 0.0;
    for (int n = 0; n < ns; ++n) {
        if (n == pin) continue;
        for (int l = 0; l < D; ++l) obj += 0.5 * s[n * D + l] * s[n * D + l];
    }
    for (int i = 0; i < ns * D; ++i) obj += fabs(q0[i]);
    for (int n = 0; n < ns - 1; ++n) {
        double nrm = 0.0;
        for (int l = 0; l < D; ++l) nrm += q1[n * D + l] * q1[n * D + l];
        obj += a * sqrt(nrm);
    }
    for (int n = 0; n < ns - 2; ++n) {
        double nrm = 0.0;
        for (int l = 0; l < D; ++l) nrm += q2[n * D + l] * q2[n * D + l];
        obj += b * sqrt(nrm);
    }
    if (pin >= 0) {
        const int p = pin;
        for (int l = 0; l < D; ++l) {
            obj -= q0[p * D + l] * pv[l];
            if (p <= ns - 2) obj -= q1[p * D + l] * pv[l];
            if (p >= 1) obj += q1[(p - 1) * D + l] * pv[l];
            if (p <= ns - 3) obj += q2[p * D + l] * pv[l];
            if (1 <= p && p <= ns - 2) obj -= 2.0 * q2[(p - 1) * D + l] * pv[l];
            if (p >= 2) obj += q2[(p - 2) * D + l] * pv[l];
        }
    }
    return obj;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide (sum, sum of |.|) with a fixed reduction tree; result broadcast.
__device__ __forceinline__ void block_sum2(double& x, double& y, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) {
        red[w] = x;
        red[32 + w] = y;
    }
    __syncthreads();
    if (w == 0) {
        double a = lane < nw ? red[lane] : 0.0;
        double b = lane < nw ? red[32 + lane] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
            red[64] = a;
            red[65] = b;
        }
    }
    __syncthreads();
    x = red[64];
    y = red[65];
}

// Dual prox of sample n (projection.py:186-213): z0 = tau (y0/tau + s - clamp(...)),
// z1 / z2 = tau * ball-projection residuals of the first / second differences.  Used by
// the prox pass, recomputed bit-identically by the update pass and the serial restart
// fallback instead of storing z (three state arrays of HBM traffic per iteration).
template <int D>
__device__ __forceinline__ void prox_sample(int n, int ns, const double* __restrict__ s,
                                            const double* __restrict__ y0,
                                            const double* __restrict__ y1,
                                            const double* __restrict__ y2, double a, double b,
                                            double tau, double inv_tau, double (&z0)[D],
                                            double (&z1)[D], double (&z2)[D]) {
#pragma unroll
    for (int l = 0; l < D; ++l) {
        const int e = n * D + l;
        const double z = y0[e] * inv_tau + s[e];
        const double pz = clamp_unit(z);
        z0[l] = tau * (z - pz);
    }
    if (n <= ns - 2) {
        double zv[D];
        double nrm = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
            const int e = n * D + l;
            const double z = y1[e] * inv_tau + (s[e + D] - s[e]);
            zv[l] = z;
            nrm += z * z;
        }
        nrm = sqrt(nrm);
        const double scale = (nrm <= a) ? 0.0 : 1.0 - a / nrm;
#pragma unroll
        for (int l = 0; l < D; ++l) z1[l] = tau * zv[l] * scale;
    }
    if (n <= ns - 3) {
        double zv[D];
        double nrm = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
            const int e = n * D + l;
            const double z = y2[e] * inv_tau + (s[e + 2 * D] - 2.0 * s[e + D] + s[e]);
            zv[l] = z;
            nrm += z * z;
        }
        nrm = sqrt(nrm);
        const double scale = (nrm <= b) ? 0.0 : 1.0 - b / nrm;
#pragma unroll
        for (int l = 0; l < D; ++l) z2[l] = tau * zv[l] * scale;
    }
}

template <int D>
__global__ void __launch_bounds__(PJ_THREADS) fista_kernel(const ProjArgs A) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double red[72];
    __shared__ int flag_sh[2];
    const int ns = A.ns;
    const int nd = ns * D;
    const long long c = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;

    double* W = A.ws + c * A.ws_stride;
    double* k = W;
    double* q0 = W + 1 * (size_t)nd;
    double* q1 = W + 2 * (size_t)nd;
    double* q2 = W + 3 * (size_t)nd;
    double* y0 = W + 4 * (size_t)nd;  // (shared memory when smem_arrays == 2)
    double* z0 = W + 5 * (size_t)nd;
    double* z1 = W + 6 * (size_t)nd;
    double* z2 = W + 7 * (size_t)nd;
    double* so = W + 8 * (size_t)nd;  // scratch primal for objectives
    double *s, *y1, *y2;
    if (A.smem_arrays) {
        s = smem;
        y1 = smem + nd;
        y2 = smem + 2 * nd;
        if (A.smem_arrays == 2) y0 = smem + 3 * nd;
    } else {
        s = W + 9 * (size_t)nd;
        y1 = W + 10 * (size_t)nd;
        y2 = W + 11 * (size_t)nd;
    }
    const double* pv = A.pv;
    const double a = A.a, b = A.b, tau = A.tau;
    const double inv_tau = 1.0 / tau;
    const double* in = A.in + c * (size_t)nd;
    const double* gr = A.grad ? A.grad + c * (size_t)nd : nullptr;

    if (tid == 0) flag_sh[0] = 0;
    __syncthreads();
    int bad = 0;
    const double eta = A.eta_shot ? A.eta_shot[c] : A.eta;
    for (int i = tid; i < nd; i += nt) {
        double kv = in[i];
        if (gr) kv = kv - eta * gr[i];  // pattern.coords - eta * grad (optimizer.py:326)
        if (!isfinite(kv)) bad = 1;
        k[i] = kv;
        q0[i] = 0.0;
        q1[i] = 0.0;
        q2[i] = 0.0;
        y0[i] = 0.0;
        y1[i] = 0.0;
        y2[i] = 0.0;
    }
    if (bad) flag_sh[0] = 1;
    __syncthreads();
    if (tid == 0 && flag_sh[0] && A.nonfinite) atomicExch(A.nonfinite, 1);

    const int n1 = (ns - 1) * D, n2 = (ns - 2) * D;
    const int nterms = nd + (n1 > 0 ? n1 : 0) + (n2 > 0 ? n2 : 0);
    const double ebound = 2.02 * (double)nterms * 1.1102230246251565e-16;
    double t = 1.0, best = INFINITY;

    for (int it = 0; it < A.n_pit; ++it) {
        // ---- s = primal(y)
        for (int n = tid; n < ns; n += nt) {
            primal_row<D>(k, y0, y1, y2, ns, n, s);
            if (n == A.pin)
                for (int l = 0; l < D; ++l) s[n * D + l] = pv[l];
        }
        __syncthreads();
        // ---- dual prox -> z, restart terms (z stored only when the monotone objective
        // needs it; otherwise it is recomputed by the update pass)
        double gd = 0.0, ga = 0.0;
        const bool keep_z = A.monotone;
        for (int n = tid; n < ns; n += nt) {
            double zz0[D], zz1[D], zz2[D];
            prox_sample<D>(n, ns, s, y0, y1, y2, a, b, tau, inv_tau, zz0, zz1, zz2);
#pragma unroll
            for (int l = 0; l < D; ++l) {
                const int e = n * D + l;
                if (keep_z) z0[e] = zz0[l];
                const double term = (y0[e] - zz0[l]) * (zz0[l] - q0[e]);
                gd += term;
                ga += fabs(term);
            }
            if (n <= ns - 2) {
#pragma unroll
                for (int l = 0; l < D; ++l) {
                    const int e = n * D + l;
                    if (keep_z) z1[e] = zz1[l];
                    const double term = (y1[e] - zz1[l]) * (zz1[l] - q1[e]);
                    gd += term;
                    ga += fabs(term);
                }
            }
            if (n <= ns - 3) {
#pragma unroll
                for (int l = 0; l < D; ++l) {
                    const int e = n * D + l;
                    if (keep_z) z2[e] = zz2[l];
                    const double term = (y2[e] - zz2[l]) * (zz2[l] - q2[e]);
                    gd += term;
                    ga += fabs(term);
                }
            }
        }
        block_sum2(gd, ga, red);  // contains __syncthreads: z*, y* visible block-wide
        int restart;
        if (fabs(gd) > ebound * ga) {
            restart = gd > 0.0;
        } else {
            // Sign not certified: reproduce the reference's sequential sum exactly.
            if (tid == 0) {
                double g = 0.0;
                if (keep_z) {
                    for (int i = 0; i < nd; ++i) g += (y0[i] - z0[i]) * (z0[i] - q0[i]);
                    for (int i = 0; i < n1; ++i) g += (y1[i] - z1[i]) * (z1[i] - q1[i]);
                    for (int i = 0; i < n2; ++i) g += (y2[i] - z2[i]) * (z2[i] - q2[i]);
                } else {  // same terms, same order, z recomputed
                    double zz0[D], zz1[D], zz2[D];
                    for (int pass = 0; pass < 3; ++pass)
                        for (int n = 0; n < ns - pass; ++n) {
                            prox_sample<D>(n, ns, s, y0, y1, y2, a, b, tau, inv_tau, zz0, zz1,
                                           zz2);
                            for (int l = 0; l < D; ++l) {
                                const int e = n * D + l;
                                if (pass == 0) g += (y0[e] - zz0[l]) * (zz0[l] - q0[e]);
                                else if (pass == 1) g += (y1[e] - zz1[l]) * (zz1[l] - q1[e]);
                                else g += (y2[e] - zz2[l]) * (zz2[l] - q2[e]);
                            }
                        }
                }
                flag_sh[1] = g > 0.0;
            }
            __syncthreads();
            restart = flag_sh[1];
        }
        int accept = 1;
        if (A.monotone) {
            // objective of the candidate z (projection.py:221-227)
            for (int n = tid; n < ns; n += nt) {
                primal_row<D>(k, z0, z1, z2, ns, n, so);
                if (n == A.pin)
                    for (int l = 0; l < D; ++l) so[n * D + l] = pv[l];
            }
            __syncthreads();
            if (tid == 0) {
                const double obj = dual_objective_serial<D>(so, z0, z1, z2, ns, A.pin, pv, a, b);
                int acc = 1;
                if (obj > best) acc = 0;
                else best = obj;
                flag_sh[0] = acc;
                red[70] = best;
            }
            __syncthreads();
            accept = flag_sh[0];
            best = red[70];
        }
        if (restart) t = 1.0;
        const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
        if (A.monotone) {
            const double mom_z = t / t_next;
            const double mom_q = (t - 1.0) / t_next;
            for (int n = tid; n < ns; n += nt) {
#pragma unroll
                for (int l = 0; l < D; ++l) {
                    const int e = n * D + l;
                    double nq = accept ? z0[e] : q0[e];
                    y0[e] = nq + mom_z * (z0[e] - nq) + mom_q * (nq - q0[e]);
                    q0[e] = nq;
                    if (n <= ns - 2) {
                        nq = accept ? z1[e] : q1[e];
                        y1[e] = nq + mom_z * (z1[e] - nq) + mom_q * (nq - q1[e]);
                        q1[e] = nq;
                    }
                    if (n <= ns - 3) {
                        nq = accept ? z2[e] : q2[e];
                        y2[e] = nq + mom_z * (z2[e] - nq) + mom_q * (nq - q2[e]);
                        q2[e] = nq;
                    }
                }
            }
        } else {
            const double mom = (t - 1.0) / t_next;
            for (int n = tid; n < ns; n += nt) {
                double zz0[D], zz1[D], zz2[D];
                prox_sample<D>(n, ns, s, y0, y1, y2, a, b, tau, inv_tau, zz0, zz1, zz2);
#pragma unroll
                for (int l = 0; l < D; ++l) {
                    const int e = n * D + l;
                    y0[e] = zz0[l] + mom * (zz0[l] - q0[e]);
                    q0[e] = zz0[l];
                    if (n <= ns - 2) {
                        y1[e] = zz1[l] + mom * (zz1[l] - q1[e]);
                        q1[e] = zz1[l];
                    }
                    if (n <= ns - 3) {
                        y2[e] = zz2[l] + mom * (zz2[l] - q2[e]);
                        q2[e] = zz2[l];
                    }
                }
            }
        }
        t = t_next;
        __syncthreads();
        if (A.trace) {
            for (int n = tid; n < ns; n += nt) {
                primal_row<D>(k, q0, q1, q2, ns, n, so);
                if (n == A.pin)
                    for (int l = 0; l < D; ++l) so[n * D + l] = pv[l];
            }
            __syncthreads();
            if (tid == 0)
                A.trace[c * A.n_pit + it] =
                    dual_objective_serial<D>(so, q0, q1, q2, ns, A.pin, pv, a, b);
            __syncthreads();
        }
    }
    // ---- out = primal(q)
    double* out = A.out + c * (size_t)nd;
    for (int n = tid; n < ns; n += nt) {
        primal_row<D>(k, q0, q1, q2, ns, n, out);
        if (n == A.pin)
            for (int l = 0; l < D; ++l) out[n * D + l] = pv[l];
    }
}

// ------------------------------------------------------------------- feasibility polish
// The polish (_feasibility_polish, projection.py:287-373) is a Gauss-Seidel recurrence:
// every sweep is box(all) -> speed pairs n = 0..ns-2 -> accel triples n = 0..ns-3, and
// sweeps repeat until the worst violation of a sweep is <= tol.  It is run as a
// SYSTOLIC WAVEFRONT: lane g of the CTA executes sweep (base + g).  At its local step t a
// lane applies
//     S(t)     speed pair (t, t+1)
//     A(t-2)   accel triple (t-2, t-1, t)       -> sample t-2 is now final for this sweep
//     B(t+2)   box of sample t+2 (pin set first) on the value handed over by lane g-1
// which touches each sample in exactly the reference's per-sample operation order.  The
// samples a lane is working on live in registers (a 4-sample window); finished samples
// are handed to the next sweep with a warp shuffle (shared memory across warp
// boundaries, one extra step of lag).  Lane g runs 4 steps behind lane g-1, the minimum
// for which the windows of consecutive sweeps never overlap out of order.  A batch of
// B = 32 W sweeps reads the state from one shared buffer and the last sweep writes the
// other, so the batch input doubles as the checkpoint: if sweep j < B-1 is the stopping
// sweep, the batch is replayed with j + 1 lanes.  Every element sees the same IEEE fp64
// operations in the same order as the reference => bit-identical results and sweep count.
constexpr int PL_LAG = 4;
#ifndef SPK_BOX_FAST
#define SPK_BOX_FAST 1
#endif

template <int D>
struct Sample {
    double v[D];
};

template <int D>
__device__ __forceinline__ void box_sample(Sample<D>& s, double& worst) {
#if SPK_BOX_FAST
    // almost every sample is inside the box: one compare per axis (|v| > 1 is false for
    // |v| <= 1 and for NaN, exactly the reference's no-op cases) and a warp-uniform skip
    bool out = fabs(s.v[0]) > 1.0 || fabs(s.v[1]) > 1.0;
    if (D == 3) out = out || fabs(s.v[D - 1]) > 1.0;
    if (!out) return;
#endif
    // the excess |v| - 1 equals the reference's v - 1 / -1 - v bit for bit, and fmax
    // leaves worst (>= 0) unchanged when |v| <= 1 or v is NaN; only |v| > 1 replaces v,
    // by +-1 with v's sign (NaN and +-0 pass through)
#pragma unroll
    for (int l = 0; l < D; ++l) {
        const double v = s.v[l];
        const double av = fabs(v);
        worst = fmax(worst, av - 1.0);
        s.v[l] = av > 1.0 ? copysign(1.0, v) : v;
    }
}

// Speed pair (n, n+1) on registers x0 = s[n], x1 = s[n+1] (projection.py:313-345).
template <int D>
__device__ __forceinline__ void speed_pair(Sample<D>& x0, Sample<D>& x1, int n, double a,
                                           int pin, double& worst) {
    const double omega = 1.8;
    double df[D];  // x1 - x0, reused by the update (the samples do not change in between)
    double nrm = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
        df[l] = x1.v[l] - x0.v[l];
        nrm += df[l] * df[l];
    }
    // exact early out: a*a*(1 - 1e-15) < a^2 in real arithmetic, so nrm^2 below it means
    // sqrt(nrm^2) < a, i.e. the reference's `nrm > a` is false -- skips the IEEE sqrt
    // for the (typically many) pairs well inside the bound; NaN takes the full path
    if (nrm <= a * a * (1.0 - 1e-15)) return;
    nrm = sqrt(nrm);
    if (!(nrm > a)) return;
    if (nrm - a > worst) worst = nrm - a;
    if (n == pin || n + 1 == pin) {
        // move only the free endpoint of a pinned pair
        const double shrink = omega * (nrm - a) / nrm;
        if (n == pin) {
#pragma unroll
            for (int l = 0; l < D; ++l) x1.v[l] -= 1.0 * shrink * df[l];
        } else {
#pragma unroll
            for (int l = 0; l < D; ++l) x0.v[l] -= -1.0 * shrink * df[l];
        }
        return;
    }
    const double shrink = omega * 0.5 * (nrm - a) / nrm;
#pragma unroll
    for (int l = 0; l < D; ++l) {
        x0.v[l] += shrink * df[l];
        x1.v[l] -= shrink * df[l];
    }
}

// Accel triple (n, n+1, n+2) (projection.py:346-371).
template <int D>
__device__ __forceinline__ void accel_triple(Sample<D>& x0, Sample<D>& x1, Sample<D>& x2, int n,
                                             double b, int pin, double& worst) {
    const double omega = 1.8;
    double w[D];  // second differences, reused by the update
    double nrm = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
        w[l] = x0.v[l] - 2.0 * x1.v[l] + x2.v[l];
        nrm += w[l] * w[l];
    }
    if (nrm <= b * b * (1.0 - 1e-15)) return;  // exact early out, as in speed_pair
    nrm = sqrt(nrm);
    if (!(nrm > b)) return;
    if (nrm - b > worst) worst = nrm - b;
    if (pin != n && pin != n + 1 && pin != n + 2) {
        // unpinned triple: c = (1, -2, 1), denom = 6 exactly; step * 1 and step * -2 are
        // exact, so this is the general branch below with the constants folded
        const double step = omega * (nrm - b) / (6.0 * nrm);
        const double step1 = step * -2.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
            x0.v[l] -= step * w[l];
            x1.v[l] -= step1 * w[l];
            x2.v[l] -= step * w[l];
        }
        return;
    }
    double c0 = 1.0, c1 = -2.0, c2 = 1.0;
    if (pin == n) c0 = 0.0;
    else if (pin == n + 1) c1 = 0.0;
    else if (pin == n + 2) c2 = 0.0;
    const double denom = c0 * c0 + c1 * c1 + c2 * c2;
    if (denom > 0.0) {
        const double step = omega * (nrm - b) / (denom * nrm);
#pragma unroll
        for (int l = 0; l < D; ++l) {
            x0.v[l] -= step * c0 * w[l];
            x1.v[l] -= step * c1 * w[l];
            x2.v[l] -= step * c2 * w[l];
        }
    }
}

__device__ __forceinline__ int lane_offset(int g) { return PL_LAG * g + (g >> 5); }

// One batch of `nsw` (1..blockDim) sweeps from s_in to s_out; returns this lane's worst.
template <int D>
__device__ double systolic_batch(const double* __restrict__ s_in, double* __restrict__ s_out,
                                 double* xfer, int ns, double a, double b, int pin,
                                 const double* pv, int nsw) {
    const int g = threadIdx.x;
    const int lane = g & 31;
    const int warp = g >> 5;
    const bool active = g < nsw;
    const bool last = g == nsw - 1;
    const int off = lane_offset(g);
    const int n_steps = ns + 4 + lane_offset(nsw - 1);
    double worst = 0.0;
    Sample<D> w0, w1, w2, w3;
#pragma unroll
    for (int l = 0; l < D; ++l) w0.v[l] = w1.v[l] = w2.v[l] = w3.v[l] = 0.0;
    for (int st = 0; st < n_steps; ++st) {
        const int t = st - 2 - off;
        const bool on = active && t >= -2 && t <= ns + 1;
        Sample<D> emit;
#pragma unroll
        for (int l = 0; l < D; ++l) emit.v[l] = 0.0;
        if (on) {
            if (t >= 0 && t <= ns - 2) speed_pair<D>(w2, w3, t, a, pin, worst);
            if (t >= 2 && t <= ns - 1) accel_triple<D>(w0, w1, w2, t - 2, b, pin, worst);
            emit = w0;  // sample t-2, final for this sweep when t >= 2
            if (last && t >= 2) {
#pragma unroll
                for (int l = 0; l < D; ++l) s_out[(t - 2) * D + l] = emit.v[l];
            }
        }
        // hand finished samples to the next sweep
        Sample<D> recv;
#pragma unroll
        for (int l = 0; l < D; ++l) recv.v[l] = __shfl_up_sync(0xffffffffu, emit.v[l], 1);
        if (lane == 31) {
            double* x = xfer + ((warp * 2 + (st & 1)) * D);
#pragma unroll
            for (int l = 0; l < D; ++l) x[l] = emit.v[l];
        }
        if (on) {
            const int m = t + 2;
            if (m <= ns - 1) {
                if (g == 0) {
#pragma unroll
                    for (int l = 0; l < D; ++l) recv.v[l] = s_in[m * D + l];
                } else if (lane == 0) {
                    const double* x = xfer + (((warp - 1) * 2 + ((st - 1) & 1)) * D);
#pragma unroll
                    for (int l = 0; l < D; ++l) recv.v[l] = x[l];
                }
                if (m == pin) {
#pragma unroll
                    for (int l = 0; l < D; ++l) recv.v[l] = pv[l];
                }
                box_sample<D>(recv, worst);
            }
            w0 = w1;
            w1 = w2;
            w2 = w3;
            w3 = recv;
        }
        if (blockDim.x > 32) __syncthreads();
        else __syncwarp();
    }
    return worst;
}

// Continuous ring: lane g runs sweeps g, g+B, g+2B, ...; sweep k starts at global step
// (k / B) * P + lane_offset(k % B) with period P = 4 B + W >= ns + 4, so consecutive
// sweeps stay exactly 4 steps apart (5 across a warp or the wrap-around boundary) and
// no lane idles between rounds (for B ~ ns / 4).  The last lane writes every round's
// output stream into a ping-pong snapshot; when sweep k* is the first whose worst
// violation is <= tol, the ring stops and sweeps j B .. k* are replayed (systolic_batch)
// from the snapshot after sweep j B - 1 (j = k* / B), which the ring has not
// overwritten yet because P >= ns + 4.  Bit-identical to the sequential polish.
// State of one ring lane between steps.
template <int D>
struct RingLane {
    Sample<D> slot[4];  // register window, roles rotate with the global step (mod 4)
    double worst;
    int t, j, k;        // local step in the current round, round, sweep index
#ifdef SPK_POLISH_PROF
    unsigned long long prof[7];
    unsigned long long tp;
#endif
};

#ifdef SPK_POLISH_PROF
// Per-phase cycle sums of one observed lane (block 0, thread 40): speed, accel,
// hand-over, box, barrier, steps.  Diagnostic build only (scripts/polish_profile.sh).
__device__ unsigned long long spk_polish_prof[3][7];
#define SPK_PROF_MARK(L, i)                                                              \
    {                                                                                    \
        const unsigned long long now__ = clock64();                                      \
        (L).prof[i] += now__ - (L).tp;                                                   \
        (L).tp = now__;                                                                  \
    }
#else
#define SPK_PROF_MARK(L, i)
#endif

// Ring lanes lag by 4 steps, the minimum for which the windows of consecutive sweeps
// never overlap out of order.  (A variant running S(t) and A(t-3) concurrently at lag 5
// was measured slower: the per-step latency is dominated by control flow, not by the
// S -> A fp64 chain.)  Across a warp boundary the lag is 4 + RING_K: the sample lane 31 of
// warp w-1 emits at step s is consumed by lane 0 of warp w at step s + RING_K, through a
// 2 RING_K-deep shared-memory slot ring, so the CTA only needs a barrier every RING_K
// steps (a producer write and its consumer read always straddle one) instead of every
// step.  The period grows from 4 B + W to 4 B + RING_K W.
#ifndef SPK_RING_K
#define SPK_RING_K 4
#endif
constexpr int RING_K = SPK_RING_K;
static_assert(RING_K >= 1 && (RING_K & (RING_K - 1)) == 0, "RING_K must be a power of two");
__device__ __forceinline__ int ring_offset(int g) { return PL_LAG * g + RING_K * (g >> 5); }

// One global step of the ring.  R = st mod 4 fixes which window slot plays w0..w3
// (w0 = s[t-2] = slot[R], ..., w3 = s[t+1] = slot[R+3]); the received sample s[t+2]
// overwrites slot[R] (the old w0, handed on this step), so the window never moves
// between registers.  Per sample the operation order is the reference's:
// B(m) @ m-2, S(m-1) @ m-1, S(m) @ m, A(m-2) @ m, A(m-1) @ m+1, A(m) @ m+2.
template <int D, int R>
__device__ __forceinline__ void ring_step(RingLane<D>& L, int st, int ns, int B, int P, int g,
                                          int lane, int warp, int max_sweeps, int kl,
                                          double a, double b, int pin, double pv0,
                                          double pv1, double pv2, double tol,
                                          const double* __restrict__ s0, double* snap0,
                                          double* res, double* xfer, double* wrap0,
                                          int wstride, int* stop_sh) {  // stop_sh[2]
    Sample<D>& w0 = L.slot[R & 3];
    Sample<D>& w1 = L.slot[(R + 1) & 3];
    Sample<D>& w2 = L.slot[(R + 2) & 3];
    Sample<D>& w3 = L.slot[(R + 3) & 3];
    const int t = L.t;
    const bool on = t >= -2 && t <= ns + 1 && L.k < max_sweeps;
    if (on) {
        if (t == -2) L.worst = 0.0;
#ifdef SPK_EXP_SA_INDEP
        Sample<D> w2c = w2;  // experiment: A reads sample t before S(t) (wrong results)
#endif
#ifndef SPK_EXP_NOSPEED
        if (t >= 0 && t <= ns - 2) speed_pair<D>(w2, w3, t, a, pin, L.worst);
#endif
        SPK_PROF_MARK(L, 0)
#ifndef SPK_EXP_NOACCEL
#ifdef SPK_EXP_SA_INDEP
        if (t >= 2 && t <= ns - 1) accel_triple<D>(w0, w1, w2c, t - 2, b, pin, L.worst);
#else
        if (t >= 2 && t <= ns - 1) accel_triple<D>(w0, w1, w2, t - 2, b, pin, L.worst);
#endif
#endif
        SPK_PROF_MARK(L, 1)
#ifndef SPK_EXP_NOSNAP
        if (t >= 2) {
            if (g == B - 1) {
                // round j's output stream: wrap buffer j & 1 (both the same buffer when
                // single-buffered, which then needs the global ping-pong snapshots)
                double* wb = wrap0 + (L.j & 1) * wstride;
#pragma unroll
                for (int l = 0; l < D; ++l) wb[(t - 2) * D + l] = w0.v[l];
                if (wstride == 0) {  // single wrap buffer: ping-pong snapshots in global
                    double* sn = snap0 + (L.j & 1) * (ns * D);
#pragma unroll
                    for (int l = 0; l < D; ++l) sn[(t - 2) * D + l] = w0.v[l];
                }
            }
            if (L.k == kl) {
#pragma unroll
                for (int l = 0; l < D; ++l) res[(t - 2) * D + l] = w0.v[l];
            }
        }
#endif
        // stop flags alternate per barrier block: a lane already in the next block cannot
        // change the flag the others are about to read at the end of this one
        if (t == ns + 1 && L.worst <= tol) atomicMin(&stop_sh[(st / RING_K) & 1], L.k);
    }
    // hand the finished sample w0 (= s[t-2]) to the next sweep; it is replaced in slot R
    Sample<D> recv;
#pragma unroll
    for (int l = 0; l < D; ++l) recv.v[l] = __shfl_up_sync(0xffffffffu, w0.v[l], 1);
#ifndef SPK_EXP_NOXFER
    if (lane == 31) {
        double* x = xfer + ((warp * 2 * RING_K + (st & (2 * RING_K - 1))) * D);
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = w0.v[l];
    }
#endif
    if (on) {
        const int m = t + 2;
        if (m <= ns - 1) {
            if (g == 0) {
                // first sweep of a round: the previous round's last sweep (the initial
                // state for round 0, staged at kernel start), through the wrap buffer
                const double* rb = wrap0 + ((L.j + 1) & 1) * wstride;  // round j - 1's stream
#pragma unroll
                for (int l = 0; l < D; ++l) recv.v[l] = rb[m * D + l];
            }
#ifndef SPK_EXP_NOXFER
            else if (lane == 0) {
                // emitted by lane 31 of warp - 1 at step st - RING_K
                const double* x =
                    xfer + (((warp - 1) * 2 * RING_K + ((st + RING_K) & (2 * RING_K - 1))) * D);
#pragma unroll
                for (int l = 0; l < D; ++l) recv.v[l] = x[l];
            }
#endif
            if (m == pin) {
                recv.v[0] = pv0;
                recv.v[1] = pv1;
                if (D == 3) recv.v[D - 1] = pv2;
            }
            SPK_PROF_MARK(L, 2)
#ifndef SPK_EXP_NOBOX
            box_sample<D>(recv, L.worst);
#endif
            SPK_PROF_MARK(L, 3)
        }
    }
    w0 = recv;  // slot R now holds s[t+2] (w3 at the next step)
    if (++L.t == P - 2) {
        L.t = -2;
        ++L.j;
        L.k += B;
    }
    SPK_PROF_MARK(L, 4)
#ifndef SPK_EXP_NOSYNC
    if (((st + 1) & (RING_K - 1)) == 0) __syncthreads();
#endif
#ifdef SPK_POLISH_PROF
    SPK_PROF_MARK(L, 5)
    L.prof[6] += 1;
#endif
}

// Continuous ring: lane g runs sweeps g, g+B, g+2B, ...; sweep k starts at global step
// (k / B) * P + ring_offset(k % B) with P = max(4 B + W, ns + 4).  The last lane writes
// every round's output stream into a ping-pong snapshot (and the wrap buffer that feeds
// lane 0 of the next round); when sweep k* is the first whose worst violation is
// <= tol, the ring stops and sweeps j B .. k* are replayed (systolic_batch) from the
// snapshot after sweep j B - 1 (j = k* / B), which the ring has not overwritten yet
// because P >= ns + 4.  Bit-identical to the sequential polish.
template <int D, int MAXT, int MINB, bool PEERS>
__global__ void __launch_bounds__(MAXT, MINB) polish_kernel(double* shots, int ns, double a,
                                                      double b, int pin, double pv0,
                                                      double pv1, double pv2, double tol,
                                                      int max_sweeps, double* ws,
                                                      int32_t* sweeps_out, float4* pos4,
                                                      int wrap_mode,
                                                      const int32_t* __restrict__ shot_ids,
                                                      int* sm_busy,
                                                      float4* const* __restrict__ peers,
                                                      int n_peers, long long peer_off) {
    // wrap_mode 2: two wrap buffers in shared memory (round parity), which double as the
    // replay snapshot -- no global snapshot stores on the ring's critical path;
    // 1: one shared wrap buffer + global ping-pong snapshots; 0: wrap in the workspace.
    extern __shared__ __align__(16) double xfer[];  // [W][2 RING_K][D], then wrap [1|2][ns][D]
    __shared__ int stop_sh[2];
    // shot of this CTA: the launch's shot list (a subset in any order) or blockIdx.x
    const long long c = shot_ids ? (long long)shot_ids[blockIdx.x] : (long long)blockIdx.x;
    // optional SM occupancy count: lattice-sum CTAs launched beside the polish wait for
    // their SM to hold no polish CTA (nbody_kernel, sm_busy), so they use only idle SMs
    if (sm_busy && threadIdx.x == 0) atomicAdd(&sm_busy[sm_id()], 1);
    const int B = blockDim.x;
    const int W = B >> 5;
    const int P = max(4 * B + RING_K * W, ns + 4);
    const int nd4 = ns * D;
    // wrap buffer(s) in shared memory, or (very long shots) in the per-shot workspace
    double* wrap0 = wrap_mode == 0 ? ws + c * (size_t)(4 * nd4) + 3 * nd4
                                   : xfer + W * 2 * RING_K * D;
    const int wstride = wrap_mode == 2 ? nd4 : 0;
    double* wrap1 = wrap0 + wstride;
    const int g = threadIdx.x;
    const int lane = g & 31;
    const int warp = g >> 5;
    const int off = ring_offset(g);
    const int nd = ns * D;
    const double pv[3] = {pv0, pv1, pv2};
    double* s0 = shots + c * (size_t)nd;
    double* snap0 = ws + c * (size_t)(4 * nd);
    double* snap1 = snap0 + nd;
    double* res = snap1 + nd;
    if (g == 0) stop_sh[0] = stop_sh[1] = 0x7fffffff;
    // stage the initial state in the wrap buffer: lane 0 then reads round 0 from it like
    // every later round (no global-load latency on the ring's critical path).  Lane B-1
    // overwrites position q only 4 + ring_offset(B-1) steps after lane 0 has read it.
    for (int i = g; i < nd; i += B) wrap1[i] = s0[i];  // round 0 reads buffer (0 - 1) & 1
    __syncthreads();
    const int kl = max_sweeps - 1;
    const int last_step = (kl / B) * P + ring_offset(kl % B) + ns + 3;
    RingLane<D> L;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int l = 0; l < D; ++l) L.slot[q].v[l] = 0.0;
    L.worst = 0.0;
    L.t = -2 - off;  // lane g starts its first sweep at global step off
#ifdef SPK_POLISH_PROF
    for (int q = 0; q < 7; ++q) L.prof[q] = 0;
    L.tp = clock64();
#endif
    L.j = 0;
    L.k = g;
#define SPK_RING_STEP(R)                                                                   \
    {                                                                                      \
        ring_step<D, R>(L, st + R, ns, B, P, g, lane, warp, max_sweeps, kl, a, b, pin,     \
                        pv0, pv1, pv2, tol, s0, snap0, res, xfer, wrap0, wstride,          \
                        stop_sh);                                                          \
        if (((st + R + 1) & (RING_K - 1)) == 0 &&                                          \
            stop_sh[((st + R) / RING_K) & 1] != 0x7fffffff)                                \
            break;                                                                         \
        if (st + R >= last_step) break;                                                    \
    }
    for (int st = 0;; st += 4) {
        SPK_RING_STEP(0)
        SPK_RING_STEP(1)
        SPK_RING_STEP(2)
        SPK_RING_STEP(3)
    }
#undef SPK_RING_STEP
#ifdef SPK_POLISH_PROF
    if (blockIdx.x == 0) {
        const int slot = g == 5 ? 0 : g == 40 ? 1 : g == B - 9 ? 2 : -1;
        if (slot >= 0)
            for (int q = 0; q < 7; ++q) spk_polish_prof[slot][q] = L.prof[q];
    }
#endif
    __syncthreads();  // the last_step exit can fall between barriers
    const int kstar = min(stop_sh[0], stop_sh[1]);
    int total = max_sweeps;
    if (kstar != 0x7fffffff) {
        const int jj = kstar / B;
        const double* src = jj == 0    ? s0
                            : wstride ? ((jj - 1) & 1 ? wrap1 : wrap0)
                                     : ((jj - 1) & 1 ? snap1 : snap0);
        __syncthreads();
        systolic_batch<D>(src, res, xfer, ns, a, b, pin, pv, kstar - jj * B + 1);
        total = kstar + 1;
    }
    __syncthreads();
    for (int i = g; i < nd; i += B) s0[i] = res[i];
    if (pos4) {
        for (int n = g; n < ns; n += B) {
            const double* r = res + n * D;
            pos4[c * ns + n] = pos_record(r[0], r[1], D == 3 ? r[2] : 0.0);
        }
        if (PEERS) {
            // multi-GPU: the shot's records into every other rank's position buffer (peer
            // memory over NVLink) -- the all-gather of positions fused into the epilogue.
            // Re-read from this CTA's own (L1/L2-resident) stores so the ring above keeps
            // its register budget; a separate instantiation, so the single-GPU kernel is
            // unchanged.
            __syncthreads();
            const float4* mine = pos4 + c * ns;
            for (int k = 0; k < n_peers; ++k) {
                float4* dst = peers[k] + peer_off + c * ns;
                for (int n = g; n < ns; n += B) dst[n] = mine[n];
            }
        }
    }
    if (g == 0 && sweeps_out) sweeps_out[c] = total;
    if (sm_busy) {
        __syncthreads();
        if (threadIdx.x == 0) atomicSub(&sm_busy[sm_id()], 1);
    }
}

// Positions of the listed shots into every peer buffer (the fused gather's path for the
// wide rings, launched right after their polish).
__global__ void peer_copy_kernel(const float4* __restrict__ pos4,
                                 const int32_t* __restrict__ shot_ids, int ns,
                                 float4* const* __restrict__ peers, int n_peers,
                                 long long peer_off) {
    const long long c = shot_ids ? (long long)shot_ids[blockIdx.x] : (long long)blockIdx.x;
    for (int k = 0; k < n_peers; ++k)
        for (int n = threadIdx.x; n < ns; n += blockDim.x)
            peers[k][peer_off + c * ns + n] = pos4[c * ns + n];
}

// CTAs per SM the <= 8-warp polish instantiation is register-budgeted for.
#ifndef SPK_POLISH_MINB
#define SPK_POLISH_MINB 3
#endif
constexpr int PL_MINB = SPK_POLISH_MINB;
// Wider rings (> 8 warps, N_s > 1283): the instantiation's thread bound and CTAs per SM.
#ifndef SPK_POLISH_WIDE_T
#define SPK_POLISH_WIDE_T 1024
#endif
#ifndef SPK_POLISH_WIDE_MINB
#define SPK_POLISH_WIDE_MINB 1
#endif
constexpr int PL_WIDE_T = SPK_POLISH_WIDE_T;
constexpr int PL_WIDE_MINB = SPK_POLISH_WIDE_MINB;

// Ring width: W warps; SPK_POLISH_WARPS overrides (fewer warps -> more shots resident
// per SM, longer per-sweep latency).
inline int polish_warps(int ns) {
    // 4 B + RING_K W >= ns + 4: no idle lane in the ring
    int w = (ns + 4 + 127 + RING_K) / (128 + RING_K);
    if (const char* e = getenv("SPK_POLISH_WARPS")) w = atoi(e);
    return w < 1 ? 1 : (w > 32 ? 32 : w);
}

// ------------------------------------------------------------------ residuals
constexpr int RS_THREADS = 256;

template <int D>
__global__ void residual_kernel(const double* __restrict__ co, int ns, int pin, double pv0,
                                double pv1, double pv2, double* __restrict__ per_shot) {
    __shared__ double red[4][RS_THREADS];
    const long long c = blockIdx.x;
    const double* x = co + c * (size_t)ns * D;
    const double pv[3] = {pv0, pv1, pv2};
    double amp = 0.0, sp = -INFINITY, ac = -INFINITY, pe = 0.0;
    for (int n = threadIdx.x; n < ns; n += RS_THREADS) {
        for (int l = 0; l < D; ++l) amp = fmax(amp, fabs(x[n * D + l]));
        if (n <= ns - 2) {
            double q = 0.0;
            for (int l = 0; l < D; ++l) {
                const double df = x[(n + 1) * D + l] - x[n * D + l];
                q = (l == 0) ? df * df : q + df * df;
            }
            sp = fmax(sp, sqrt(q));
        }
        if (n <= ns - 3) {
            double q = 0.0;
            for (int l = 0; l < D; ++l) {
                // np.diff(coords, 2) = diff of diffs
                const double d2 = (x[(n + 2) * D + l] - x[(n + 1) * D + l]) -
                                  (x[(n + 1) * D + l] - x[n * D + l]);
                q = (l == 0) ? d2 * d2 : q + d2 * d2;
            }
            ac = fmax(ac, sqrt(q));
        }
        if (n == pin)
            for (int l = 0; l < D; ++l) pe = fmax(pe, fabs(x[n * D + l] - pv[l]));
    }
    red[0][threadIdx.x] = amp;
    red[1][threadIdx.x] = sp;
    red[2][threadIdx.x] = ac;
    red[3][threadIdx.x] = pe;
    __syncthreads();
    for (int w = RS_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 4; ++q)
                red[q][threadIdx.x] = fmax(red[q][threadIdx.x], red[q][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x < 4) per_shot[c * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void residual_final_kernel(const double* __restrict__ per_shot_all, long long n_shots,
                                      double a, double b, int has_pin,
                                      double* __restrict__ out_all) {
    // one block per group of n_shots shots (a single pattern: one block)
    __shared__ double red[4][RS_THREADS];
    const double* per_shot = per_shot_all + (long long)blockIdx.x * n_shots * 4;
    double* out = out_all + (long long)blockIdx.x * 5;
    double m[4] = {0.0, -INFINITY, -INFINITY, 0.0};
    for (long long c = threadIdx.x; c < n_shots; c += RS_THREADS)
        for (int q = 0; q < 4; ++q) m[q] = fmax(m[q], per_shot[c * 4 + q]);
    for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = m[q];
    __syncthreads();
    for (int w = RS_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 4; ++q)
                red[q][threadIdx.x] = fmax(red[q][threadIdx.x], red[q][threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        // feasibility_residuals (projection.py:435-452)
        const double amp = fmax(red[0][0] - 1.0, 0.0);
        const double sp = fmax(red[1][0] - a, 0.0);
        const double ac = fmax(red[2][0] - b, 0.0);
        const double pe = has_pin ? red[3][0] : 0.0;
        out[0] = amp;
        out[1] = sp;
        out[2] = ac;
        out[3] = pe;
        out[4] = fmax(fmax(amp, sp), fmax(ac, pe));
    }
}

// ------------------------------------------------------------------ upsample
__global__ void upsample_kernel(const double* __restrict__ in, double* __restrict__ out,
                                long long n_shots, int ns, int dims) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long total = n_shots * 2 * ns * dims;
    if (idx >= total) return;
    const int l = (int)(idx % dims);
    const long long m = (idx / dims) % (2 * ns);
    const long long c = idx / ((long long)dims * 2 * ns);
    const double* x = in + c * (long long)ns * dims;
    double v;
    if ((m & 1) == 0) {
        v = x[(m / 2) * dims + l];
    } else if (m < 2 * ns - 1) {
        const long long j = m / 2;
        v = 0.5 * (x[j * dims + l] + x[(j + 1) * dims + l]);
    } else {
        const double last = x[(ns - 1) * dims + l];
        v = last + 0.5 * (last - x[(ns - 2) * dims + l]);
    }
    v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);  // np.clip
    out[idx] = v;
}

// ------------------------------------------------------- field-path attraction
// Mirrors attraction.py:116-255 (_clamp_points, _interp2/3, _cell_grad2/3), fp64.
__global__ void field_eval_kernel(const double* __restrict__ pts, long long p, int dims,
                                  const double* __restrict__ pot,
                                  const double* __restrict__ force, long long n, int mode,
                                  double* __restrict__ vals, double* __restrict__ grad,
                                  unsigned long long* __restrict__ n_clamped) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= p) return;
    const long long side = 2 * n + 1;
    const double hi = 2.0 * (double)n;
    double u[3] = {0, 0, 0};
    bool bad = false;
    for (int l = 0; l < dims; ++l) {
        double v = (pts[i * dims + l] + 1.0) * (double)n;
        if (v < 0.0) {
            v = 0.0;
            bad = true;
        } else if (v > hi) {
            v = hi;
            bad = true;
        }
        u[l] = v;
    }
    if (bad) atomicAdd(n_clamped, 1ull);
    long long i0 = (long long)u[0], j0 = (long long)u[1], k0 = dims == 3 ? (long long)u[2] : 0;
    i0 = i0 < side - 2 ? i0 : side - 2;
    j0 = j0 < side - 2 ? j0 : side - 2;
    k0 = k0 < side - 2 ? k0 : side - 2;
    const double fx = u[0] - (double)i0, fy = u[1] - (double)j0;
    const double fz = dims == 3 ? u[2] - (double)k0 : 0.0;
    const double scale = (double)n;
    if (dims == 2) {
        auto G = [&](const double* g, long long a, long long bb) { return g[a * side + bb]; };
        auto interp2 = [&](const double* g) {
            return (1 - fx) * (1 - fy) * G(g, i0, j0) + fx * (1 - fy) * G(g, i0 + 1, j0) +
                   (1 - fx) * fy * G(g, i0, j0 + 1) + fx * fy * G(g, i0 + 1, j0 + 1);
        };
        vals[i] = interp2(pot);
        if (mode == 0) {
            double gx0 = G(pot, i0 + 1, j0) - G(pot, i0, j0);
            double gx1 = G(pot, i0 + 1, j0 + 1) - G(pot, i0, j0 + 1);
            if (fx == 0.0 && i0 > 0) {
                gx0 = 0.5 * (G(pot, i0 + 1, j0) - G(pot, i0 - 1, j0));
                gx1 = 0.5 * (G(pot, i0 + 1, j0 + 1) - G(pot, i0 - 1, j0 + 1));
            }
            grad[i * 2] = scale * ((1 - fy) * gx0 + fy * gx1);
            double gy0 = G(pot, i0, j0 + 1) - G(pot, i0, j0);
            double gy1 = G(pot, i0 + 1, j0 + 1) - G(pot, i0 + 1, j0);
            if (fy == 0.0 && j0 > 0) {
                gy0 = 0.5 * (G(pot, i0, j0 + 1) - G(pot, i0, j0 - 1));
                gy1 = 0.5 * (G(pot, i0 + 1, j0 + 1) - G(pot, i0 + 1, j0 - 1));
            }
            grad[i * 2 + 1] = scale * ((1 - fx) * gy0 + fx * gy1);
        } else {
            const long long plane = side * side;
            grad[i * 2] = interp2(force);
            grad[i * 2 + 1] = interp2(force + plane);
        }
        return;
    }
    auto G3 = [&](const double* g, long long a, long long bb, long long cc) {
        return g[(a * side + bb) * side + cc];
    };
    auto interp3 = [&](const double* g) {
        double v = 0.0;
        for (int ii = 0; ii < 2; ++ii) {
            const double wx = ii == 1 ? fx : 1 - fx;
            for (int jj = 0; jj < 2; ++jj) {
                const double wy = jj == 1 ? fy : 1 - fy;
                for (int kk = 0; kk < 2; ++kk) {
                    const double wz = kk == 1 ? fz : 1 - fz;
                    v += wx * wy * wz * G3(g, i0 + ii, j0 + jj, k0 + kk);
                }
            }
        }
        return v;
    };
    vals[i] = interp3(pot);
    if (mode == 0) {
        for (int ax = 0; ax < 3; ++ax) {
            const double f_ax = ax == 0 ? fx : (ax == 1 ? fy : fz);
            const long long a0 = ax == 0 ? i0 : (ax == 1 ? j0 : k0);
            const bool central = f_ax == 0.0 && a0 > 0;
            double g = 0.0;
            for (int jj = 0; jj < 2; ++jj) {
                for (int kk = 0; kk < 2; ++kk) {
                    double w, hv, lv;
                    if (ax == 0) {
                        w = (jj == 1 ? fy : 1 - fy) * (kk == 1 ? fz : 1 - fz);
                        hv = G3(pot, i0 + 1, j0 + jj, k0 + kk);
                        lv = central ? G3(pot, i0 - 1, j0 + jj, k0 + kk)
                                     : G3(pot, i0, j0 + jj, k0 + kk);
                    } else if (ax == 1) {
                        w = (jj == 1 ? fx : 1 - fx) * (kk == 1 ? fz : 1 - fz);
                        hv = G3(pot, i0 + jj, j0 + 1, k0 + kk);
                        lv = central ? G3(pot, i0 + jj, j0 - 1, k0 + kk)
                                     : G3(pot, i0 + jj, j0, k0 + kk);
                    } else {
                        w = (jj == 1 ? fx : 1 - fx) * (kk == 1 ? fy : 1 - fy);
                        hv = G3(pot, i0 + jj, j0 + kk, k0 + 1);
                        lv = central ? G3(pot, i0 + jj, j0 + kk, k0 - 1)
                                     : G3(pot, i0 + jj, j0 + kk, k0);
                    }
                    g += w * (hv - lv);
                }
            }
            if (central) g *= 0.5;
            grad[i * 3 + ax] = scale * g;
        }
    } else {
        const long long vol = side * side * side;
        for (int ax = 0; ax < 3; ++ax) grad[i * 3 + ax] = interp3(force + ax * vol);
    }
}

}  // namespace spk

using namespace spk;

static size_t proj_state_doubles(int n_s, int dims) {
    return (size_t)PJ_WS_ARRAYS * (size_t)n_s * dims;
}

extern "C" {

#ifdef SPK_POLISH_PROF
int spk_polish_prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, spk_polish_prof, sizeof(unsigned long long) * 21) ==
                   cudaSuccess
               ? 0
               : 4;
}
#endif

size_t spk_project_workspace_bytes(int64_t n_shots, int n_s, int dims, int with_trace) {
    (void)with_trace;
    return (size_t)n_shots * proj_state_doubles(n_s, dims) * sizeof(double) + 256;
}

static int launch_fista(const double* in, const double* grad, double eta,
                        const double* eta_per_shot, double* out, int64_t n_shots, int n_s,
                        int dims, double a, double b, int pin_idx, const double* pin_val,
                        int n_pit, double tau, int monotone, double* trace,
                        int32_t* nonfinite, void* ws, cudaStream_t stream) {
    ProjArgs A;
    A.in = in;
    A.grad = grad;
    A.eta = eta;
    A.eta_shot = eta_per_shot;
    A.out = out;
    A.n_shots = n_shots;
    A.ns = n_s;
    A.a = a;
    A.b = b;
    A.pin = pin_idx < 0 ? -1 : pin_idx;
    for (int l = 0; l < 3; ++l) A.pv[l] = (pin_idx >= 0 && l < dims) ? pin_val[l] : 0.0;
    A.n_pit = n_pit;
    A.tau = tau;
    A.monotone = monotone;
    A.trace = trace;
    A.nonfinite = nonfinite;
    A.ws = static_cast<double*>(ws);
    A.ws_stride = (long long)proj_state_doubles(n_s, dims);
    const size_t smem3 = (size_t)3 * n_s * dims * sizeof(double);
    const size_t smem4 = (size_t)4 * n_s * dims * sizeof(double);
    A.smem_arrays = smem4 <= (size_t)PJ_SMEM_LIMIT ? 2 : smem3 <= (size_t)PJ_SMEM_LIMIT ? 1 : 0;
    const size_t dyn = A.smem_arrays == 2 ? smem4 : A.smem_arrays == 1 ? smem3 : 0;
    int nt = PJ_THREADS;
    if (n_s < PJ_THREADS) nt = ((n_s + 31) / 32) * 32;
    if (dims == 3) {
        cudaFuncSetAttribute(fista_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn);
        fista_kernel<3><<<(unsigned)n_shots, nt, dyn, stream>>>(A);
    } else {
        cudaFuncSetAttribute(fista_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn);
        fista_kernel<2><<<(unsigned)n_shots, nt, dyn, stream>>>(A);
    }
    SPK_CHECK_LAUNCH("fista_kernel");
    return SPK_OK;
}

// Polish (systolic ring, one CTA of 32 pw lanes per shot) of n_ids shots: shot_ids[i]
// (or i when shot_ids is null).  Snapshots + result live in that shot's slot of the FISTA
// workspace, warp hand-over slots and wrap buffers in shared memory.
static int launch_polish(double* shots, const int32_t* shot_ids, int64_t n_ids, int n_s,
                         int dims, double a, double b, int pin_idx, const double* pin_val,
                         double tol, int max_sweeps, void* pos4, int32_t* sweeps, void* ws,
                         cudaStream_t stream, int* sm_busy = nullptr,
                         float4* const* peers = nullptr, int n_peers = 0,
                         long long peer_off = 0) {
    if (n_ids <= 0) return SPK_OK;
    const int pin = pin_idx < 0 ? -1 : pin_idx;
    double pv[3] = {0, 0, 0};
    for (int l = 0; l < dims; ++l)
        if (pin_idx >= 0) pv[l] = pin_val[l];
    const int pw = polish_warps(n_s);
    const size_t xb = (size_t)pw * 2 * RING_K * dims * sizeof(double);
    const size_t wb = (size_t)n_s * dims * sizeof(double);
    const int wrap_mode = xb + 2 * wb <= 200 * 1024 ? 2 : xb + wb <= 200 * 1024 ? 1 : 0;
    const size_t psm = xb + (wrap_mode == 2 ? 2 * wb : wrap_mode == 1 ? wb : 0);
    double* pws = static_cast<double*>(ws);
    // <= 8 warps (N_s <= 1283): a register budget of 80 keeps the ring window in registers
    // with 3 CTAs per SM; wider rings use the 1024-thread instantiation
    const dim3 grid((unsigned)n_ids), block(32 * pw);
#define PL_LAUNCH1(DD, TT, MB, PP)                                                         \
    do {                                                                                   \
        cudaFuncSetAttribute(polish_kernel<DD, TT, MB, PP>,                                \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);       \
        polish_kernel<DD, TT, MB, PP><<<grid, block, psm, stream>>>(                       \
            shots, n_s, a, b, pin, pv[0], pv[1], pv[2], tol, max_sweeps, pws, sweeps,       \
            (float4*)pos4, wrap_mode, shot_ids, sm_busy, peers, n_peers, peer_off);         \
    } while (0)
#define PL_LAUNCH(DD, TT, MB)                           \
    do {                                                \
        if (n_peers > 0) PL_LAUNCH1(DD, TT, MB, true);  \
        else PL_LAUNCH1(DD, TT, MB, false);             \
    } while (0)
    if (pw <= 8) {
        if (dims == 3) PL_LAUNCH(3, 256, PL_MINB);
        else PL_LAUNCH(2, 256, PL_MINB);
    } else {
        // wide rings run at the 64-register edge: the peer epilogue would add spills to
        // the ring, so they keep the single-GPU kernel and copy to the peers right after
        const int np = n_peers;
        n_peers = 0;
        if (32 * pw <= PL_WIDE_T) {
            if (dims == 3) PL_LAUNCH(3, PL_WIDE_T, PL_WIDE_MINB);
            else PL_LAUNCH(2, PL_WIDE_T, PL_WIDE_MINB);
        } else {
            if (dims == 3) PL_LAUNCH(3, 1024, 1);
            else PL_LAUNCH(2, 1024, 1);
        }
        if (np > 0)
            peer_copy_kernel<<<(unsigned)n_ids, 256, 0, stream>>>(
                (const float4*)pos4, shot_ids, n_s, peers, np, peer_off);
    }
#undef PL_LAUNCH1
#undef PL_LAUNCH
    SPK_CHECK_LAUNCH("polish_kernel");
    return SPK_OK;
}

#define SPK_PROJECT_CHECKS                                                                 \
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);  \
    SPK_REQUIRE(n_s >= 2, SPK_ERR_ARG, "projection needs at least 2 samples per shot");    \
    SPK_REQUIRE(pin_idx < n_s, SPK_ERR_ARG, "pinned_index %d out of range for N_s=%d",     \
                pin_idx, n_s)

int spk_project_all(const double* in, const double* grad, double eta,
                    const double* eta_per_shot, double* out,
                    int64_t n_shots, int n_s, int dims, double a, double b, int pin_idx,
                    const double* pin_val, int n_pit, double tau, int monotone, double tol,
                    int max_sweeps, void* pos4, int32_t* sweeps, double* trace,
                    int32_t* nonfinite, void* ws, size_t ws_bytes, spk_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SPK_PROJECT_CHECKS;
    SPK_REQUIRE(n_pit >= 1, SPK_ERR_ARG, "n_pit must be >= 1");
    SPK_REQUIRE(max_sweeps >= 1, SPK_ERR_ARG, "max_sweeps must be >= 1");
    if (n_shots <= 0) return SPK_OK;
    const size_t need = spk_project_workspace_bytes(n_shots, n_s, dims, trace != nullptr);
    SPK_REQUIRE(ws != nullptr && ws_bytes >= need, SPK_ERR_WORKSPACE,
                "projection workspace too small: need %zu, got %zu", need, ws_bytes);
    int rc = launch_fista(in, grad, eta, eta_per_shot, out, n_shots, n_s, dims, a, b, pin_idx,
                          pin_val, n_pit, tau, monotone, trace, nonfinite, ws, stream);
    if (rc != SPK_OK) return rc;
    return launch_polish(out, nullptr, n_shots, n_s, dims, a, b, pin_idx, pin_val, tol,
                         max_sweeps, pos4, sweeps, ws, stream);
}

int spk_project_fista(const double* in, const double* grad, double eta,
                      const double* eta_per_shot, double* out, int64_t n_shots, int n_s,
                      int dims, double a, double b, int pin_idx, const double* pin_val,
                      int n_pit, double tau, int monotone, double* trace, int32_t* nonfinite,
                      void* ws, size_t ws_bytes, spk_stream_t stream) {
    SPK_PROJECT_CHECKS;
    SPK_REQUIRE(n_pit >= 1, SPK_ERR_ARG, "n_pit must be >= 1");
    if (n_shots <= 0) return SPK_OK;
    const size_t need = spk_project_workspace_bytes(n_shots, n_s, dims, trace != nullptr);
    SPK_REQUIRE(ws != nullptr && ws_bytes >= need, SPK_ERR_WORKSPACE,
                "projection workspace too small: need %zu, got %zu", need, ws_bytes);
    return launch_fista(in, grad, eta, eta_per_shot, out, n_shots, n_s, dims, a, b, pin_idx,
                        pin_val, n_pit, tau, monotone, trace, nonfinite, ws,
                        (cudaStream_t)stream);
}

int spk_polish_shots(double* shots, const int32_t* shot_ids, int64_t n_ids, int64_t n_shots,
                     int n_s, int dims, double a, double b, int pin_idx, const double* pin_val,
                     double tol, int max_sweeps, void* pos4, int32_t* sweeps,
                     int32_t* sm_busy, void* const* peer_pos4, int n_peers,
                     int64_t peer_offset, void* ws, size_t ws_bytes, spk_stream_t stream) {
    SPK_PROJECT_CHECKS;
    SPK_REQUIRE(max_sweeps >= 1, SPK_ERR_ARG, "max_sweeps must be >= 1");
    SPK_REQUIRE(n_ids >= 0 && n_ids <= n_shots, SPK_ERR_ARG, "polish: %lld ids for %lld shots",
                (long long)n_ids, (long long)n_shots);
    SPK_REQUIRE(n_peers >= 0 && (n_peers == 0 || (peer_pos4 != nullptr && pos4 != nullptr)),
                SPK_ERR_ARG, "polish: %d peer buffers need the peer table and pos4", n_peers);
    if (n_ids <= 0) return SPK_OK;
    const size_t need = spk_project_workspace_bytes(n_shots, n_s, dims, 0);
    SPK_REQUIRE(ws != nullptr && ws_bytes >= need, SPK_ERR_WORKSPACE,
                "projection workspace too small: need %zu, got %zu", need, ws_bytes);
    return launch_polish(shots, shot_ids, n_ids, n_s, dims, a, b, pin_idx, pin_val, tol,
                         max_sweeps, pos4, sweeps, ws, (cudaStream_t)stream, sm_busy,
                         reinterpret_cast<float4* const*>(peer_pos4), n_peers, peer_offset);
}

size_t spk_residuals_workspace_bytes(int64_t n_shots) {
    return (size_t)n_shots * 4 * sizeof(double) + 256;
}

int spk_feasibility_residuals(const double* coords, int64_t n_shots, int n_s, int dims,
                              double a, double b, int pin_idx, const double* pin_val,
                              double* out, void* ws, size_t ws_bytes, spk_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    SPK_REQUIRE(n_shots >= 1 && n_s >= 1, SPK_ERR_ARG, "empty pattern");
    SPK_REQUIRE(ws_bytes >= spk_residuals_workspace_bytes(n_shots), SPK_ERR_WORKSPACE,
                "residual workspace too small");
    double pv[3] = {0, 0, 0};
    if (pin_idx >= 0)
        for (int l = 0; l < dims; ++l) pv[l] = pin_val[l];
    double* per = static_cast<double*>(ws);
    if (dims == 3)
        residual_kernel<3><<<(unsigned)n_shots, RS_THREADS, 0, stream>>>(
            coords, n_s, pin_idx, pv[0], pv[1], pv[2], per);
    else
        residual_kernel<2><<<(unsigned)n_shots, RS_THREADS, 0, stream>>>(
            coords, n_s, pin_idx, pv[0], pv[1], pv[2], per);
    residual_final_kernel<<<1, RS_THREADS, 0, stream>>>(per, n_shots, a, b, pin_idx >= 0, out);
    SPK_CHECK_LAUNCH("feasibility_residuals");
    return SPK_OK;
}

int spk_feasibility_residuals_batched(const double* coords, int64_t n_groups,
                                      int64_t shots_per_group, int n_s, int dims, double a,
                                      double b, int pin_idx, const double* pin_val, double* out,
                                      void* ws, size_t ws_bytes, spk_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    SPK_REQUIRE(n_groups >= 1 && shots_per_group >= 1 && n_s >= 1, SPK_ERR_ARG, "empty batch");
    const long long n_shots = n_groups * shots_per_group;
    SPK_REQUIRE(ws_bytes >= spk_residuals_workspace_bytes(n_shots), SPK_ERR_WORKSPACE,
                "residual workspace too small");
    double pv[3] = {0, 0, 0};
    if (pin_idx >= 0)
        for (int l = 0; l < dims; ++l) pv[l] = pin_val[l];
    double* per = static_cast<double*>(ws);
    if (dims == 3)
        residual_kernel<3><<<(unsigned)n_shots, RS_THREADS, 0, stream>>>(
            coords, n_s, pin_idx, pv[0], pv[1], pv[2], per);
    else
        residual_kernel<2><<<(unsigned)n_shots, RS_THREADS, 0, stream>>>(
            coords, n_s, pin_idx, pv[0], pv[1], pv[2], per);
    residual_final_kernel<<<(unsigned)n_groups, RS_THREADS, 0, stream>>>(
        per, shots_per_group, a, b, pin_idx >= 0, out);
    SPK_CHECK_LAUNCH("feasibility_residuals_batched");
    return SPK_OK;
}

int spk_upsample_shots(const double* in, double* out, int64_t n_shots, int n_s, int dims,
                       spk_stream_t stream) {
    SPK_REQUIRE(n_s >= 2, SPK_ERR_ARG, "need at least 2 samples to upsample");
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    const long long total = n_shots * 2LL * n_s * dims;
    if (total == 0) return SPK_OK;
    upsample_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        in, out, n_shots, n_s, dims);
    SPK_CHECK_LAUNCH("upsample_shots");
    return SPK_OK;
}

int spk_field_eval(const double* pts, int64_t p, int dims, const double* potential,
                   const double* force, int64_t grid_n, int mode, double* vals, double* grad,
                   int64_t* n_clamped, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3");
    SPK_REQUIRE(mode == 0 || mode == 1, SPK_ERR_ARG, "unknown grad mode %d", mode);
    SPK_REQUIRE(grid_n >= 1, SPK_ERR_ARG, "grid_n must be >= 1");
    SPK_REQUIRE(mode == 0 || force != nullptr, SPK_ERR_ARG, "smooth mode needs force grids");
    cudaMemsetAsync(n_clamped, 0, sizeof(int64_t), (cudaStream_t)stream);
    if (p <= 0) return SPK_OK;
    field_eval_kernel<<<(unsigned)((p + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        pts, p, dims, potential, force, grid_n, mode, vals, grad,
        reinterpret_cast<unsigned long long*>(n_clamped));
    SPK_CHECK_LAUNCH("field_eval");
    return SPK_OK;
}

}  // extern "C"
