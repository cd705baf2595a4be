/*
 * spk_oracle.c -- CPU restatement of the vdtraj hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 kernels in paper_2108_02991_b200/csrc.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path never links it.
 *
 * Every function restates one reference routine (paths relative to
 * /root/reference/pkg/src/vdtraj/) in plain C, fp64, with the reference's operation
 * order so that results are bit-identical to the numba kernels (numba compiles with
 * fastmath off: no FMA contraction, IEEE sqrt/div).  Build with -ffp-contract=off and
 * without -ffast-math (see oracle/Makefile).  Bitwise agreement is pinned against
 * fixtures generated from the reference itself (tests/golden/make_golden.py).
 *
 * Layouts: positions (p, d) row-major f64; shots (n_shots, ns, d) row-major f64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Row sums for a block of target rows.  For every row the source loop is the reference's
 * sequential j = 0..p-1 loop with the reference's operations (_treecode.py:515-534):
 * r2 = eps2 + dx*dx + dy*dy (+ dz*dz), h = sqrt(r2), v += h, gradient term only when
 * h > 0.  Rows are processed in blocks over cache-sized source tiles; that changes the
 * interleaving between rows, never the order of any row's own accumulation, so results
 * stay bit-identical to the reference. */
#define ROW_BLOCK 8
#define SRC_TILE 2048

static void rows_block(const double* pos, int64_t p, int d, const double* tcoords, int nr,
                       double eps2, double* val, double* grad) {
    double v[ROW_BLOCK] = {0}, gx[ROW_BLOCK] = {0}, gy[ROW_BLOCK] = {0}, gz[ROW_BLOCK] = {0};
    for (int64_t j0 = 0; j0 < p; j0 += SRC_TILE) {
        const int64_t j1 = (j0 + SRC_TILE < p) ? j0 + SRC_TILE : p;
        for (int r = 0; r < nr; ++r) {
            const double xi = tcoords[r * d + 0];
            const double yi = tcoords[r * d + 1];
            const double zi = (d == 3) ? tcoords[r * d + 2] : 0.0;
            double vv = v[r], ax = gx[r], ay = gy[r], az = gz[r];
            if (d == 3) {
                for (int64_t j = j0; j < j1; ++j) {
                    const double* q = pos + j * 3;
                    double dx = xi - q[0];
                    double dy = yi - q[1];
                    double r2 = eps2 + dx * dx + dy * dy;
                    double dz = zi - q[2];
                    r2 += dz * dz;
                    double h = sqrt(r2);
                    vv += h;
                    if (h > 0.0) {
                        double inv = 1.0 / h;
                        ax += dx * inv;
                        ay += dy * inv;
                        az += dz * inv;
                    }
                }
            } else {
                for (int64_t j = j0; j < j1; ++j) {
                    const double* q = pos + j * 2;
                    double dx = xi - q[0];
                    double dy = yi - q[1];
                    double r2 = eps2 + dx * dx + dy * dy;
                    double h = sqrt(r2);
                    vv += h;
                    if (h > 0.0) {
                        double inv = 1.0 / h;
                        ax += dx * inv;
                        ay += dy * inv;
                    }
                }
            }
            v[r] = vv;
            gx[r] = ax;
            gy[r] = ay;
            gz[r] = az;
        }
    }
    for (int r = 0; r < nr; ++r) {
        val[r] = v[r];
        grad[r * d + 0] = gx[r];
        grad[r * d + 1] = gy[r];
        if (d == 3) grad[r * d + 2] = gz[r];
    }
}

/* Target rows come from `tcoords` (m, d) when given, else from pos[targets[r]] (or
 * pos[r] when targets is NULL). */
static void rows_all(const double* pos, int64_t p, int d, const int64_t* targets,
                     const double* tcoords, int64_t m, double eps2, double* val,
                     double* grad) {
    const int64_t nblk = (m + ROW_BLOCK - 1) / ROW_BLOCK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nblk; ++b) {
        double tc[ROW_BLOCK * 3];
        const int64_t r0 = b * ROW_BLOCK;
        const int nr = (int)((m - r0 < ROW_BLOCK) ? m - r0 : ROW_BLOCK);
        for (int r = 0; r < nr; ++r) {
            const double* src = tcoords ? tcoords + (r0 + r) * d
                                        : pos + (targets ? targets[r0 + r] : r0 + r) * d;
            for (int l = 0; l < d; ++l) tc[r * d + l] = src[l];
        }
        rows_block(pos, p, d, tc, nr, eps2, val + r0, grad + r0 * d);
    }
}

/* direct_sums (_treecode.py:506-534): exact all-pairs kernel sums. */
void or_direct_sums(const double* pos, int64_t p, int d, double eps2,
                    double* val, double* grad, int nthreads) {
    set_threads(nthreads);
    rows_all(pos, p, d, NULL, NULL, p, eps2, val, grad);
}

/* direct_sums_subset (_treecode.py:474-503): rows for a list of targets.  Also used
 * as the big-p oracle on strided row samples. */
void or_direct_sums_subset(const double* pos, int64_t p, int d, const int64_t* targets,
                           int64_t m, double eps2, double* val, double* grad, int nthreads) {
    set_threads(nthreads);
    rows_all(pos, p, d, targets, NULL, m, eps2, val, grad);
}

/* Rows for arbitrary target points against the sources `pos` (the sharded form:
 * this rank's samples as targets, all samples as sources). */
void or_cross_sums(const double* tgt, int64_t m, const double* pos, int64_t p, int d,
                   double eps2, double* val, double* grad, int nthreads) {
    set_threads(nthreads);
    rows_all(pos, p, d, NULL, tgt, m, eps2, val, grad);
}

/* Exact density-weighted attraction sums over a (2N_a+1)-per-axis node grid.
 * For target x: v = sum_y rho(y) sqrt(|x-y|^2 + eps2), g = sum_y rho(y)(x-y)/h.
 * Node i on axis a sits at (i - N_a)/N_a (density.py:58-67, 99-113).  Loop
 * structure follows direct_sums with the weight applied to both terms; cells are
 * visited in row-major (i, j, k) order for every target.  At grid-node targets this
 * equals precompute_field's linear convolution (attraction.py:62-113) to rounding
 * (pinned in tests/test_oracle.py). */
void or_grid_sums(const double* tgt, int64_t m, int d, const double* rho,
                  const int64_t* side, double eps2, double* val, double* grad,
                  int nthreads) {
    set_threads(nthreads);
    const int64_t s0 = side[0], s1 = side[1], s2 = (d == 3) ? side[2] : 1;
    const int64_t h0 = (s0 - 1) / 2, h1 = (s1 - 1) / 2, h2 = (d == 3) ? (s2 - 1) / 2 : 1;
    double* ax0 = (double*)malloc(sizeof(double) * (size_t)(s0 + s1 + s2));
    double* ax1 = ax0 + s0;
    double* ax2 = ax1 + s1;
    for (int64_t i = 0; i < s0; ++i) ax0[i] = (double)(i - h0) / (double)h0;
    for (int64_t i = 0; i < s1; ++i) ax1[i] = (double)(i - h1) / (double)h1;
    for (int64_t i = 0; i < s2; ++i) ax2[i] = (d == 3) ? (double)(i - h2) / (double)h2 : 0.0;
    const int64_t nblk = (m + ROW_BLOCK - 1) / ROW_BLOCK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t bk = 0; bk < nblk; ++bk) {
        const int64_t r0 = bk * ROW_BLOCK;
        const int nr = (int)((m - r0 < ROW_BLOCK) ? m - r0 : ROW_BLOCK);
        double v[ROW_BLOCK] = {0}, gx[ROW_BLOCK] = {0}, gy[ROW_BLOCK] = {0},
               gz[ROW_BLOCK] = {0};
        for (int64_t i = 0; i < s0; ++i) {          /* one slab of cells at a time */
            const double* slab = rho + i * s1 * s2;
            for (int r = 0; r < nr; ++r) {
                const double* t = tgt + (r0 + r) * d;
                const double xi = t[0], yi = t[1], zi = (d == 3) ? t[2] : 0.0;
                const double dx = xi - ax0[i];
                double vv = v[r], gxx = gx[r], gyy = gy[r], gzz = gz[r];
                for (int64_t j = 0; j < s1; ++j) {
                    const double dy = yi - ax1[j];
                    const double* row = slab + j * s2;
                    for (int64_t k = 0; k < s2; ++k) {
                        const double w = row[k];
                        double r2 = eps2 + dx * dx + dy * dy;
                        double dz = 0.0;
                        if (d == 3) {
                            dz = zi - ax2[k];
                            r2 += dz * dz;
                        }
                        double h = sqrt(r2);
                        vv += w * h;
                        if (h > 0.0) {
                            double winv = w / h;
                            gxx += dx * winv;
                            gyy += dy * winv;
                            gzz += dz * winv;
                        }
                    }
                }
                v[r] = vv;
                gx[r] = gxx;
                gy[r] = gyy;
                gz[r] = gzz;
            }
        }
        for (int r = 0; r < nr; ++r) {
            val[r0 + r] = v[r];
            grad[(r0 + r) * d + 0] = gx[r];
            grad[(r0 + r) * d + 1] = gy[r];
            if (d == 3) grad[(r0 + r) * d + 2] = gz[r];
        }
    }
    free(ax0);
}

/* ------------------------------------------------------------------------------
 * Shot projection (projection.py).  Arrays: k, s (ns, d); q0,y0,z0 (ns, d);
 * q1,y1,z1 (ns-1, d); q2,y2,z2 (ns-2, d).
 * ---------------------------------------------------------------------------- */

#define AT(arr, n, l) (arr)[(n) * d + (l)]

/* _dual_to_primal (projection.py:103-123). */
static void dual_to_primal(const double* k, const double* q0, const double* q1,
                           const double* q2, int ns, int d, int pin_idx,
                           const double* pin_val, double* s) {
    for (int n = 0; n < ns; ++n) {
        for (int l = 0; l < d; ++l) {
            double r = AT(q0, n, l);
            if (n <= ns - 2) r -= AT(q1, n, l);
            if (n >= 1) r += AT(q1, n - 1, l);
            if (n <= ns - 3) r += AT(q2, n, l);
            if (1 <= n && n <= ns - 2) r -= 2.0 * AT(q2, n - 1, l);
            if (n >= 2) r += AT(q2, n - 2, l);
            AT(s, n, l) = AT(k, n, l) - r;
        }
    }
    if (pin_idx >= 0)
        for (int l = 0; l < d; ++l) AT(s, pin_idx, l) = pin_val[l];
}

/* _dual_objective (projection.py:126-166). */
static double dual_objective(const double* k, const double* q0, const double* q1,
                             const double* q2, int ns, int d, int pin_idx,
                             const double* pin_val, double a, double b, double* s) {
    dual_to_primal(k, q0, q1, q2, ns, d, pin_idx, pin_val, s);
    double obj = 0.0;
    for (int n = 0; n < ns; ++n) {
        if (n == pin_idx) continue;
        for (int l = 0; l < d; ++l) obj += 0.5 * AT(s, n, l) * AT(s, n, l);
    }
    for (int n = 0; n < ns; ++n)
        for (int l = 0; l < d; ++l) obj += fabs(AT(q0, n, l));
    for (int n = 0; n < ns - 1; ++n) {
        double nrm = 0.0;
        for (int l = 0; l < d; ++l) nrm += AT(q1, n, l) * AT(q1, n, l);
        obj += a * sqrt(nrm);
    }
    for (int n = 0; n < ns - 2; ++n) {
        double nrm = 0.0;
        for (int l = 0; l < d; ++l) nrm += AT(q2, n, l) * AT(q2, n, l);
        obj += b * sqrt(nrm);
    }
    if (pin_idx >= 0) {
        const int p = pin_idx;
        for (int l = 0; l < d; ++l) {
            obj -= AT(q0, p, l) * pin_val[l];
            if (p <= ns - 2) obj -= AT(q1, p, l) * pin_val[l];
            if (p >= 1) obj += AT(q1, p - 1, l) * pin_val[l];
            if (p <= ns - 3) obj += AT(q2, p, l) * pin_val[l];
            if (1 <= p && p <= ns - 2) obj -= 2.0 * AT(q2, p - 1, l) * pin_val[l];
            if (p >= 2) obj += AT(q2, p - 2, l) * pin_val[l];
        }
    }
    return obj;
}

static inline double clamp1(double z) {
    /* min(max(z, -1.0), 1.0) (projection.py:196) */
    double m = (z > -1.0) ? z : -1.0;
    return (m < 1.0) ? m : 1.0;
}

/* _project_shot (projection.py:169-284): dual FISTA with gradient restart.
 * work must hold 10*ns*d doubles.  trace may be NULL. */
void or_project_shot(const double* k, int ns, int d, double a, double b, int pin_idx,
                     const double* pin_val, int n_iter, double tau, int monotone,
                     double* out, double* trace, double* work) {
    const int n0 = ns * d, n1 = (ns - 1) * d, n2 = (ns - 2) * d;
    const int m1 = n1 > 0 ? n1 : 0, m2 = n2 > 0 ? n2 : 0;
    double* q0 = work;
    double* q1 = q0 + n0;
    double* q2 = q1 + m1;
    double* y0 = q2 + m2;
    double* y1 = y0 + n0;
    double* y2 = y1 + m1;
    double* z0 = y2 + m2;
    double* z1 = z0 + n0;
    double* z2 = z1 + m1;
    double* s = z2 + m2;
    memset(q0, 0, sizeof(double) * (size_t)(n0 + m1 + m2) * 2); /* q*, y* */
    double t = 1.0;
    double best = INFINITY;
    const double inv_tau = 1.0 / tau;

    for (int it = 0; it < n_iter; ++it) {
        dual_to_primal(k, y0, y1, y2, ns, d, pin_idx, pin_val, s);
        for (int n = 0; n < ns; ++n)
            for (int l = 0; l < d; ++l) {
                double z = AT(y0, n, l) * inv_tau + AT(s, n, l);
                double pz = clamp1(z);
                AT(z0, n, l) = tau * (z - pz);
            }
        for (int n = 0; n < ns - 1; ++n) {
            double nrm = 0.0;
            for (int l = 0; l < d; ++l) {
                double z = AT(y1, n, l) * inv_tau + (AT(s, n + 1, l) - AT(s, n, l));
                AT(z1, n, l) = z;
                nrm += z * z;
            }
            nrm = sqrt(nrm);
            double scale = (nrm <= a) ? 0.0 : 1.0 - a / nrm;
            for (int l = 0; l < d; ++l) AT(z1, n, l) = tau * AT(z1, n, l) * scale;
        }
        for (int n = 0; n < ns - 2; ++n) {
            double nrm = 0.0;
            for (int l = 0; l < d; ++l) {
                double z = AT(y2, n, l) * inv_tau +
                           (AT(s, n + 2, l) - 2.0 * AT(s, n + 1, l) + AT(s, n, l));
                AT(z2, n, l) = z;
                nrm += z * z;
            }
            nrm = sqrt(nrm);
            double scale = (nrm <= b) ? 0.0 : 1.0 - b / nrm;
            for (int l = 0; l < d; ++l) AT(z2, n, l) = tau * AT(z2, n, l) * scale;
        }

        int accept = 1;
        if (monotone) {
            double obj = dual_objective(k, z0, z1, z2, ns, d, pin_idx, pin_val, a, b, s);
            if (obj > best) accept = 0;
            else best = obj;
        }

        double g_dot = 0.0;
        for (int i = 0; i < n0; ++i) g_dot += (y0[i] - z0[i]) * (z0[i] - q0[i]);
        for (int i = 0; i < n1; ++i) g_dot += (y1[i] - z1[i]) * (z1[i] - q1[i]);
        for (int i = 0; i < n2; ++i) g_dot += (y2[i] - z2[i]) * (z2[i] - q2[i]);
        if (g_dot > 0.0) t = 1.0;
        double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));

        if (monotone) {
            double mom_z = t / t_next;
            double mom_q = (t - 1.0) / t_next;
#define MF(Y, Z, Q, N)                                                             \
    for (int i = 0; i < (N); ++i) {                                                \
        double nq = accept ? Z[i] : Q[i];                                          \
        Y[i] = nq + mom_z * (Z[i] - nq) + mom_q * (nq - Q[i]);                     \
        Q[i] = nq;                                                                 \
    }
            MF(y0, z0, q0, n0)
            MF(y1, z1, q1, n1)
            MF(y2, z2, q2, n2)
#undef MF
        } else {
            double mom = (t - 1.0) / t_next;
#define FF(Y, Z, Q, N)                                                             \
    for (int i = 0; i < (N); ++i) {                                                \
        Y[i] = Z[i] + mom * (Z[i] - Q[i]);                                         \
        Q[i] = Z[i];                                                               \
    }
            FF(y0, z0, q0, n0)
            FF(y1, z1, q1, n1)
            FF(y2, z2, q2, n2)
#undef FF
        }
        t = t_next;
        if (trace) trace[it] = dual_objective(k, q0, q1, q2, ns, d, pin_idx, pin_val, a, b, s);
    }
    dual_to_primal(k, q0, q1, q2, ns, d, pin_idx, pin_val, out);
}

/* _feasibility_polish (projection.py:287-373).  Returns the number of sweeps run. */
int or_polish(double* s, int ns, int d, double a, double b, int pin_idx,
              const double* pin_val, double tol, int max_sweeps) {
    const double omega = 1.8;
    int sweep = 0;
    while (sweep < max_sweeps) {
        ++sweep;
        double worst = 0.0;
        if (pin_idx >= 0)
            for (int l = 0; l < d; ++l) AT(s, pin_idx, l) = pin_val[l];
        for (int i = 0; i < ns * d; ++i) {
            double v = s[i];
            if (v > 1.0) {
                if (v - 1.0 > worst) worst = v - 1.0;
                s[i] = 1.0;
            } else if (v < -1.0) {
                if (-1.0 - v > worst) worst = -1.0 - v;
                s[i] = -1.0;
            }
        }
        for (int n = 0; n < ns - 1; ++n) {
            double nrm = 0.0;
            for (int l = 0; l < d; ++l) {
                double df = AT(s, n + 1, l) - AT(s, n, l);
                nrm += df * df;
            }
            nrm = sqrt(nrm);
            if (n == pin_idx || n + 1 == pin_idx) {
                const int free_n = (n == pin_idx) ? n + 1 : n;
                const double sign = (free_n == n + 1) ? 1.0 : -1.0;
                if (nrm > a) {
                    if (nrm - a > worst) worst = nrm - a;
                    double shrink = omega * (nrm - a) / nrm;
                    for (int l = 0; l < d; ++l) {
                        double df = AT(s, n + 1, l) - AT(s, n, l);
                        AT(s, free_n, l) -= sign * shrink * df;
                    }
                }
                continue;
            }
            if (nrm > a) {
                if (nrm - a > worst) worst = nrm - a;
                double shrink = omega * 0.5 * (nrm - a) / nrm;
                for (int l = 0; l < d; ++l) {
                    double df = AT(s, n + 1, l) - AT(s, n, l);
                    AT(s, n, l) += shrink * df;
                    AT(s, n + 1, l) -= shrink * df;
                }
            }
        }
        for (int n = 0; n < ns - 2; ++n) {
            double nrm = 0.0;
            for (int l = 0; l < d; ++l) {
                double w = AT(s, n, l) - 2.0 * AT(s, n + 1, l) + AT(s, n + 2, l);
                nrm += w * w;
            }
            nrm = sqrt(nrm);
            if (nrm > b) {
                if (nrm - b > worst) worst = nrm - b;
                double c0 = 1.0, c1 = -2.0, c2 = 1.0;
                if (pin_idx == n) c0 = 0.0;
                else if (pin_idx == n + 1) c1 = 0.0;
                else if (pin_idx == n + 2) c2 = 0.0;
                double denom = c0 * c0 + c1 * c1 + c2 * c2;
                if (denom > 0.0) {
                    double step = omega * (nrm - b) / (denom * nrm);
                    for (int l = 0; l < d; ++l) {
                        double w = AT(s, n, l) - 2.0 * AT(s, n + 1, l) + AT(s, n + 2, l);
                        AT(s, n, l) -= step * c0 * w;
                        AT(s, n + 1, l) -= step * c1 * w;
                        AT(s, n + 2, l) -= step * c2 * w;
                    }
                }
            }
        }
        if (worst <= tol) break;
    }
    return sweep;
}

/* _project_all (projection.py:376-382): FISTA then polish, shot by shot.
 * sweeps_out (nullable) receives the polish sweep count per shot. */
void or_project_all(const double* shots, int64_t n_shots, int ns, int d, double a,
                    double b, int pin_idx, const double* pin_val, int n_iter,
                    double tau, int monotone, double tol, int max_sweeps, double* out,
                    int32_t* sweeps_out, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel
    {
        double* work = (double*)malloc(sizeof(double) * (size_t)10 * ns * d + 64);
#pragma omp for schedule(dynamic, 1)
        for (int64_t c = 0; c < n_shots; ++c) {
            const size_t off = (size_t)c * ns * d;
            or_project_shot(shots + off, ns, d, a, b, pin_idx, pin_val, n_iter, tau,
                            monotone, out + off, NULL, work);
            int sw = or_polish(out + off, ns, d, a, b, pin_idx, pin_val, tol, max_sweeps);
            if (sweeps_out) sweeps_out[c] = sw;
        }
        free(work);
    }
}
#undef AT
