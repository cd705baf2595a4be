/* abi_demo.c -- a torch-free consumer of the C ABI (include/sparkling_b200.h).
 *
 * Reads fp64 inputs written by tests/test_gpu_abi_demo.py, runs
 *   1. spk_pack_positions + spk_direct_sums   (_treecode.direct_sums, _treecode.py:506-534)
 *   2. spk_project_all                          (_project_all, projection.py:376-382)
 * with plain cudaMalloc'd buffers on the default stream, and writes the outputs back.
 *
 *   usage: abi_demo <in.bin> <out.bin>
 *   in.bin:  int64 p, dims, n_shots, n_s, pin; f64 eps, a, b, tau, tol, pin_val[3];
 *            f64 pts[p*dims]; f64 shots[n_shots*n_s*dims]
 *   out.bin: f64 val[p], grad[p*dims], projected[n_shots*n_s*dims]; int32 sweeps[n_shots]
 * Build: gcc -O2 -I include examples/abi_demo.c -L paper_2108_02991_b200/_lib
 *        -lsparkling_b200 -L /usr/local/cuda/lib64 -lcudart -o abi_demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "sparkling_b200.h"

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
            return 2;                                                             \
        }                                                                         \
    } while (0)
#define SPK(x)                                                                    \
    do {                                                                          \
        if ((x) != SPK_OK) {                                                      \
            fprintf(stderr, "%s: %s\n", #x, spk_last_error());                    \
            return 3;                                                             \
        }                                                                         \
    } while (0)

static int read_all(FILE* f, void* dst, size_t n) { return fread(dst, 1, n, f) == n ? 0 : 1; }

int main(int argc, char** argv) {
    if (argc != 3) {
        fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
        return 1;
    }
    FILE* fi = fopen(argv[1], "rb");
    if (!fi) return 1;
    int64_t hdr[5];
    double par[8];
    if (read_all(fi, hdr, sizeof hdr) || read_all(fi, par, sizeof par)) return 1;
    const int64_t p = hdr[0], dims = hdr[1], n_shots = hdr[2], n_s = hdr[3], pin = hdr[4];
    const double eps = par[0], a = par[1], b = par[2], tau = par[3], tol = par[4];
    const size_t np = (size_t)p * dims, ns = (size_t)n_shots * n_s * dims;
    double* h_pts = malloc(np * 8);
    double* h_shots = malloc(ns * 8);
    if (read_all(fi, h_pts, np * 8) || read_all(fi, h_shots, ns * 8)) return 1;
    fclose(fi);

    /* 1. repulsion raw sums, all targets against all sources */
    double *d_pts, *d_val, *d_grad;
    void *d_pos4, *d_ws;
    CK(cudaMalloc((void**)&d_pts, np * 8));
    CK(cudaMalloc(&d_pos4, (size_t)p * 16));
    CK(cudaMalloc((void**)&d_val, (size_t)p * 8));
    CK(cudaMalloc((void**)&d_grad, np * 8));
    const size_t ws_nb = spk_nbody_workspace_bytes(p, 0, p);
    CK(cudaMalloc(&d_ws, ws_nb));
    CK(cudaMemcpy(d_pts, h_pts, np * 8, cudaMemcpyHostToDevice));
    SPK(spk_pack_positions(d_pts, p, (int)dims, d_pos4, NULL));
    SPK(spk_direct_sums(d_pos4, p, d_pos4, p, (int)dims, (float)(eps * eps), d_val, d_grad,
                        d_ws, ws_nb, NULL));

    /* 2. projection of every shot (no step), the reference's 50000-sweep cap */
    double *d_in, *d_out;
    int32_t* d_sweeps;
    void* d_pws;
    CK(cudaMalloc((void**)&d_in, ns * 8));
    CK(cudaMalloc((void**)&d_out, ns * 8));
    CK(cudaMalloc((void**)&d_sweeps, (size_t)n_shots * 4));
    const size_t pws_nb = spk_project_workspace_bytes(n_shots, (int)n_s, (int)dims, 0);
    CK(cudaMalloc(&d_pws, pws_nb));
    CK(cudaMemcpy(d_in, h_shots, ns * 8, cudaMemcpyHostToDevice));
    SPK(spk_project_all(d_in, NULL, 0.0, NULL, d_out, n_shots, (int)n_s, (int)dims, a, b,
                        (int)pin, par + 5, 100, tau, 0, tol, 50000, NULL, d_sweeps, NULL, NULL,
                        d_pws, pws_nb, NULL));
    CK(cudaDeviceSynchronize());

    double* h_val = malloc((size_t)p * 8);
    double* h_grad = malloc(np * 8);
    double* h_out = malloc(ns * 8);
    int32_t* h_sw = malloc((size_t)n_shots * 4);
    CK(cudaMemcpy(h_val, d_val, (size_t)p * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_grad, d_grad, np * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_out, d_out, ns * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_sw, d_sweeps, (size_t)n_shots * 4, cudaMemcpyDeviceToHost));
    FILE* fo = fopen(argv[2], "wb");
    if (!fo) return 1;
    fwrite(h_val, 8, (size_t)p, fo);
    fwrite(h_grad, 8, np, fo);
    fwrite(h_out, 8, ns, fo);
    fwrite(h_sw, 4, (size_t)n_shots, fo);
    fclose(fo);
    printf("abi_demo: ok (p=%lld, shots=%lld x %lld)\n", (long long)p, (long long)n_shots,
           (long long)n_s);
    return 0;
}
