// tree.cu -- GPU kernels of the treecode repulsion backend (RepulsionConfig(backend="tree")).
//
// The reference accelerates repulsion with a dual-tree Chebyshev black-box FMM on the
// CPU (/root/reference/pkg/src/vdtraj/repulsion.py:90-200, _treecode.py:77-471) and
// promises `tree_precision` relative error on the cost and the gradient l2 norm.  The
// B200 design keeps that contract with a scheme whose every hot loop is the N-body pair
// kernel of nbody.cu:
//
//  * sources are sorted along a Morton curve (CUB radix sort) and an octree is built over
//    the sorted keys (host, tree_host.cpp);
//  * a far source node is replaced by q^d proxy sources on its tight bounding box (tensor
//    Chebyshev points, weights = sum of the Lagrange basis over its particles: the
//    source-side interpolation of particle-cluster treecodes);
//  * targets are taken in Morton order in groups of <= TR_GROUP that follow the octree
//    (packed sibling subtrees, tree_host.cpp); each group gets a list of source segments
//    (near particles or far proxies) and one warp evaluates the weighted kernel sum over
//    the concatenated list with packed f32x2 FMA + MUFU.RSQ, staging the segments
//    through shared memory with cp.async double buffering.
//
// Deterministic: the tree, the lists and every reduction have a fixed order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>

#include "spk_common.cuh"

namespace spk {

constexpr int TR_THREADS = 128;            // 4 warps per CTA, one target group per warp
constexpr int TR_WARPS = TR_THREADS / 32;
constexpr int TR_GROUP = 64;               // targets per group (32 lanes x one f32x2 pair)
constexpr int TR_BATCH = 256;              // source records per warp and stage
constexpr int P2M_THREADS = 128;
constexpr int P2M_MAX_ORDER = 8;

// ---------------------------------------------------------------- Morton keys
__device__ __forceinline__ uint64_t spread3(uint32_t v) {  // 21 bits -> every 3rd bit
    uint64_t x = v & 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}
__device__ __forceinline__ uint64_t spread2(uint32_t v) {  // 31 bits -> every 2nd bit
    uint64_t x = v & 0x7fffffffULL;
    x = (x | x << 16) & 0x0000ffff0000ffffULL;
    x = (x | x << 8) & 0x00ff00ff00ff00ffULL;
    x = (x | x << 4) & 0x0f0f0f0f0f0f0f0fULL;
    x = (x | x << 2) & 0x3333333333333333ULL;
    x = (x | x << 1) & 0x5555555555555555ULL;
    return x;
}
__device__ __forceinline__ uint32_t quantize(float x, int bits) {
    const double u = ((double)x + 1.0) * 0.5 * (double)(1ULL << bits);
    long long q = (long long)floor(u);
    q = q < 0 ? 0 : q;
    const long long hi = (1LL << bits) - 1;
    return (uint32_t)(q > hi ? hi : q);
}

__global__ void keys_kernel(const float4* __restrict__ pos, long long n, int dims,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 r = pos[i];
    uint64_t k;
    if (dims == 3)
        k = (spread3(quantize(r.x, 21)) << 2) | (spread3(quantize(r.y, 21)) << 1) |
            spread3(quantize(r.z, 21));
    else
        k = (spread2(quantize(r.x, 31)) << 1) | spread2(quantize(r.y, 31));
    keys[i] = k;
    idx[i] = (int32_t)i;
}

// sorted records {x, y, z, w}: w = 1 (repulsion) or weights[perm[i]]
__global__ void gather_kernel(const float4* __restrict__ pos, const int32_t* __restrict__ perm,
                              long long n, const float* __restrict__ weights,
                              float4* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t j = perm[i];
    const float4 r = pos[j];
    out[i] = make_float4(r.x, r.y, r.z, weights ? weights[j] : 1.0f);
}

// ---------------------------------------------------------------- boxes
// Tight bounding box {min xyz, max xyz} of every record range (leaves and target groups).
__global__ void boxes_kernel(const float4* __restrict__ rec, const long long* __restrict__ begin,
                             const long long* __restrict__ end, int dims,
                             float* __restrict__ box, const int32_t* __restrict__ dst) {
    const long long r = blockIdx.x;
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (long long i = begin[r] + threadIdx.x; i < end[r]; i += blockDim.x) {
        const float4 p = rec[i];
        lo[0] = fminf(lo[0], p.x), hi[0] = fmaxf(hi[0], p.x);
        lo[1] = fminf(lo[1], p.y), hi[1] = fmaxf(hi[1], p.y);
        lo[2] = fminf(lo[2], p.z), hi[2] = fmaxf(hi[2], p.z);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    }
    __shared__ float s[32][6];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
        for (int a = 0; a < 3; ++a) s[w][a] = lo[a], s[w][3 + a] = hi[a];
    __syncthreads();
    if (threadIdx.x < 6) {
        const int c = threadIdx.x;
        float v = s[0][c];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            v = c < 3 ? fminf(v, s[k][c]) : fmaxf(v, s[k][c]);
        if (dims == 2 && (c == 2 || c == 5)) v = 0.0f;
        box[(dst ? (long long)dst[r] : r) * 6 + c] = v;
    }
}

// ---------------------------------------------------------------- P2M
// Chebyshev points of the first kind t_i = cos((2i+1) pi / 2q) (the reference's
// chebyshev_tables nodes, _treecode.py:20-44) and the Lagrange denominators.
struct ChebTable {
    float t[P2M_MAX_ORDER];
    float inv_den[P2M_MAX_ORDER];
};

__device__ __forceinline__ void lagrange(float u, int q, const ChebTable& T, float* L) {
    // L_k(u) = prod_{i != k} (u - t_i) / (t_k - t_i), via prefix / suffix products
    float diff[P2M_MAX_ORDER];
#pragma unroll
    for (int i = 0; i < P2M_MAX_ORDER; ++i) diff[i] = i < q ? u - T.t[i] : 1.0f;
    float pre = 1.0f;
    float prefix[P2M_MAX_ORDER];
#pragma unroll
    for (int i = 0; i < P2M_MAX_ORDER; ++i) {
        prefix[i] = pre;
        pre *= diff[i];
    }
    float suf = 1.0f;
#pragma unroll
    for (int i = P2M_MAX_ORDER - 1; i >= 0; --i) {
        if (i < q) L[i] = prefix[i] * suf * T.inv_den[i];
        suf *= diff[i];
    }
}

// One CTA per unit = (proxy slot, particle range); partial weights -> part[unit][m].
__global__ void __launch_bounds__(P2M_THREADS) p2m_kernel(
    const float4* __restrict__ rec, const int32_t* __restrict__ unit_slot,
    const long long* __restrict__ unit_begin, const long long* __restrict__ unit_end,
    const float* __restrict__ slot_box, int q, int dims, ChebTable T,
    double* __restrict__ part) {
    __shared__ float L[3][P2M_MAX_ORDER][P2M_THREADS];
    __shared__ float W[P2M_THREADS];
    const int tid = threadIdx.x;
    const long long u = blockIdx.x;
    const int slot = unit_slot[u];
    const float* bx = slot_box + (size_t)slot * 6;  // center xyz, half xyz
    const int m = dims == 3 ? q * q * q : q * q;
    constexpr int KMAX = (P2M_MAX_ORDER * P2M_MAX_ORDER * P2M_MAX_ORDER) / P2M_THREADS;
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.0;
    for (long long c = unit_begin[u]; c < unit_end[u]; c += P2M_THREADS) {
        const long long j = c + tid;
        float l[3][P2M_MAX_ORDER] = {};
        float w = 0.0f;
        if (j < unit_end[u]) {
            const float4 p = rec[j];
            w = p.w;
            lagrange((p.x - bx[0]) / bx[3], q, T, l[0]);
            lagrange((p.y - bx[1]) / bx[4], q, T, l[1]);
            if (dims == 3) lagrange((p.z - bx[2]) / bx[5], q, T, l[2]);
        }
        for (int i = 0; i < q; ++i) {
            L[0][i][tid] = l[0][i];
            L[1][i][tid] = l[1][i];
            L[2][i][tid] = dims == 3 ? l[2][i] : 1.0f;
        }
        W[tid] = w;
        __syncthreads();
        const int cnt = (int)min((long long)P2M_THREADS, unit_end[u] - c);
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) {
            const int k = tid + kk * P2M_THREADS;
            if (k < m) {
                int kx, ky, kz;
                if (dims == 3) {
                    kx = k / (q * q), ky = (k / q) % q, kz = k % q;
                } else {
                    kx = k / q, ky = k % q, kz = 0;
                }
                const float* lx = L[0][kx];
                const float* ly = L[1][ky];
                const float* lz = L[2][dims == 3 ? kz : 0];
                float s = 0.0f;
                for (int jj = 0; jj < cnt; ++jj) s = fmaf(W[jj] * lx[jj], ly[jj] * lz[jj], s);
                acc[kk] += (double)s;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk) {
        const int k = tid + kk * P2M_THREADS;
        if (k < m) part[(size_t)u * m + k] = acc[kk];
    }
}

// Sum the units of every slot in order; write the proxy records {x, y, z, W}.
__global__ void p2m_final_kernel(const double* __restrict__ part,
                                 const long long* __restrict__ slot_unit_off,
                                 const float* __restrict__ slot_box, int q, int dims,
                                 ChebTable T, float4* __restrict__ proxies) {
    const int slot = blockIdx.x;
    const int m = dims == 3 ? q * q * q : q * q;
    const float* bx = slot_box + (size_t)slot * 6;
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        double s = 0.0;
        for (long long u = slot_unit_off[slot]; u < slot_unit_off[slot + 1]; ++u)
            s += part[(size_t)u * m + k];
        int kx, ky, kz;
        if (dims == 3) {
            kx = k / (q * q), ky = (k / q) % q, kz = k % q;
        } else {
            kx = k / q, ky = k % q, kz = 0;
        }
        const float x = fmaf(bx[3], T.t[kx], bx[0]);
        const float y = fmaf(bx[4], T.t[ky], bx[1]);
        const float z = dims == 3 ? fmaf(bx[5], T.t[kz], bx[2]) : 0.0f;
        proxies[(size_t)slot * m + k] = make_float4(x, y, z, (float)s);
    }
}


// ---------------------------------------------------------------- device octree build
// Level-synchronous construction over the sorted Morton keys, identical to the host
// builder (tree_host.cpp spk_tree_host_build): BFS node order, children contiguous and in
// child-digit order, a node splits when it holds more than leaf_cap particles and is above
// the finest level.  One thread per node of the current level finds its children by
// binary search; a scan of the child counts places the next level.
__device__ __forceinline__ long long lower_bound_u64(const uint64_t* __restrict__ keys,
                                                     long long lo, long long hi, uint64_t v) {
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (keys[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void split_kernel(const uint64_t* __restrict__ keys, const long long* __restrict__ nbeg,
                             const long long* __restrict__ nend, long long lv_b, long long lv_e,
                             int level, int dims, int bits, long long cap, int min_level,
                             int32_t* __restrict__ nchild, long long* __restrict__ child) {
    const long long v = lv_b + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= lv_e) return;
    const long long b = nbeg[v], e = nend[v];
    const long long w = v - lv_b;
    // split when over capacity, or (min_level) when the cell is still coarse
    const bool split = e - b > cap || (level < min_level && e - b > 1);
    if (!split || level >= bits) {
        nchild[w] = 0;
        return;
    }
    const int nc = 1 << dims;
    const int shift = dims * (bits - level - 1);
    const uint64_t prefix = keys[b] >> (shift + dims);
    long long lo = b;
    int cnt = 0;
    for (int c = 0; c < nc; ++c) {
        long long hi = e;
        if (c + 1 < nc) hi = lower_bound_u64(keys, lo, e, ((prefix << dims) | (uint64_t)(c + 1)) << shift);
        if (hi > lo) {
            child[w * 16 + 2 * cnt] = lo;
            child[w * 16 + 2 * cnt + 1] = hi;
            ++cnt;
        }
        lo = hi;
    }
    nchild[w] = cnt;
}

__global__ void link_kernel(const int32_t* __restrict__ nchild, const int32_t* __restrict__ off,
                            const long long* __restrict__ child, long long lv_b, long long lv_e,
                            long long* __restrict__ nbeg, long long* __restrict__ nend,
                            int32_t* __restrict__ first_child, int32_t* __restrict__ n_child) {
    const long long v = lv_b + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= lv_e) return;
    const long long w = v - lv_b;
    const int nc = nchild[w];
    n_child[v] = nc;
    first_child[v] = nc ? (int32_t)(lv_e + off[w]) : -1;
    for (int k = 0; k < nc; ++k) {
        const long long u = lv_e + off[w] + k;
        nbeg[u] = child[w * 16 + 2 * k];
        nend[u] = child[w * 16 + 2 * k + 1];
    }
}

__global__ void root_kernel(long long n, long long* nbeg, long long* nend) {
    nbeg[0] = 0;
    nend[0] = n;
}

__global__ void leaf_flag_kernel(const int32_t* __restrict__ n_child, long long n_nodes,
                                 int32_t* __restrict__ flag) {
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v < n_nodes) flag[v] = n_child[v] == 0;
}

__global__ void leaf_write_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                                  long long n_nodes, int32_t* __restrict__ leaf_node) {
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v < n_nodes && flag[v]) leaf_node[pos[v]] = (int32_t)v;
}

// Target groups (tree_host.cpp spk_tree_host_groups): under every internal node, maximal
// runs of consecutive leaf children with <= cap particles are packed greedily into groups
// of <= cap; oversized leaves are cut into chunks; a root leaf with <= cap particles is
// one group.  Pass 0 counts per node, pass 1 writes; the groups are
// then sorted by their first particle.
template <int PASS>
__global__ void groups_kernel(const long long* __restrict__ nbeg, const long long* __restrict__ nend,
                              const int32_t* __restrict__ first_child,
                              const int32_t* __restrict__ n_child, long long n_nodes,
                              long long cap, const uint8_t* __restrict__ cut,
                              long long* __restrict__ cnt_out,
                              const long long* __restrict__ off, long long* __restrict__ gb,
                              long long* __restrict__ ge) {
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n_nodes) return;
    const long long b = nbeg[v], e = nend[v];
    long long k = 0;
    const long long o = PASS ? off[v] : 0;
    auto emit = [&](long long x, long long y) {
        if (PASS) {
            gb[o + k] = x;
            ge[o + k] = y;
        }
        ++k;
    };
    if (n_child[v] == 0) {
        if (e - b > cap) {
            for (long long x = b; x < e; x += cap) emit(x, min(e, x + cap));
        } else if (v == 0) {
            emit(b, e);
        }
    } else {
        // pack runs of consecutive small LEAF children; other children group themselves
        long long cb = -1, ce = -1;
        for (int c = 0; c < n_child[v]; ++c) {
            const long long u = first_child[v] + c;
            const long long ub = nbeg[u], ue = nend[u];
            if (ue - ub > cap || n_child[u] != 0) {
                if (cb >= 0) emit(cb, ce);
                cb = -1;
                continue;
            }
            // `cut` marks the first particles of enclosing groups (far-level parents):
            // a group never straddles one
            if (cb >= 0 && ue - cb <= cap && !(cut && cut[ub])) {
                ce = ue;
            } else {
                if (cb >= 0) emit(cb, ce);
                cb = ub;
                ce = ue;
            }
        }
        if (cb >= 0) emit(cb, ce);
    }
    if (!PASS) cnt_out[v] = k;
}

// ---------------------------------------------------------------- device plan
// Node boxes bottom-up: leaves reduce their particles (boxes_kernel with dst = node id),
// internal nodes of one BFS level take the union of their children's boxes.
__global__ void level_boxes_kernel(const int32_t* __restrict__ fchild,
                                   const int32_t* __restrict__ nchild, long long lv_begin,
                                   long long lv_end, float* __restrict__ box) {
    const long long v = lv_begin + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= lv_end || nchild[v] == 0) return;
    float o[6] = {FLT_MAX, FLT_MAX, FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int c = 0; c < nchild[v]; ++c) {
        const float* cb = box + (size_t)(fchild[v] + c) * 6;
        for (int a = 0; a < 3; ++a) {
            o[a] = fminf(o[a], cb[a]);
            o[3 + a] = fmaxf(o[3 + a], cb[3 + a]);
        }
    }
    for (int k = 0; k < 6; ++k) box[(size_t)v * 6 + k] = o[k];
}

// Center and half-diagonal of a {min, max} box with explicit roundings: identical to the
// host planner (tree_host.cpp make_box), so both produce the same interaction lists.
struct CR {
    float c[3], h[3], r;
};
__device__ __forceinline__ CR center_radius(const float* lohi, int dims) {
    CR b;
    float r2 = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b.c[a] = __fmul_rn(0.5f, __fadd_rn(lohi[a], lohi[3 + a]));
        b.h[a] = a < dims ? __fmul_rn(0.5f, __fsub_rn(lohi[3 + a], lohi[a])) : 0.0f;
        r2 = __fadd_rn(r2, __fmul_rn(b.h[a], b.h[a]));
    }
    b.r = __fsqrt_rn(r2);
    return b;
}

struct TravParams {
    const long long* nbeg;
    const long long* nend;
    const int32_t* fchild;
    const int32_t* nchild;
    const float* nbox;  // [n_nodes][6]
    const float* gbox;  // [n_groups][6]
    long long n_groups;
    int dims;
    float theta;
    int m;
    long long n_src;
    int32_t* is_proxy;         // pass 0 out (zeroed by the caller)
    long long* seg_cnt;        // pass 0 out [n_groups]
    const int32_t* slot_of;    // pass 1 in
    const long long* seg_off;  // pass 1 in
    long long* seg_start;      // pass 1 out
    int32_t* seg_count;        // pass 1 out
    const float* pbox;         // optional far-level parents: [n_parents][6]
    const int32_t* gparent;    // group -> parent
    int far_only;              // parents' own walk: emit far nodes only (no near leaves)
    unsigned long long* overflow;  // pass 0: groups whose walk overflowed the stack
    long long* sub_cnt;        // sub-walks, pass 0 out [n_groups * TR_FRONT]
    const long long* sub_off;  // sub-walks, pass 1 in [n_groups * TR_FRONT + 1]
};
// Sub-walks of the plain traversal: every group's walk is split at the octree's second
// level -- one thread per (group, frontier node), TR_FRONT = 8 x 8 (3D) / 4 x 4 (2D)
// frontier slots -- instead of one thread walking the whole tree.  The outputs
// concatenated in frontier order are the serial walk's with contiguous particle ranges
// merged only within a frontier subtree (the host planner follows the same rule).
constexpr int TR_FRONT = 64;
static_assert(TR_FRONT == SPK_TREE_FRONT, "sparkling_b200.h SPK_TREE_FRONT");
// Stack bound: a depth-first walk holds at most (children - 1) pending siblings per level
// plus the current node.  Keys have 21 bits per axis in 3D (21 levels of 8 children) and
// 31 in 2D (31 levels of 4 children).
constexpr int TR_STACK = 224;
static_assert(TR_STACK >= 21 * 7 + 1 && TR_STACK >= 31 * 3 + 1,
              "traversal stack too small for the Morton key depth");

// One thread per target group walks the source octree (dual_traverse's opening test,
// _treecode.py:173-244, applied group-to-node).  Pass 0 counts segments and flags proxy
// nodes, pass 1 writes them.  Contiguous particle ranges merge; proxies do not.
template <int PASS>
__global__ void __launch_bounds__(128) traverse_kernel(const TravParams P) {
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g >= P.n_groups) return;
    const CR tb = center_radius(P.gbox + g * 6, P.dims);
    const float th2 = __fmul_rn(P.theta, P.theta);
    CR pb{};
    if (P.pbox) pb = center_radius(P.pbox + (size_t)P.gparent[g] * 6, P.dims);
    int32_t stk[TR_STACK];
    int sp = 0;
    stk[sp++] = 0;
    long long pend_start = 0, pend_cnt = 0, n_out = 0;
    bool pend_direct = false;
    const long long o = PASS ? P.seg_off[g] : 0;
    auto flush = [&]() {
        if (pend_cnt > 0) {
            if (PASS) {
                P.seg_start[o + n_out] = pend_start;
                P.seg_count[o + n_out] = (int32_t)pend_cnt;
            }
            ++n_out;
            pend_cnt = 0;
        }
    };
    // Far level: stack entries carry bit 30 once inside a subtree in which no node can be
    // far from the parent ("strongly near": r_P >= theta (|c_P - c_u| + r_u)).
    constexpr int32_t FREE = 1 << 30;
    while (sp > 0) {
        const int32_t ent = stk[--sp];
        const int32_t v = ent & (FREE - 1);
        bool free_sub = (ent & FREE) != 0;
        const CR sb = center_radius(P.nbox + (size_t)v * 6, P.dims);
        float d2 = 0.0f;
        for (int a = 0; a < P.dims; ++a) {
            const float d = __fsub_rn(tb.c[a], sb.c[a]);
            d2 = __fadd_rn(d2, __fmul_rn(d, d));
        }
        if (P.pbox && !free_sub) {
            // nodes far from the group's parent are the far level's (interpolated) share:
            // skip them with their subtrees, exactly where the parent's walk stopped
            float pd2 = 0.0f;
            for (int a = 0; a < P.dims; ++a) {
                const float d = __fsub_rn(pb.c[a], sb.c[a]);
                pd2 = __fadd_rn(pd2, __fmul_rn(d, d));
            }
            const float plhs = __fadd_rn(pb.r, sb.r);
            if (__fmul_rn(plhs, plhs) < __fmul_rn(th2, pd2)) continue;
            // below a node that is not strongly near, descendants may still be parent-far:
            // descend without the group's own opening test (leaves are the group's)
            free_sub = pb.r >= __fmul_rn(P.theta, __fadd_rn(__fsqrt_rn(pd2), sb.r));
            if (!free_sub && P.nchild[v] != 0) {
                const int nc = P.nchild[v];
                if (sp + nc > TR_STACK) {  // cannot happen within the key depth (above)
                    if (PASS == 0) atomicAdd(P.overflow, 1ULL);
                    continue;
                }
                for (int c = nc - 1; c >= 0; --c) stk[sp++] = P.fchild[v] + c;
                continue;
            }
        }
        const float lhs = __fadd_rn(tb.r, sb.r);
        const bool far = __fmul_rn(lhs, lhs) < __fmul_rn(th2, d2);
        const long long b = P.nbeg[v], e = P.nend[v];
        if (far && e - b > P.m) {
            flush();
            if (PASS == 0) P.is_proxy[v] = 1;
            else pend_start = P.n_src + (long long)P.slot_of[v] * P.m;
            pend_cnt = P.m;
            pend_direct = false;
            flush();
        } else if (far || P.nchild[v] == 0) {
            if (!far && P.far_only) continue;
            if (pend_cnt > 0 && pend_direct && pend_start + pend_cnt == b &&
                pend_cnt + (e - b) < (1LL << 30)) {
                pend_cnt += e - b;
            } else {
                flush();
                pend_start = b;
                pend_cnt = e - b;
                pend_direct = true;
            }
        } else {
            const int nc = P.nchild[v];
            if (sp + nc > TR_STACK) {  // cannot happen within the key depth (above)
                if (PASS == 0) atomicAdd(P.overflow, 1ULL);
                continue;
            }
            const int32_t flag = free_sub ? FREE : 0;
            for (int c = nc - 1; c >= 0; --c) stk[sp++] = (P.fchild[v] + c) | flag;
        }
    }
    flush();
    if (PASS == 0) P.seg_cnt[g] = n_out;
}

template <int PASS>
__global__ void __launch_bounds__(128) traverse_sub_kernel(const TravParams P, int front,
                                                           int fan) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= P.n_groups * front) return;
    const long long g = idx / front;
    const int f = (int)(idx - g * front);
    const int c1 = f / fan, c2 = f - (f / fan) * fan;
    long long pend_start = 0, pend_cnt = 0, n_out = 0;
    bool pend_direct = false;
    const long long o = PASS ? P.sub_off[idx] : 0;
    auto flush = [&]() {
        if (pend_cnt > 0) {
            if (PASS) {
                P.seg_start[o + n_out] = pend_start;
                P.seg_count[o + n_out] = (int32_t)pend_cnt;
            }
            ++n_out;
            pend_cnt = 0;
        }
    };
    auto done = [&]() {
        flush();
        if (PASS == 0) P.sub_cnt[idx] = n_out;
    };
    // this slot's frontier node (depth 2, or a leaf above it) and its ancestors, in DFS
    // order; slots past a node's child count are empty
    int anc[2];
    bool first[2];
    int n_anc = 0, start;
    if (P.nchild[0] == 0) {
        if (f != 0) return done();
        start = 0;
    } else {
        if (c1 >= P.nchild[0]) return done();
        const int n1 = P.fchild[0] + c1;
        anc[n_anc] = 0;
        first[n_anc++] = f == 0;
        if (P.nchild[n1] == 0) {
            if (c2 != 0) return done();
            start = n1;
        } else {
            if (c2 >= P.nchild[n1]) return done();
            anc[n_anc] = n1;
            first[n_anc++] = c2 == 0;
            start = P.fchild[n1] + c2;
        }
    }
    const CR tb = center_radius(P.gbox + g * 6, P.dims);
    const float th2 = __fmul_rn(P.theta, P.theta);
    auto is_far = [&](int v) {
        const CR sb = center_radius(P.nbox + (size_t)v * 6, P.dims);
        float d2 = 0.0f;
        for (int a = 0; a < P.dims; ++a) {
            const float d = __fsub_rn(tb.c[a], sb.c[a]);
            d2 = __fadd_rn(d2, __fmul_rn(d, d));
        }
        const float lhs = __fadd_rn(tb.r, sb.r);
        return __fmul_rn(lhs, lhs) < __fmul_rn(th2, d2);
    };
    auto emit = [&](int v, bool far) {
        const long long b = P.nbeg[v], e = P.nend[v];
        if (far && e - b > P.m) {
            flush();
            if (PASS == 0) P.is_proxy[v] = 1;
            else pend_start = P.n_src + (long long)P.slot_of[v] * P.m;
            pend_cnt = P.m;
            pend_direct = false;
            flush();
        } else {
            if (!far && P.far_only) return;
            if (pend_cnt > 0 && pend_direct && pend_start + pend_cnt == b &&
                pend_cnt + (e - b) < (1LL << 30)) {
                pend_cnt += e - b;
            } else {
                flush();
                pend_start = b;
                pend_cnt = e - b;
                pend_direct = true;
            }
        }
    };
    // a far ancestor ends the walk there: the ancestor's first frontier slot emits it
    for (int k = 0; k < n_anc; ++k) {
        if (is_far(anc[k])) {
            if (first[k]) emit(anc[k], true);
            return done();
        }
    }
    int32_t stk[TR_STACK];
    int sp = 0;
    stk[sp++] = start;
    while (sp > 0) {
        const int32_t v = stk[--sp];
        const bool far = is_far(v);
        if (far || P.nchild[v] == 0) {
            emit(v, far);
        } else {
            const int nc = P.nchild[v];
            if (sp + nc > TR_STACK) {  // cannot happen within the key depth
                if (PASS == 0) atomicAdd(P.overflow, 1ULL);
                continue;
            }
            for (int c = nc - 1; c >= 0; --c) stk[sp++] = P.fchild[v] + c;
        }
    }
    done();
}

// Group offsets from the sub-walk offsets: seg_off[g] = sub_off[g * front].
__global__ void group_offsets_kernel(const long long* __restrict__ sub_off, long long n_groups,
                                     int front, long long* __restrict__ seg_off) {
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g <= n_groups) seg_off[g] = sub_off[g * front];
}

constexpr long long P2M_UNIT = 4096;  // particles per P2M unit (tree_host.cpp P2M_UNIT)

// Proxy slots in node order: slot box (degenerate axes inflated like the host planner)
// and the number of P2M units of each slot.
__global__ void slots_kernel(const long long* __restrict__ nbeg, const long long* __restrict__ nend,
                             const float* __restrict__ nbox, const int32_t* __restrict__ is_proxy,
                             const int32_t* __restrict__ slot_of, long long n_nodes, int dims,
                             int32_t* __restrict__ slot_node, float* __restrict__ slot_box,
                             long long* __restrict__ units_per_slot) {
    const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (v >= n_nodes || !is_proxy[v]) return;
    const int s = slot_of[v];
    slot_node[s] = (int32_t)v;
    const CR b = center_radius(nbox + (size_t)v * 6, dims);
    float hmax = 0.0f;
    for (int a = 0; a < dims; ++a) hmax = fmaxf(hmax, b.h[a]);
    for (int a = 0; a < 3; ++a) {
        slot_box[(size_t)s * 6 + a] = b.c[a];
        slot_box[(size_t)s * 6 + 3 + a] =
            a < dims ? fmaxf(b.h[a], __fadd_rn(__fmul_rn(1e-6f, hmax), 1e-30f)) : 1.0f;
    }
    units_per_slot[s] = (nend[v] - nbeg[v] + P2M_UNIT - 1) / P2M_UNIT;
}

__global__ void units_kernel(const long long* __restrict__ nbeg, const long long* __restrict__ nend,
                             const int32_t* __restrict__ slot_node,
                             const long long* __restrict__ slot_unit_off, long long n_slots,
                             int32_t* __restrict__ unit_slot, long long* __restrict__ unit_begin,
                             long long* __restrict__ unit_end) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    const int32_t v = slot_node[s];
    long long u = slot_unit_off[s];
    for (long long lo = nbeg[v]; lo < nend[v]; lo += P2M_UNIT, ++u) {
        unit_slot[u] = (int32_t)s;
        unit_begin[u] = lo;
        unit_end[u] = min(nend[v], lo + P2M_UNIT);
    }
}

__global__ void totals_kernel(const long long* __restrict__ seg_off, long long n_groups,
                              const int32_t* __restrict__ slot_of,
                              const int32_t* __restrict__ is_proxy,
                              const long long* __restrict__ slot_unit_off, long long n_nodes,
                              long long* __restrict__ totals) {
    totals[0] = seg_off[n_groups];
    totals[1] = (long long)slot_of[n_nodes - 1] + is_proxy[n_nodes - 1];
    totals[2] = slot_unit_off[n_nodes];  // units_per_slot is zero past the last slot
    // totals[3]: stack overflows counted by the traversal (the caller fails on nonzero)
}


// ---------------------------------------------------------------- far level (P2L / L2P)
// Far-level parents (target groups of <= 512 particles) evaluate their far list at the
// q^d tensor Chebyshev points of their box (P2L: an ordinary eval over those points) and
// every target interpolates value and gradient from them (L2P) -- the target-side
// interpolation of the reference's black-box FMM (m2l + l2p, _treecode.py:330-426).
__global__ void cheb_targets_kernel(const float* __restrict__ pbox, long long n_par, int q,
                                    int dims, ChebTable T, float4* __restrict__ pts,
                                    float* __restrict__ pcb) {
    const long long p = blockIdx.x;
    const CR b = center_radius(pbox + (size_t)p * 6, dims);
    float h[3];
    float hmax = 0.0f;
    for (int a = 0; a < dims; ++a) hmax = fmaxf(hmax, b.h[a]);
    for (int a = 0; a < 3; ++a)
        h[a] = a < dims ? fmaxf(b.h[a], __fadd_rn(__fmul_rn(1e-6f, hmax), 1e-30f)) : 1.0f;
    if (threadIdx.x < 6) pcb[p * 6 + threadIdx.x] = threadIdx.x < 3 ? b.c[threadIdx.x] : h[threadIdx.x - 3];
    const int m = dims == 3 ? q * q * q : q * q;
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        int kx, ky, kz;
        if (dims == 3) {
            kx = k / (q * q), ky = (k / q) % q, kz = k % q;
        } else {
            kx = k / q, ky = k % q, kz = 0;
        }
        pts[p * m + k] = make_float4(fmaf(h[0], T.t[kx], b.c[0]), fmaf(h[1], T.t[ky], b.c[1]),
                                     dims == 3 ? fmaf(h[2], T.t[kz], b.c[2]) : 0.0f, 0.0f);
    }
}

__global__ void parent_ids_kernel(const long long* __restrict__ pb, const long long* __restrict__ pe,
                                  long long n_par, int32_t* __restrict__ pid) {
    const long long p = blockIdx.x;
    for (long long i = pb[p] + threadIdx.x; i < pe[p]; i += blockDim.x) pid[i] = (int32_t)p;
}

template <int D>
__global__ void l2p_kernel(const float4* __restrict__ tgt, const int32_t* __restrict__ perm,
                           long long n_t, const int32_t* __restrict__ pid,
                           const float* __restrict__ pcb, const double* __restrict__ pval,
                           const double* __restrict__ pgrad, int q, ChebTable T,
                           double* __restrict__ val, double* __restrict__ grad) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_t) return;
    const float4 x = tgt[i];
    const long long p = pid[i];
    const float* bx = pcb + p * 6;
    float l[3][P2M_MAX_ORDER] = {};
    lagrange((x.x - bx[0]) / bx[3], q, T, l[0]);
    lagrange((x.y - bx[1]) / bx[4], q, T, l[1]);
    if (D == 3) lagrange((x.z - bx[2]) / bx[5], q, T, l[2]);
    const int m = D == 3 ? q * q * q : q * q;
    const double* pv = pval + p * m;
    const double* pg = pgrad + p * m * D;
    double v = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
    for (int k = 0; k < m; ++k) {
        int kx, ky, kz;
        if (D == 3) {
            kx = k / (q * q), ky = (k / q) % q, kz = k % q;
        } else {
            kx = k / q, ky = k % q, kz = 0;
        }
        const double w = (double)l[0][kx] * l[1][ky] * (D == 3 ? l[2][kz] : 1.0f);
        v += w * pv[k];
        g0 += w * pg[k * D];
        g1 += w * pg[k * D + 1];
        if (D == 3) g2 += w * pg[k * D + 2];
    }
    const long long o = perm[i];
    val[o] += v;
    grad[o * D] += g0;
    grad[o * D + 1] += g1;
    if (D == 3) grad[o * D + 2] += g2;
}

// ---------------------------------------------------------------- evaluation
__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float2 bcast(float v) { return make_float2(v, v); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct EvalParams {
    const float4* tgt;       // sorted targets
    const int32_t* tgt_perm; // sorted -> original target index
    const long long* grp_begin;  // target group g = sorted targets [begin, end), <= TR_GROUP
    const long long* grp_end;
    const float4* src;       // [sorted sources | proxies], {x, y, z, w}
    const long long* seg_off;   // [n_lists + 1]
    const int32_t* grp_list;    // optional group -> list (several groups share a list)
    const long long* seg_start; // record offset into src
    const int32_t* seg_count;
    float eps2;
    double* val;
    double* grad;
};

// Cursor over the concatenated segment list of one group (uniform across the warp).  The
// segment descriptors are fetched 32 at a time (lane i holds descriptor base + i) so the
// staging loop does not wait on one dependent global load per segment.
struct SegCursor {
    long long s, s_end;
    int off;
    long long base;  // first descriptor held in the lane window
    long long w_start;
    int w_cnt;
};

__device__ __forceinline__ void load_window(SegCursor& c, const EvalParams& P, int lane) {
    c.base = c.s;
    const long long d = c.s + lane;
    c.w_start = d < c.s_end ? P.seg_start[d] : 0;
    c.w_cnt = d < c.s_end ? P.seg_count[d] : 0;
}

// The warp stages the next TR_BATCH records of its concatenated segment list.
__device__ __forceinline__ int fill_batch(float4* buf, SegCursor& c, const EvalParams& P,
                                          int lane) {
    int filled = 0;
    while (filled < TR_BATCH && c.s < c.s_end) {
        if (c.s - c.base >= 32) load_window(c, P, lane);
        const int k = (int)(c.s - c.base);
        const int cnt = __shfl_sync(0xffffffffu, c.w_cnt, k);
        const long long start = __shfl_sync(0xffffffffu, c.w_start, k);
        const int take = min(TR_BATCH - filled, cnt - c.off);
        const float4* g = P.src + start + c.off;
        for (int i = lane; i < take; i += 32) cp_async16(buf + filled + i, g + i);
        filled += take;
        c.off += take;
        if (c.off == cnt) {
            ++c.s;
            c.off = 0;
        }
    }
    cp_async_commit();
    return filled;
}

template <int D, bool G>
__device__ __forceinline__ void pair_step(const float4 s, float2 X, float2 Y, float2 Z, float2 e2,
                                          float2& av, float2& ax, float2& ay, float2& az) {
    const float2 dx = __fadd2_rn(X, bcast(-s.x));
    const float2 dy = __fadd2_rn(Y, bcast(-s.y));
    float2 r2 = __ffma2_rn(dx, dx, e2);
    r2 = __ffma2_rn(dy, dy, r2);
    float2 dz;
    if (D == 3) {
        dz = __fadd2_rn(Z, bcast(-s.z));
        r2 = __ffma2_rn(dz, dz, r2);
    }
    float2 inv;
    inv.x = rsqrt_approx(r2.x);
    inv.y = rsqrt_approx(r2.y);
    if (G) {
        inv.x = r2.x >= FLT_MIN ? inv.x : 0.0f;  // rsqrt.approx.ftz flushes subnormal r2
        inv.y = r2.y >= FLT_MIN ? inv.y : 0.0f;
    }
    const float2 wi = __fmul2_rn(inv, bcast(s.w));
    av = __ffma2_rn(r2, wi, av);  // w h = w r2 / h
    ax = __ffma2_rn(dx, wi, ax);
    ay = __ffma2_rn(dy, wi, ay);
    if (D == 3) az = __ffma2_rn(dz, wi, az);
}

// Two accumulator sets (even / odd records) so that consecutive sources do not serialise
// on the accumulator FFMA2 latency at the low occupancy of this kernel.
template <int D, bool G>
__device__ __forceinline__ void eval_batch(const float4* __restrict__ buf, int cnt, float2 X,
                                           float2 Y, float2 Z, float2 e2, float2& av,
                                           float2& ax, float2& ay, float2& az) {
    float2 bv = bcast(0.f), bx = bcast(0.f), by = bcast(0.f), bz = bcast(0.f);
    int j = 0;
#pragma unroll 2
    for (; j + 1 < cnt; j += 2) {
        pair_step<D, G>(buf[j], X, Y, Z, e2, av, ax, ay, az);
        pair_step<D, G>(buf[j + 1], X, Y, Z, e2, bv, bx, by, bz);
    }
    if (j < cnt) pair_step<D, G>(buf[j], X, Y, Z, e2, av, ax, ay, az);
    av = __fadd2_rn(av, bv);
    ax = __fadd2_rn(ax, bx);
    ay = __fadd2_rn(ay, by);
    if (D == 3) az = __fadd2_rn(az, bz);
}

// One warp per target group (<= 64 targets, two per lane as one f32x2 pair): small
// groups keep the near field small (near pairs per target grow with the group's
// volume), and the warp walks its own segment list, double-buffered with cp.async.
template <int D, bool G>
__global__ void __launch_bounds__(TR_THREADS, 4) tree_eval_kernel(const EvalParams P,
                                                                  long long n_groups) {
    __shared__ __align__(16) float4 buf[TR_WARPS][2][TR_BATCH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long g = (long long)blockIdx.x * TR_WARPS + warp;
    if (g >= n_groups) return;
    const long long gb = P.grp_begin[g], ge = P.grp_end[g];
    const long long i0 = gb + lane, i1 = i0 + 32;
    const float4 a = P.tgt[min(i0, ge - 1)];
    const float4 b = P.tgt[min(i1, ge - 1)];
    const float2 X = make_float2(a.x, b.x), Y = make_float2(a.y, b.y),
                 Z = make_float2(a.z, b.z);
    const float2 e2 = bcast(P.eps2);
    double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};

    const long long lg = P.grp_list ? (long long)P.grp_list[g] : g;
    SegCursor c{P.seg_off[lg], P.seg_off[lg + 1], 0, 0, 0, 0};
    load_window(c, P, lane);
    int cnt = fill_batch(buf[warp][0], c, P, lane);
    int stage = 0;
    while (cnt > 0) {
        const int next = fill_batch(buf[warp][stage ^ 1], c, P, lane);
        cp_async_wait<1>();
        __syncwarp();
        float2 av = bcast(0.f), ax = bcast(0.f), ay = bcast(0.f), az = bcast(0.f);
        eval_batch<D, G>(buf[warp][stage], cnt, X, Y, Z, e2, av, ax, ay, az);
        acc[0][0] += av.x, acc[1][0] += av.y;
        acc[0][1] += ax.x, acc[1][1] += ax.y;
        acc[0][2] += ay.x, acc[1][2] += ay.y;
        if (D == 3) acc[0][3] += az.x, acc[1][3] += az.y;
        __syncwarp();
        cnt = next;
        stage ^= 1;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const long long i = t == 0 ? i0 : i1;
        if (i < ge) {
            const long long o = P.tgt_perm[i];
            if (P.val) P.val[o] = acc[t][0];
            if (P.grad) {
                P.grad[o * D] = acc[t][1];
                P.grad[o * D + 1] = acc[t][2];
                if (D == 3) P.grad[o * D + 2] = acc[t][3];
            }
        }
    }
}

static ChebTable cheb_table(int q) {
    ChebTable T{};
    for (int i = 0; i < q; ++i)
        T.t[i] = (float)cos((2.0 * i + 1.0) * 3.14159265358979323846 / (2.0 * q));
    for (int k = 0; k < q; ++k) {
        double den = 1.0;
        const double tk = cos((2.0 * k + 1.0) * 3.14159265358979323846 / (2.0 * q));
        for (int i = 0; i < q; ++i)
            if (i != k) den *= tk - cos((2.0 * i + 1.0) * 3.14159265358979323846 / (2.0 * q));
        T.inv_den[k] = (float)(1.0 / den);
    }
    return T;
}

}  // namespace spk

using namespace spk;

extern "C" {

int spk_tree_keys(const void* pos, int64_t n, int dims, uint64_t* keys, int32_t* idx,
                  spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(n >= 0 && n < (1LL << 31), SPK_ERR_ARG, "tree: %lld points out of range",
                (long long)n);
    if (n == 0) return SPK_OK;
    keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const float4*>(pos), n, dims, keys, idx);
    SPK_CHECK_LAUNCH("spk_tree_keys");
    return SPK_OK;
}

size_t spk_tree_sort_workspace_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr,
                                    (uint64_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, 64);
    return bytes + 256;
}

int spk_tree_sort(const uint64_t* keys_in, const int32_t* idx_in, uint64_t* keys_out,
                  int32_t* idx_out, int64_t n, int dims, void* ws, size_t ws_bytes,
                  spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    if (n == 0) return SPK_OK;
    const int end_bit = dims == 3 ? 63 : 62;
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in, keys_out, idx_in, idx_out, (int)n,
                                    0, end_bit, (cudaStream_t)stream);
    SPK_REQUIRE(ws_bytes >= need, SPK_ERR_WORKSPACE, "tree sort: workspace %zu < %zu bytes",
                ws_bytes, need);
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(
        ws, need, keys_in, keys_out, idx_in, idx_out, (int)n, 0, end_bit, (cudaStream_t)stream);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree sort: %s", cudaGetErrorString(e));
    return SPK_OK;
}

int spk_tree_gather(const void* pos, const int32_t* perm, int64_t n, const float* weights,
                    void* out, spk_stream_t stream) {
    if (n == 0) return SPK_OK;
    gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const float4*>(pos), perm, n, weights, static_cast<float4*>(out));
    SPK_CHECK_LAUNCH("spk_tree_gather");
    return SPK_OK;
}

int spk_tree_boxes(const void* rec, int64_t n_ranges, const int64_t* begin,
                   const int64_t* end, int dims, float* box, spk_stream_t stream) {
    if (n_ranges == 0) return SPK_OK;
    boxes_kernel<<<(unsigned)n_ranges, 256, 0, (cudaStream_t)stream>>>(
        static_cast<const float4*>(rec), reinterpret_cast<const long long*>(begin),
        reinterpret_cast<const long long*>(end), dims, box, nullptr);
    SPK_CHECK_LAUNCH("spk_tree_boxes");
    return SPK_OK;
}

size_t spk_tree_p2m_workspace_bytes(int64_t n_units, int order, int dims) {
    const int64_t m = dims == 3 ? (int64_t)order * order * order : (int64_t)order * order;
    return (size_t)(n_units * m) * sizeof(double);
}

int spk_tree_p2m(const void* rec, int64_t n_units, const int32_t* unit_slot,
                 const int64_t* unit_begin, const int64_t* unit_end, int64_t n_slots,
                 const int64_t* slot_unit_off, const float* slot_box, int order, int dims,
                 void* proxies, void* ws, size_t ws_bytes, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(order >= 2 && order <= P2M_MAX_ORDER, SPK_ERR_ARG,
                "interpolation order must be in [2, %d], got %d", P2M_MAX_ORDER, order);
    if (n_slots == 0) return SPK_OK;
    SPK_REQUIRE(ws_bytes >= spk_tree_p2m_workspace_bytes(n_units, order, dims),
                SPK_ERR_WORKSPACE, "tree p2m: workspace too small");
    const ChebTable T = cheb_table(order);
    double* part = static_cast<double*>(ws);
    cudaStream_t s = (cudaStream_t)stream;
    p2m_kernel<<<(unsigned)n_units, P2M_THREADS, 0, s>>>(
        static_cast<const float4*>(rec), unit_slot, reinterpret_cast<const long long*>(unit_begin),
        reinterpret_cast<const long long*>(unit_end), slot_box, order, dims, T, part);
    SPK_CHECK_LAUNCH("spk_tree_p2m");
    p2m_final_kernel<<<(unsigned)n_slots, 128, 0, s>>>(
        part, reinterpret_cast<const long long*>(slot_unit_off), slot_box, order, dims, T,
        static_cast<float4*>(proxies));
    SPK_CHECK_LAUNCH("spk_tree_p2m(final)");
    return SPK_OK;
}

int spk_tree_eval(const void* tgt_sorted, const int32_t* tgt_perm, int64_t n_groups,
                  const int64_t* grp_begin, const int64_t* grp_end, const int32_t* grp_list,
                  const void* src, const int64_t* seg_off, const int64_t* seg_start,
                  const int32_t* seg_count, int dims, float eps2, double* val, double* grad,
                  spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    if (n_groups == 0) return SPK_OK;
    EvalParams P;
    P.tgt = static_cast<const float4*>(tgt_sorted);
    P.tgt_perm = tgt_perm;
    P.grp_begin = reinterpret_cast<const long long*>(grp_begin);
    P.grp_end = reinterpret_cast<const long long*>(grp_end);
    P.src = static_cast<const float4*>(src);
    P.seg_off = reinterpret_cast<const long long*>(seg_off);
    P.grp_list = grp_list;
    P.seg_start = reinterpret_cast<const long long*>(seg_start);
    P.seg_count = seg_count;
    P.eps2 = eps2;
    P.val = val;
    P.grad = grad;
    const bool guard = !(eps2 >= FLT_MIN);
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)((n_groups + TR_WARPS - 1) / TR_WARPS);
    if (dims == 3) {
        if (guard) tree_eval_kernel<3, true><<<blocks, TR_THREADS, 0, s>>>(P, n_groups);
        else tree_eval_kernel<3, false><<<blocks, TR_THREADS, 0, s>>>(P, n_groups);
    } else {
        if (guard) tree_eval_kernel<2, true><<<blocks, TR_THREADS, 0, s>>>(P, n_groups);
        else tree_eval_kernel<2, false><<<blocks, TR_THREADS, 0, s>>>(P, n_groups);
    }
    SPK_CHECK_LAUNCH("spk_tree_eval");
    return SPK_OK;
}

int spk_tree_node_boxes(const void* rec, int64_t n_nodes, const int32_t* first_child,
                        const int32_t* n_child, int64_t n_leaves, const int32_t* leaf_node,
                        const int64_t* leaf_begin, const int64_t* leaf_end, int64_t n_levels,
                        const int64_t* level_off, int dims, float* node_box,
                        spk_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n_nodes == 0) return SPK_OK;
    boxes_kernel<<<(unsigned)n_leaves, 256, 0, s>>>(
        static_cast<const float4*>(rec), reinterpret_cast<const long long*>(leaf_begin),
        reinterpret_cast<const long long*>(leaf_end), dims, node_box, leaf_node);
    SPK_CHECK_LAUNCH("spk_tree_node_boxes(leaves)");
    for (int64_t l = n_levels - 1; l >= 0; --l) {  // host array of level offsets
        const long long b = level_off[l], e = level_off[l + 1];
        if (e <= b) continue;
        level_boxes_kernel<<<(unsigned)((e - b + 127) / 128), 128, 0, s>>>(first_child, n_child,
                                                                          b, e, node_box);
    }
    SPK_CHECK_LAUNCH("spk_tree_node_boxes(levels)");
    return SPK_OK;
}

size_t spk_tree_plan_workspace_bytes(int64_t n_nodes, int64_t n_groups) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)n_nodes);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long*)nullptr, (long long*)nullptr,
                                  (int)(n_groups * TR_FRONT + 1));
    cub::DeviceScan::ExclusiveSum(nullptr, c, (const long long*)nullptr, (long long*)nullptr,
                                  (int)(n_nodes + 1));
    const size_t cub_bytes = std::max(a, std::max(b, c));
    // is_proxy [n_nodes] i32, seg_cnt [n_groups * TR_FRONT + 1] i64 (per group, or per
    // sub-walk), units_per_slot [n_nodes + 1] i64
    return ((cub_bytes + 255) & ~(size_t)255) + (size_t)n_nodes * 4 + 256 +
           (size_t)(n_groups * TR_FRONT + 1) * 8 + 256 + (size_t)(n_nodes + 1) * 8 + 256;
}

static void plan_ws(void* ws, int64_t n_nodes, int64_t n_groups, size_t cub_bytes,
                    void** cub_tmp, int32_t** is_proxy, long long** seg_cnt,
                    long long** units_per_slot) {
    char* p = static_cast<char*>(ws);
    *cub_tmp = p;
    p += (cub_bytes + 255) & ~(size_t)255;
    *is_proxy = reinterpret_cast<int32_t*>(p);
    p += ((size_t)n_nodes * 4 + 255) & ~(size_t)255;
    *seg_cnt = reinterpret_cast<long long*>(p);
    p += ((size_t)(n_groups * TR_FRONT + 1) * 8 + 255) & ~(size_t)255;
    *units_per_slot = reinterpret_cast<long long*>(p);
}

int spk_tree_plan_count(const int64_t* node_begin, const int64_t* node_end,
                        const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                        const float* node_box, const float* group_box, int64_t n_groups,
                        double theta, int order, int dims, int64_t n_src, int32_t* slot_of,
                        int32_t* slot_node, float* slot_box, int64_t* slot_unit_off,
                        int64_t* seg_off, int64_t* totals, const float* parent_box,
                        const int32_t* group_parent, int far_only, int64_t* sub_off, void* ws,
                        size_t ws_bytes, spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(n_nodes > 0 && n_groups > 0, SPK_ERR_ARG, "tree plan: empty tree or groups");
    SPK_REQUIRE(sub_off == nullptr || parent_box == nullptr, SPK_ERR_ARG,
                "tree plan: sub-walks are for the plain traversal (no far-level parents)");
    SPK_REQUIRE(ws_bytes >= spk_tree_plan_workspace_bytes(n_nodes, n_groups), SPK_ERR_WORKSPACE,
                "tree plan: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    size_t cub_bytes = ws_bytes - ((size_t)n_nodes * 4 + 256 +
                                   (size_t)(n_groups * TR_FRONT + 1) * 8 + 256 +
                                   (size_t)(n_nodes + 1) * 8 + 256);
    cub_bytes &= ~(size_t)255;
    void* tmp;
    int32_t* is_proxy;
    long long* seg_cnt;
    long long* ups;
    plan_ws(ws, n_nodes, n_groups, cub_bytes, &tmp, &is_proxy, &seg_cnt, &ups);
    cudaMemsetAsync(is_proxy, 0, (size_t)n_nodes * 4, s);
    cudaMemsetAsync(seg_cnt, 0, (size_t)(n_groups * TR_FRONT + 1) * 8, s);
    cudaMemsetAsync(ups, 0, (size_t)(n_nodes + 1) * 8, s);
    const int m = dims == 3 ? order * order * order : order * order;
    TravParams P{};
    P.nbeg = reinterpret_cast<const long long*>(node_begin);
    P.nend = reinterpret_cast<const long long*>(node_end);
    P.fchild = first_child;
    P.nchild = n_child;
    P.nbox = node_box;
    P.gbox = group_box;
    P.n_groups = n_groups;
    P.dims = dims;
    P.theta = (float)theta;
    P.m = m;
    P.n_src = n_src;
    P.is_proxy = is_proxy;
    P.seg_cnt = seg_cnt;
    P.pbox = parent_box;
    P.gparent = group_parent;
    P.far_only = far_only;
    P.overflow = reinterpret_cast<unsigned long long*>(totals + 3);
    cudaMemsetAsync(totals + 3, 0, sizeof(int64_t), s);
    const int fan = dims == 3 ? 8 : 4, front = fan * fan;
    if (sub_off) {
        P.sub_cnt = seg_cnt;
        const long long nt = n_groups * front;
        traverse_sub_kernel<0><<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(P, front, fan);
    } else {
        traverse_kernel<0><<<(unsigned)((n_groups + 127) / 128), 128, 0, s>>>(P);
    }
    SPK_CHECK_LAUNCH("spk_tree_plan_count(traverse)");
    size_t t = cub_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, t, is_proxy, slot_of, (int)n_nodes, s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree plan scan: %s", cudaGetErrorString(e));
    t = cub_bytes;
    if (sub_off) {
        e = cub::DeviceScan::ExclusiveSum(tmp, t, seg_cnt, reinterpret_cast<long long*>(sub_off),
                                          (int)(n_groups * front + 1), s);
        SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree plan scan: %s", cudaGetErrorString(e));
        group_offsets_kernel<<<(unsigned)((n_groups + 1 + 127) / 128), 128, 0, s>>>(
            reinterpret_cast<const long long*>(sub_off), n_groups, front,
            reinterpret_cast<long long*>(seg_off));
    } else {
        e = cub::DeviceScan::ExclusiveSum(tmp, t, seg_cnt, reinterpret_cast<long long*>(seg_off),
                                          (int)(n_groups + 1), s);
    }
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree plan scan: %s", cudaGetErrorString(e));
    slots_kernel<<<(unsigned)((n_nodes + 127) / 128), 128, 0, s>>>(
        P.nbeg, P.nend, node_box, is_proxy, slot_of, n_nodes, dims, slot_node, slot_box, ups);
    SPK_CHECK_LAUNCH("spk_tree_plan_count(slots)");
    t = cub_bytes;
    e = cub::DeviceScan::ExclusiveSum(tmp, t, ups, reinterpret_cast<long long*>(slot_unit_off),
                                      (int)(n_nodes + 1), s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree plan scan: %s", cudaGetErrorString(e));
    totals_kernel<<<1, 1, 0, s>>>(reinterpret_cast<const long long*>(seg_off), n_groups, slot_of,
                                  is_proxy, reinterpret_cast<const long long*>(slot_unit_off),
                                  n_nodes, reinterpret_cast<long long*>(totals));
    SPK_CHECK_LAUNCH("spk_tree_plan_count(totals)");
    return SPK_OK;
}

int spk_tree_plan_write(const int64_t* node_begin, const int64_t* node_end,
                        const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                        const float* node_box, const float* group_box, int64_t n_groups,
                        double theta, int order, int dims, int64_t n_src,
                        const int32_t* slot_of, const int32_t* slot_node,
                        const int64_t* slot_unit_off, int64_t n_slots, const int64_t* seg_off,
                        int64_t* seg_start, int32_t* seg_count, int32_t* unit_slot,
                        int64_t* unit_begin, int64_t* unit_end, const float* parent_box,
                        const int32_t* group_parent, int far_only, const int64_t* sub_off,
                        spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    cudaStream_t s = (cudaStream_t)stream;
    TravParams P{};
    P.nbeg = reinterpret_cast<const long long*>(node_begin);
    P.nend = reinterpret_cast<const long long*>(node_end);
    P.fchild = first_child;
    P.nchild = n_child;
    P.nbox = node_box;
    P.gbox = group_box;
    P.n_groups = n_groups;
    P.dims = dims;
    P.theta = (float)theta;
    P.m = dims == 3 ? order * order * order : order * order;
    P.n_src = n_src;
    P.slot_of = slot_of;
    P.seg_off = reinterpret_cast<const long long*>(seg_off);
    P.seg_start = reinterpret_cast<long long*>(seg_start);
    P.seg_count = seg_count;
    P.pbox = parent_box;
    P.gparent = group_parent;
    P.far_only = far_only;
    if (sub_off) {
        const int fan = dims == 3 ? 8 : 4, front = fan * fan;
        P.sub_off = reinterpret_cast<const long long*>(sub_off);
        const long long nt = n_groups * front;
        traverse_sub_kernel<1><<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(P, front, fan);
    } else {
        traverse_kernel<1><<<(unsigned)((n_groups + 127) / 128), 128, 0, s>>>(P);
    }
    SPK_CHECK_LAUNCH("spk_tree_plan_write(traverse)");
    if (n_slots > 0) {
        units_kernel<<<(unsigned)((n_slots + 127) / 128), 128, 0, s>>>(
            P.nbeg, P.nend, slot_node, reinterpret_cast<const long long*>(slot_unit_off), n_slots,
            unit_slot, reinterpret_cast<long long*>(unit_begin),
            reinterpret_cast<long long*>(unit_end));
        SPK_CHECK_LAUNCH("spk_tree_plan_write(units)");
    }
    return SPK_OK;
}

size_t spk_tree_build_workspace_bytes(int64_t n, int64_t node_capacity) {
    const long long m = node_capacity + 1;
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr, (int)m);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long*)nullptr, (long long*)nullptr,
                                  (int)m);
    cub::DeviceRadixSort::SortPairs(nullptr, c, (const long long*)nullptr, (long long*)nullptr,
                                    (const long long*)nullptr, (long long*)nullptr, (int)m);
    d = std::max(std::max(a, b), c);
    // nchild i32 + off i32 (m each), child ranges (16 i64 per node), group counts/offsets
    // (2 x m i64), group sort buffers (4 x m i64)
    return ((d + 255) & ~(size_t)255) + (size_t)m * (4 + 4 + 128 + 16 + 32) + 4096;
}

namespace {
struct BuildWs {
    void* cub;
    size_t cub_bytes;
    int32_t* nchild;
    int32_t* off;
    long long* child;
    long long* gcnt;
    long long* goff;
    long long* sort_k;
    long long* sort_v;
};
BuildWs build_ws(void* ws, size_t ws_bytes, long long m) {
    BuildWs w;
    const size_t fixed = (size_t)m * (4 + 4 + 128 + 16 + 32) + 4096;
    w.cub_bytes = (ws_bytes - fixed) & ~(size_t)255;
    char* p = static_cast<char*>(ws);
    w.cub = p;
    p += w.cub_bytes;
    auto take = [&](size_t bytes) {
        char* q = p;
        p += (bytes + 255) & ~(size_t)255;
        return q;
    };
    w.nchild = reinterpret_cast<int32_t*>(take((size_t)m * 4));
    w.off = reinterpret_cast<int32_t*>(take((size_t)m * 4));
    w.child = reinterpret_cast<long long*>(take((size_t)m * 128));
    w.gcnt = reinterpret_cast<long long*>(take((size_t)m * 8));
    w.goff = reinterpret_cast<long long*>(take((size_t)m * 8));
    w.sort_k = reinterpret_cast<long long*>(take((size_t)m * 16));
    w.sort_v = reinterpret_cast<long long*>(take((size_t)m * 16));
    return w;
}
}  // namespace

int spk_tree_build(const uint64_t* keys, int64_t n, int dims, int64_t leaf_cap,
                   int min_level, int64_t node_capacity, int64_t* node_begin, int64_t* node_end,
                   int32_t* first_child, int32_t* n_child, int32_t* leaf_node,
                   int64_t* level_off, int64_t* counts, void* ws, size_t ws_bytes,
                   spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    SPK_REQUIRE(n >= 1 && leaf_cap >= 1, SPK_ERR_ARG, "tree build: n=%lld leaf_cap=%lld",
                (long long)n, (long long)leaf_cap);
    SPK_REQUIRE(ws_bytes >= spk_tree_build_workspace_bytes(n, node_capacity), SPK_ERR_WORKSPACE,
                "tree build: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const int bits = dims == 3 ? 21 : 31;
    BuildWs w = build_ws(ws, ws_bytes, node_capacity + 1);
    long long* nb = reinterpret_cast<long long*>(node_begin);
    long long* ne = reinterpret_cast<long long*>(node_end);
    root_kernel<<<1, 1, 0, s>>>(n, nb, ne);
    long long lv_b = 0, lv_e = 1;
    int level = 0;
    level_off[0] = 0;
    int32_t total_h = 0;
    while (lv_e > lv_b) {
        const long long m = lv_e - lv_b;
        SPK_REQUIRE(lv_e + 8 * m <= node_capacity, SPK_ERR_WORKSPACE,
                    "tree build: node capacity %lld exceeded", (long long)node_capacity);
        SPK_REQUIRE(level < 63, SPK_ERR_ARG, "tree build: too many levels");
        const unsigned blocks = (unsigned)((m + 127) / 128);
        split_kernel<<<blocks, 128, 0, s>>>(keys, nb, ne, lv_b, lv_e, level, dims, bits,
                                            (long long)leaf_cap, min_level, w.nchild, w.child);
        cudaMemsetAsync(w.nchild + m, 0, 4, s);
        size_t t = w.cub_bytes;
        cudaError_t e = cub::DeviceScan::ExclusiveSum(w.cub, t, w.nchild, w.off, (int)(m + 1), s);
        SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree build scan: %s", cudaGetErrorString(e));
        link_kernel<<<blocks, 128, 0, s>>>(w.nchild, w.off, w.child, lv_b, lv_e, nb, ne,
                                           first_child, n_child);
        e = cudaMemcpyAsync(&total_h, w.off + m, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree build: %s", cudaGetErrorString(e));
        level_off[++level] = lv_e;
        lv_b = lv_e;
        lv_e += total_h;
    }
    SPK_CHECK_LAUNCH("spk_tree_build(levels)");
    const long long n_nodes = lv_e;
    // leaves in BFS order
    const unsigned nb_blocks = (unsigned)((n_nodes + 255) / 256);
    leaf_flag_kernel<<<nb_blocks, 256, 0, s>>>(n_child, n_nodes, w.nchild);
    cudaMemsetAsync(w.nchild + n_nodes, 0, 4, s);
    size_t t = w.cub_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(w.cub, t, w.nchild, w.off, (int)(n_nodes + 1), s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree build scan: %s", cudaGetErrorString(e));
    leaf_write_kernel<<<nb_blocks, 256, 0, s>>>(w.nchild, w.off, n_nodes, leaf_node);
    SPK_CHECK_LAUNCH("spk_tree_build(leaves)");
    e = cudaMemcpyAsync(&total_h, w.off + n_nodes, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree build: %s", cudaGetErrorString(e));
    counts[0] = n_nodes;
    counts[1] = total_h;
    counts[2] = level;  // level_off has level + 1 entries
    return SPK_OK;
}

int spk_tree_groups(const int64_t* node_begin, const int64_t* node_end,
                    const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                    int64_t cap, const uint8_t* cut, int64_t group_capacity,
                    int64_t* grp_begin, int64_t* grp_end, int64_t* n_groups, void* ws,
                    size_t ws_bytes, spk_stream_t stream) {
    SPK_REQUIRE(cap >= 1, SPK_ERR_ARG, "tree groups: cap must be >= 1");
    SPK_REQUIRE(ws_bytes >= spk_tree_build_workspace_bytes(0, std::max(n_nodes, group_capacity)),
                SPK_ERR_WORKSPACE, "tree groups: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    BuildWs w = build_ws(ws, ws_bytes, std::max(n_nodes, group_capacity) + 1);
    const long long* nb = reinterpret_cast<const long long*>(node_begin);
    const long long* ne = reinterpret_cast<const long long*>(node_end);
    const unsigned blocks = (unsigned)((n_nodes + 127) / 128);
    groups_kernel<0><<<blocks, 128, 0, s>>>(nb, ne, first_child, n_child, n_nodes, cap, cut,
                                            w.gcnt,
                                            nullptr, nullptr, nullptr);
    cudaMemsetAsync(w.gcnt + n_nodes, 0, 8, s);
    size_t t = w.cub_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(w.cub, t, w.gcnt, w.goff, (int)(n_nodes + 1), s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree groups scan: %s", cudaGetErrorString(e));
    long long total = 0;
    e = cudaMemcpyAsync(&total, w.goff + n_nodes, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree groups: %s", cudaGetErrorString(e));
    *n_groups = total;
    SPK_REQUIRE(total <= group_capacity, SPK_ERR_WORKSPACE,
                "tree groups: %lld groups exceed capacity %lld", total, (long long)group_capacity);
    groups_kernel<1><<<blocks, 128, 0, s>>>(nb, ne, first_child, n_child, n_nodes, cap, cut,
                                            nullptr,
                                            w.goff, w.sort_k, w.sort_v);
    SPK_CHECK_LAUNCH("spk_tree_groups");
    t = w.cub_bytes;
    e = cub::DeviceRadixSort::SortPairs(w.cub, t, w.sort_k,
                                        reinterpret_cast<long long*>(grp_begin), w.sort_v,
                                        reinterpret_cast<long long*>(grp_end), (int)total, 0, 40,
                                        s);
    SPK_REQUIRE(e == cudaSuccess, SPK_ERR_CUDA, "tree groups sort: %s", cudaGetErrorString(e));
    return SPK_OK;
}

int spk_tree_cheb_targets(const float* parent_box, int64_t n_parents, int order, int dims,
                          void* points, float* parent_cheb_box, spk_stream_t stream) {
    SPK_REQUIRE(order >= 2 && order <= P2M_MAX_ORDER, SPK_ERR_ARG, "bad order %d", order);
    if (n_parents == 0) return SPK_OK;
    cheb_targets_kernel<<<(unsigned)n_parents, 128, 0, (cudaStream_t)stream>>>(
        parent_box, n_parents, order, dims, cheb_table(order), static_cast<float4*>(points),
        parent_cheb_box);
    SPK_CHECK_LAUNCH("spk_tree_cheb_targets");
    return SPK_OK;
}

int spk_tree_parent_ids(const int64_t* parent_begin, const int64_t* parent_end,
                        int64_t n_parents, int32_t* pid, spk_stream_t stream) {
    if (n_parents == 0) return SPK_OK;
    parent_ids_kernel<<<(unsigned)n_parents, 128, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const long long*>(parent_begin),
        reinterpret_cast<const long long*>(parent_end), n_parents, pid);
    SPK_CHECK_LAUNCH("spk_tree_parent_ids");
    return SPK_OK;
}

int spk_tree_l2p(const void* tgt_sorted, const int32_t* tgt_perm, int64_t n_tgt,
                 const int32_t* pid, const float* parent_cheb_box, const double* pval,
                 const double* pgrad, int order, int dims, double* val, double* grad,
                 spk_stream_t stream) {
    SPK_REQUIRE(dims == 2 || dims == 3, SPK_ERR_ARG, "dims must be 2 or 3, got %d", dims);
    if (n_tgt == 0) return SPK_OK;
    const unsigned blocks = (unsigned)((n_tgt + 127) / 128);
    const ChebTable T = cheb_table(order);
    if (dims == 3)
        l2p_kernel<3><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            static_cast<const float4*>(tgt_sorted), tgt_perm, n_tgt, pid, parent_cheb_box, pval,
            pgrad, order, T, val, grad);
    else
        l2p_kernel<2><<<blocks, 128, 0, (cudaStream_t)stream>>>(
            static_cast<const float4*>(tgt_sorted), tgt_perm, n_tgt, pid, parent_cheb_box, pval,
            pgrad, order, T, val, grad);
    SPK_CHECK_LAUNCH("spk_tree_l2p");
    return SPK_OK;
}

int spk_tree_group_size(void) { return TR_GROUP; }

}  // extern "C"
