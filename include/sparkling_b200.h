/*
 * sparkling_b200.h -- C ABI of the B200 (sm_100a) SPARKLING hot path.
 *
 * Every entry point is stream-ordered, never allocates or frees, and takes caller-owned
 * DEVICE pointers (torch tensors' data_ptr() on the Python side), sizes as int64_t,
 * scalars by value and an explicit cudaStream_t.  Scratch memory is a caller-provided
 * workspace whose size is given by the matching *_workspace_bytes() query.  Each call
 * returns SPK_OK (0) or a nonzero SPK_ERR_* code; spk_last_error() then holds a
 * one-line message.  No C++ exception crosses this boundary.
 *
 * Sample positions used by the N-body kernels are float4 records {x, y, z, |x|^2} (z = 0
 * in 2D); the density is passed as fp32 lattice weights with implicit node coordinates.
 * Trajectories are fp64 (n_shots, n_s, dims) row-major, shot-major, axis-innermost,
 * exactly the SamplingPattern.coords layout (reference src/core.py:141-186).
 *
 * Reference paths below are relative to /root/reference/pkg/src/vdtraj/.
 */
#ifndef SPARKLING_B200_H
#define SPARKLING_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* spk_stream_t; /* == cudaStream_t */

enum {
    SPK_OK = 0,
    SPK_ERR_ARG = 1,       /* invalid shape / argument (reference raises ValueError) */
    SPK_ERR_LAUNCH = 2,    /* kernel launch failure */
    SPK_ERR_WORKSPACE = 3, /* workspace too small */
    SPK_ERR_CUDA = 4       /* other CUDA runtime error */
};

int spk_version(void);

/* CUDA IPC of device buffers (the fused position all-gather between ranks): the 64-byte
 * handle of an allocation's base, and opening a peer's handle on the caller's current
 * device (peer access enabled lazily), closing it again. */
int spk_ipc_handle(const void* base, void* handle_out);
int spk_ipc_open(const void* handle, void** ptr_out);
int spk_ipc_close(void* ptr);
const char* spk_last_error(void);

/* ---------------------------------------------------------------- K1 / K2 N-body */

/* Workspace for one spk_*_sums call with n_tgt targets, n_cells lattice cells (segment 0)
 * and n_pos positions (segment 1). */
size_t spk_nbody_workspace_bytes(int64_t n_tgt, int64_t n_cells, int64_t n_pos);

/* Repulsion raw sums.  Replaces _treecode.direct_sums (_treecode.py:506-534) and
 * direct_sums_subset (:474-503): for every target i,
 *   val[i]  = sum_j sqrt(|t_i - s_j|^2 + eps2)
 *   grad[i] = sum_j (t_i - s_j) / sqrt(|t_i - s_j|^2 + eps2)   (term skipped when 0)
 * over the n_src sources (i == j included, as the reference does).  fp32 pair math on
 * the FMA + MUFU pipes, fp64 accumulation across source tiles.  val: [n_tgt] f64,
 * grad: [n_tgt, dims] f64.  Called by eval_repulsion_direct (repulsion.py:72-87). */
int spk_direct_sums(const void* tgt, int64_t n_tgt, const void* src, int64_t n_src,
                    int dims, float eps2, double* val, double* grad, void* ws,
                    size_t ws_bytes, spk_stream_t stream);

/* Attraction raw sums over the density lattice (north-star attraction):
 *   val[i]  = sum_y w_y sqrt(|t_i - y|^2 + eps2),  grad[i] = sum_y w_y (t_i - y)/h,
 * y over the side0 x side1 [x side2] node grid, node i on axis a at (i - N_a)/N_a with
 * side_a = 2 N_a + 1 (density.py:58-67); grid_w: fp32 weights, row-major, zero-padded
 * to a multiple of 4 (spk_build_grid_sources); side: host array of dims sides (<= 1023).
 * With the grid nodes themselves as targets this is precompute_field's potential and
 * force (attraction.py:62-113). */
int spk_grid_sums(const void* tgt, int64_t n_tgt, const float* grid_w, const int64_t* side,
                  int dims, float eps2, double* val, double* grad, void* ws,
                  size_t ws_bytes, spk_stream_t stream);

/* K2 for the rows of a shot subset (the multi-GPU path's attraction of shots whose polish
 * has finished, overlapped with the polish of the others): targets are the n_s records
 * of each listed shot in tgt (shot-major), results go to the same rows of val [.] and
 * grad [.][dims] (other rows untouched).  Same arithmetic as spk_grid_sums.
 * sm_busy (optional, device int32 [256], zero-initialised, shared with spk_polish_shots):
 * each CTA first waits until its SM holds no polish CTA, so the launch uses only the SMs
 * the polish has left (NULL = no waiting). */
size_t spk_grid_sums_shots_workspace_bytes(int64_t n_ids, int n_s, int64_t n_cells);
int spk_grid_sums_shots(const void* tgt, const int32_t* shot_ids, int64_t n_ids, int n_s,
                        const float* grid_w, const int64_t* side, int dims, float eps2,
                        double* val, double* grad, const int32_t* sm_busy, void* ws,
                        size_t ws_bytes, spk_stream_t stream);

/* Both sums in ONE launch (the optimize() hot loop, optimizer.py:302-303): segment 0 =
 * the density lattice (attraction), segment 1 = positions (repulsion).  Either segment
 * may be empty (grid_w = NULL or n_pos = 0). */
int spk_fused_sums(const void* tgt, int64_t n_tgt, int dims, const float* grid_w,
                   const int64_t* side, float eps2_att, const void* pos_src, int64_t n_pos,
                   float eps2_rep, double* val_att, double* grad_att, double* val_rep,
                   double* grad_rep, void* ws, size_t ws_bytes, spk_stream_t stream);

/* Stack-of-SPARKLING batch (BASELINE config 3): n_groups independent problems of per_group
 * targets each, targets contiguous by problem; problem q's repulsion sources are its own
 * n_pos positions at pos_src + q * n_pos records; the density lattice is shared.  Same
 * sums as spk_fused_sums per problem, one launch for the whole batch. */
size_t spk_nbody_batched_workspace_bytes(int64_t n_groups, int64_t per_group, int64_t n_cells,
                                         int64_t n_pos);
int spk_fused_sums_batched(const void* tgt, int64_t n_groups, int64_t per_group, int dims,
                           const float* grid_w, const int64_t* side, float eps2_att,
                           const void* pos_src, int64_t n_pos, float eps2_rep,
                           double* val_att, double* grad_att, double* val_rep,
                           double* grad_rep, void* ws, size_t ws_bytes, spk_stream_t stream);

/* Pack fp64 (p, dims) coordinates into position records float4 {x, y, z|0, |x|^2}. */
int spk_pack_positions(const double* coords, int64_t p, int dims, void* pos4,
                       spk_stream_t stream);

/* Lattice sources from an fp64 density grid (rho row-major, `side` host array of dims odd
 * sides): fp32 weights (caller allocates prod(side) rounded up to a multiple of 4
 * floats) and, if `nodes` != NULL, the node position records float4 {x, y, z|0, |x|^2}
 * (targets for precompute_field). */
int spk_build_grid_sources(const double* rho, int dims, const int64_t* side, float* weights,
                           void* nodes, spk_stream_t stream);

/* Combine raw sums into the optimizer gradient and scalars (optimizer.py:302-321):
 *   grad[i] = grad_att[i] / p_att - grad_rep[i] / (p_rep * p_rep)
 * (either term may be absent: pass NULL), and scalars written to out[0..5]:
 *   out[0] = sum val_att, out[1] = sum val_rep,
 *   out[2] = <coords - prev_coords, grad - prev_grad>, out[3] = <grad - prev_grad, ..>,
 *   out[4] = count of non-finite gradient entries, out[5] = 0.
 * prev_* may be NULL (then out[2..3] = 0).  Deterministic fixed-order reductions. */
size_t spk_combine_workspace_bytes(int64_t n);
int spk_combine_gradient(int64_t n_tgt, int dims, const double* val_att,
                         const double* grad_att, double p_att, const double* val_rep,
                         const double* grad_rep, double p_rep, const double* coords,
                         const double* prev_coords, const double* prev_grad, double* grad,
                         double* out, void* ws, size_t ws_bytes, spk_stream_t stream);

/* Per-problem form of spk_combine_gradient for a batch: out[q * 6 + 0..5]. */
size_t spk_combine_batched_workspace_bytes(int64_t n_groups, int64_t per_group);
int spk_combine_gradient_batched(int64_t n_groups, int64_t per_group, int dims,
                                 const double* val_att, const double* grad_att, double p_att,
                                 const double* val_rep, const double* grad_rep, double p_rep,
                                 const double* coords, const double* prev_coords,
                                 const double* prev_grad, double* grad, double* out, void* ws,
                                 size_t ws_bytes, spk_stream_t stream);

/* ---------------------------------------------------------------- K3 projection */

size_t spk_project_workspace_bytes(int64_t n_shots, int n_s, int dims, int with_trace);

/* Batched shot projection.  Replaces _project_all (projection.py:376-382): per shot,
 * n_pit iterations of dual FISTA with gradient restart (_project_shot, :169-284), then
 * the relaxed cyclic feasibility polish (_feasibility_polish, :287-373) to tol with at
 * most max_sweeps sweeps.  fp64, bit-identical to the reference.
 *   in:  shots (n_shots, n_s, dims) f64; if grad != NULL the projected point is
 *        in - eta * grad (the optimizer step, optimizer.py:326); eta_per_shot (device,
 *        nullable, n_shots f64) replaces eta per shot (batched independent problems).
 *   out: projected shots; pos4 (nullable) receives float4 positions of the result;
 *        sweeps (nullable) the polish sweep count per shot; trace (nullable,
 *        n_shots * n_pit f64) the dual objective per iteration (project_shot
 *        return_trace=True, :394-418); nonfinite (nullable, 1 int32) is set to 1 when
 *        the stepped input is not finite (SamplingPattern check, core.py:157).
 *   pin_idx < 0 means no pin; pin_val: host array of dims doubles. */
int spk_project_all(const double* in, const double* grad, double eta,
                    const double* eta_per_shot, double* out, int64_t n_shots, int n_s, int dims, double a, double b, int pin_idx,
                    const double* pin_val, int n_pit, double tau, int monotone, double tol,
                    int max_sweeps, void* pos4, int32_t* sweeps, double* trace,
                    int32_t* nonfinite, void* ws, size_t ws_bytes, spk_stream_t stream);

/* The two halves of spk_project_all, for callers that schedule the polish themselves:
 * FISTA for all shots (out = FISTA result, the workspace keeps no state the polish
 * needs), then the polish of a subset of shots shot_ids[0..n_ids) (null = all n_shots) in
 * place on `shots`, with the workspace of spk_project_workspace_bytes(n_shots, ...).
 * Several disjoint subsets may be polished concurrently on different streams. */
int spk_project_fista(const double* in, const double* grad, double eta,
                      const double* eta_per_shot, double* out, int64_t n_shots, int n_s,
                      int dims, double a, double b, int pin_idx, const double* pin_val,
                      int n_pit, double tau, int monotone, double* trace, int32_t* nonfinite,
                      void* ws, size_t ws_bytes, spk_stream_t stream);
/* sm_busy (optional, see spk_grid_sums_shots): every polish CTA counts itself on its SM
 * while it runs.  peer_pos4 (optional): a DEVICE array of n_peers float4 position
 * buffers of the other ranks (peer memory, e.g. CUDA IPC over NVLink); every record
 * written to pos4[c * n_s + n] is also written to peer_pos4[k][peer_offset + c * n_s + n]
 * -- the position all-gather fused into the polish epilogue (the caller orders the
 * peers' reads after a collective that follows this launch on every rank). */
int spk_polish_shots(double* shots, const int32_t* shot_ids, int64_t n_ids, int64_t n_shots,
                     int n_s, int dims, double a, double b, int pin_idx, const double* pin_val,
                     double tol, int max_sweeps, void* pos4, int32_t* sweeps,
                     int32_t* sm_busy, void* const* peer_pos4, int n_peers,
                     int64_t peer_offset, void* ws, size_t ws_bytes, spk_stream_t stream);

/* feasibility_residuals (projection.py:435-452): out[0..4] = amplitude, speed,
 * acceleration, pin (0 if no pin), max -- each already clipped at 0 like the reference. */
size_t spk_residuals_workspace_bytes(int64_t n_shots);
int spk_feasibility_residuals(const double* coords, int64_t n_shots, int n_s, int dims,
                              double a, double b, int pin_idx, const double* pin_val,
                              double* out, void* ws, size_t ws_bytes, spk_stream_t stream);

/* Per-problem residuals for a batch of n_groups x shots_per_group shots: out[q * 5 + ..]. */
int spk_feasibility_residuals_batched(const double* coords, int64_t n_groups,
                                      int64_t shots_per_group, int n_s, int dims, double a,
                                      double b, int pin_idx, const double* pin_val, double* out,
                                      void* ws, size_t ws_bytes, spk_stream_t stream);

/* upsample_shots (optimizer.py:183-199): (n_shots, n_s, d) -> (n_shots, 2 n_s, d). */
int spk_upsample_shots(const double* in, double* out, int64_t n_shots, int n_s, int dims,
                       spk_stream_t stream);

/* ------------------------------------------------------- field-path attraction */

/* eval_attraction's interpolation path (attraction.py:116-308), fp64:
 * mode 0 = "consistent" (_cell_grad2/3), 1 = "smooth" (interpolated force grids).
 * pts (p, dims) f64; potential (2N+1)^d f64; force (dims, (2N+1)^d) f64 (mode 1).
 * vals [p] = interpolated potential, grad [p, dims] (NOT divided by p),
 * n_clamped (device int64, 1) = count of clamped samples. */
int spk_field_eval(const double* pts, int64_t p, int dims, const double* potential,
                   const double* force, int64_t grid_n, int mode, double* vals,
                   double* grad, int64_t* n_clamped, spk_stream_t stream);

/* ------------------------------------------------- treecode (repulsion backend "tree")
 *
 * Replaces the reference's CPU dual-tree FMM (repulsion.py:90-200, _treecode.py:77-471)
 * behind eval_repulsion_tree with a GPU particle-cluster treecode meeting the same
 * tree_precision contract (relative error of the cost and of the gradient l2 norm).
 * Pipeline (paper_2108_02991_b200/tree.py): keys -> sort -> gather -> host octree ->
 * leaf / group boxes -> host interaction lists -> P2M proxies -> eval.
 */

/* Morton keys of float4 positions in [-1, 1]^dims (21 bits per axis in 3D, 31 in 2D);
 * idx = 0..n-1.  keys: [n] u64, idx: [n] i32 (device). */
int spk_tree_keys(const void* pos, int64_t n, int dims, uint64_t* keys, int32_t* idx,
                  spk_stream_t stream);

/* Stable radix sort of (keys, idx) pairs (CUB).  Counterpart of build_tree's sort
 * (_treecode.py:77-170). */
size_t spk_tree_sort_workspace_bytes(int64_t n);
int spk_tree_sort(const uint64_t* keys_in, const int32_t* idx_in, uint64_t* keys_out,
                  int32_t* idx_out, int64_t n, int dims, void* ws, size_t ws_bytes,
                  spk_stream_t stream);

/* out[i] = {pos[perm[i]].xyz, weights ? weights[perm[i]] : 1}. */
int spk_tree_gather(const void* pos, const int32_t* perm, int64_t n, const float* weights,
                    void* out, spk_stream_t stream);

/* Tight boxes {min xyz, max xyz} of record ranges [begin[r], end[r]) -> box [n][6]. */
int spk_tree_boxes(const void* rec, int64_t n_ranges, const int64_t* begin,
                   const int64_t* end, int dims, float* box, spk_stream_t stream);

/* Octree over sorted keys on the GPU, level by level (build_tree, _treecode.py:77-170):
 * BFS node order, children contiguous in child-digit order, a node splits when it holds
 * more than leaf_cap particles (or more than one above level min_level) and is above the
 * finest level -- the same tree as spk_tree_host_build.  Device outputs node_begin/node_end [capacity] i64, first_child /
 * n_child [capacity] i32 (first_child -1 for leaves), leaf_node [capacity] i32; HOST
 * outputs level_off [64] (level l = nodes [off[l], off[l+1])) and counts [3] = nodes,
 * leaves, levels.  Returns SPK_ERR_WORKSPACE when node_capacity is too small (retry). */
size_t spk_tree_build_workspace_bytes(int64_t n, int64_t node_capacity);
int spk_tree_build(const uint64_t* keys, int64_t n, int dims, int64_t leaf_cap,
                   int min_level, int64_t node_capacity, int64_t* node_begin, int64_t* node_end,
                   int32_t* first_child, int32_t* n_child, int32_t* leaf_node,
                   int64_t* level_off, int64_t* counts, void* ws, size_t ws_bytes,
                   spk_stream_t stream);
/* Target groups of <= cap particles following the octree (spk_tree_host_groups),
 * sorted by first particle: grp_begin/grp_end [group_capacity] i64 (device), n_groups
 * HOST.  cut (optional, [n] u8): particles that must start a group (the first particles of
 * enclosing far-level parents), so that every group lies inside one parent.  Workspace: spk_tree_build_workspace_bytes(0, max(n_nodes, group_capacity)). */
int spk_tree_groups(const int64_t* node_begin, const int64_t* node_end,
                    const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                    int64_t cap, const uint8_t* cut, int64_t group_capacity,
                    int64_t* grp_begin, int64_t* grp_end, int64_t* n_groups, void* ws,
                    size_t ws_bytes, spk_stream_t stream);

/* Node boxes {min xyz, max xyz} of an octree over sorted records: leaves reduce their
 * particles, internal nodes (BFS levels, level_off is a HOST array of n_levels + 1
 * offsets) merge their children bottom-up.  node_box: [n_nodes][6] f32 (device). */
int spk_tree_node_boxes(const void* rec, int64_t n_nodes, const int32_t* first_child,
                        const int32_t* n_child, int64_t n_leaves, const int32_t* leaf_node,
                        const int64_t* leaf_begin, const int64_t* leaf_end, int64_t n_levels,
                        const int64_t* level_off, int dims, float* node_box,
                        spk_stream_t stream);

/* Interaction lists on the GPU (dual_traverse + group_by_target, _treecode.py:173-262):
 * one thread per target group walks the octree; a node is far when
 * r_group + r_node < theta |c_group - c_node| (box half-diagonals and centers).  Far
 * nodes with more than m = order^dims particles become proxy slots (node order), other
 * far nodes and opened leaves contribute their particle ranges (contiguous ranges merge).
 * Count pass: slot_of/slot_node [n_nodes] i32, slot_box [n_nodes][6] f32 (center, half),
 * slot_unit_off [n_nodes + 1] i64, seg_off [n_groups + 1] i64, totals [4] i64 = segments,
 * slots, P2M units, traversal-stack overflows (device; the lists are invalid unless
 * totals[3] == 0 -- the Python wrapper raises).  Write pass fills seg_start/seg_count and the P2M units.
 * Optional far level: parent_box [n_parents][6] and group_parent [n_groups]; nodes far
 * from a group's parent (same opening test) are skipped -- the parent's P2L/L2P covers
 * them; far_only = 1 emits far nodes only (the parents' own walk, for their P2L).
 * Sub-walks (plain traversal only, parent_box == NULL): with sub_off != NULL
 * ([n_groups * SPK_TREE_FRONT + 1] i64, filled by the count pass and passed unchanged to
 * the write pass) every group's walk runs as SPK_TREE_FRONT threads split at the tree's
 * second level (ranges merge only within one; spk_tree_host_plan follows that rule);
 * NULL = one thread per group. */
#define SPK_TREE_FRONT 64
size_t spk_tree_plan_workspace_bytes(int64_t n_nodes, int64_t n_groups);
int spk_tree_plan_count(const int64_t* node_begin, const int64_t* node_end,
                        const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                        const float* node_box, const float* group_box, int64_t n_groups,
                        double theta, int order, int dims, int64_t n_src, int32_t* slot_of,
                        int32_t* slot_node, float* slot_box, int64_t* slot_unit_off,
                        int64_t* seg_off, int64_t* totals, const float* parent_box,
                        const int32_t* group_parent, int far_only, int64_t* sub_off, void* ws,
                        size_t ws_bytes, spk_stream_t stream);
int spk_tree_plan_write(const int64_t* node_begin, const int64_t* node_end,
                        const int32_t* first_child, const int32_t* n_child, int64_t n_nodes,
                        const float* node_box, const float* group_box, int64_t n_groups,
                        double theta, int order, int dims, int64_t n_src,
                        const int32_t* slot_of, const int32_t* slot_node,
                        const int64_t* slot_unit_off, int64_t n_slots, const int64_t* seg_off,
                        int64_t* seg_start, int32_t* seg_count, int32_t* unit_slot,
                        int64_t* unit_begin, int64_t* unit_end, const float* parent_box,
                        const int32_t* group_parent, int far_only, const int64_t* sub_off,
                        spk_stream_t stream);

/* Far level (target-side interpolation, the m2l + l2p of _treecode.py:330-426): the
 * q^dims tensor Chebyshev points of every parent box (points [n_parents * q^dims] float4,
 * parent_cheb_box [n_parents][6] = center, inflated half), the parent of every sorted
 * target, and the L2P that adds the interpolated value / gradient (pval [n_parents *
 * q^dims], pgrad [.. x dims] fp64, evaluated at those points) to val / grad. */
int spk_tree_cheb_targets(const float* parent_box, int64_t n_parents, int order, int dims,
                          void* points, float* parent_cheb_box, spk_stream_t stream);
int spk_tree_parent_ids(const int64_t* parent_begin, const int64_t* parent_end,
                        int64_t n_parents, int32_t* pid, spk_stream_t stream);
int spk_tree_l2p(const void* tgt_sorted, const int32_t* tgt_perm, int64_t n_tgt,
                 const int32_t* pid, const float* parent_cheb_box, const double* pval,
                 const double* pgrad, int order, int dims, double* val, double* grad,
                 spk_stream_t stream);

/* Source-side Chebyshev interpolation (the P2M of _treecode.py:286-313 for a
 * particle-cluster scheme): proxies[slot * m + k] = {tensor Chebyshev point k of the
 * slot box, sum over the slot's particles of w * L_k(x)}, m = order^dims.  Units are
 * (slot, particle range) pieces, units of a slot contiguous (slot_unit_off). */
size_t spk_tree_p2m_workspace_bytes(int64_t n_units, int order, int dims);
int spk_tree_p2m(const void* rec, int64_t n_units, const int32_t* unit_slot,
                 const int64_t* unit_begin, const int64_t* unit_end, int64_t n_slots,
                 const int64_t* slot_unit_off, const float* slot_box, int order, int dims,
                 void* proxies, void* ws, size_t ws_bytes, spk_stream_t stream);

/* Weighted sums over segment lists (the m2l/l2p/near_field of _treecode.py:330-471 in
 * one pass): for target group g (sorted targets [grp_begin[g], grp_end[g]), at most
 * spk_tree_group_size() of them),
 *   val[perm[i]] = sum_{records r in g's segments} w_r sqrt(|t_i - r|^2 + eps2)
 *   grad[perm[i]] = sum w_r (t_i - r) / sqrt(...)
 * seg_off: [n_lists + 1]; seg_start (record offset into src), seg_count; grp_list
 * (optional): the list of each group (default: list g), so groups can share a list. */
int spk_tree_eval(const void* tgt_sorted, const int32_t* tgt_perm, int64_t n_groups,
                  const int64_t* grp_begin, const int64_t* grp_end, const int32_t* grp_list,
                  const void* src, const int64_t* seg_off, const int64_t* seg_start,
                  const int32_t* seg_count, int dims, float eps2, double* val, double* grad,
                  spk_stream_t stream);
int spk_tree_group_size(void);

/* Host side (tree_host.cpp; HOST pointers).  An opaque octree over sorted keys:
 * nodes in BFS order with contiguous children, leaves hold <= leaf_cap particles
 * (build_tree, _treecode.py:77-170).  Returns NULL on error (spk_last_error). */
void* spk_tree_host_build(const uint64_t* keys, int64_t n, int dims, int64_t leaf_cap,
                          int min_level);
void spk_tree_host_free(void* tree);
void spk_tree_host_sizes(const void* tree, int64_t* counts /* [2]: nodes, leaves */);
int64_t spk_tree_host_levels(const void* tree, int64_t* level_off);
void spk_tree_host_leaf_nodes(const void* tree, int32_t* leaf_node);
void spk_tree_host_leaves(const void* tree, int64_t* begin, int64_t* end);
void spk_tree_host_nodes(const void* tree, int64_t* begin, int64_t* end,
                         int32_t* first_child, int32_t* n_child, int32_t* level);
void spk_tree_host_set_leaf_boxes(void* tree, const float* leaf_box);
/* Target groups (<= cap consecutive sorted particles, packed along the octree); returns
 * the count, fills begin/end when non-NULL. */
int64_t spk_tree_host_groups(const void* tree, int64_t cap, int64_t* begin, int64_t* end);
/* Host reference planner (serial; same lists as spk_tree_plan_count/_write):
 * counts[5] = segments, proxy slots, P2M units, near pairs, far pairs. */
int spk_tree_host_plan(void* tree, int64_t n_groups, const float* group_box, double theta,
                       int order, int64_t n_src, int64_t* counts);
void spk_tree_host_slot_nodes(const void* tree, int32_t* slot_node);
void spk_tree_host_export_plan(const void* tree, int64_t* seg_off, int64_t* seg_start,
                               int32_t* seg_count, float* slot_box, int32_t* unit_slot,
                               int64_t* unit_begin, int64_t* unit_end,
                               int64_t* slot_unit_off);

/* ------------------------------------------------- analysis: direct NUDFT
 *
 * Replaces analysis.py:25-69 (per-axis phase tables + matrix products).  Points k are
 * fp64 [p][dims] in [-1, 1]; grid is a HOST array of dims sizes; voxel offsets are
 * r_a = 0..n_a-1 minus n_a/2.  Complex arrays are interleaved fp64 (re, im), grid arrays
 * row-major (C order).  mode SPK_NUDFT_FP64: fp64 tables and products (the reference's
 * numerics; density compensation needs them, see nudft.cu); SPK_NUDFT_MIXED: fp32
 * products with fp64 phase generation and accumulation (opt-in, ~2x faster).
 */
enum { SPK_NUDFT_FP64 = 0, SPK_NUDFT_MIXED = 1 };
size_t spk_nudft_workspace_bytes(int64_t p, int dims, const int64_t* grid);
/* out[r] = sum_i w_i exp(+i pi k_i . r)  (nudft_adjoint, analysis.py:41-55) */
int spk_nudft_adjoint(const double* pts, const double* weights, int64_t p, int dims,
                      const int64_t* grid, int mode, double* out, void* ws, size_t ws_bytes,
                      spk_stream_t stream);
/* out[i] = sum_r image[r] exp(-i pi k_i . r)  (nudft_forward, analysis.py:58-69) */
int spk_nudft_forward(const double* pts, const double* image, int64_t p, int dims,
                      const int64_t* grid, int mode, double* out, void* ws, size_t ws_bytes,
                      spk_stream_t stream);
/* w_i <- w_i / max(|back_i|, 1e-12)  (density_compensation, analysis.py:90-96) */
int spk_dcf_update(double* weights, const double* back, int64_t p, spk_stream_t stream);
/* mag[e] = |vol[e] / total|  (compute_psf, analysis.py:126-131) */
int spk_psf_magnitude(const double* vol, int64_t n, double total, double* mag,
                      spk_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARKLING_B200_H */
