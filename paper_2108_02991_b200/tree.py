"""GPU treecode for the repulsion sums (``RepulsionConfig(backend="tree")``).

The reference's tree backend is a CPU dual-tree Chebyshev FMM
(/root/reference/pkg/src/vdtraj/repulsion.py:90-200, _treecode.py:77-471) whose contract
is ``tree_precision`` relative error on the cost and on the gradient l2 norm against
direct summation.  This module keeps the contract with a particle-cluster treecode laid
out for the B200 (csrc/tree.cu, csrc/tree_host.cpp):

  1. GPU: Morton keys of the float4 positions, CUB radix sort, gather sorted records.
  2. host: octree over the sorted keys (BFS, contiguous children, <= LEAF_CAP per leaf)
     and target groups (<= TR_GROUP consecutive targets forming sibling subtrees).
  3. GPU: tight node boxes (leaves reduce, levels merge bottom-up) and group boxes.
  4. GPU: one thread per target group walks the octree -> segments of near particles and
     of far-node proxies (q^d tensor Chebyshev points on the node's box); count pass,
     one 24-byte read-back of the totals, write pass.
  5. GPU: P2M proxy weights; one CTA per target group sums the weighted kernel over its
     segments (packed f32x2 FMA + MUFU.RSQ, fp64 accumulation per 512-record batch).

The (order, theta) table was calibrated on the B200 against the exact K1 kernel on the
SPARKLING distributions (profiles/r01_tree_calibration.jsonl): every row meets its
precision with margin on radial-spoke, perturbed and uniform clouds.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _native

# (precision floor, interpolation order, opening threshold) -- same role as the
# reference's _AUTO_PARAMS (repulsion.py:24-30), calibrated for this scheme on the B200
# (profiles/r01_tree_calibration.jsonl: worst gradient error over the C1, C2, 3D-radial
# and uniform clouds is at least 1.9x below the floor).  Below 1e-6 the fp32 pair
# arithmetic itself (~3e-7 vs fp64) is the limit: such precisions run the exact kernel.
AUTO_PARAMS = (
    (1e-2, 3, 0.8),
    (1e-3, 4, 0.8),
    (1e-4, 5, 0.8),
    (1e-5, 6, 0.7),
    (1e-6, 6, 0.5),
)
MAX_ORDER = 8
LEAF_CAP = 256  # source particles per octree leaf
# At or below this many sources the exact kernel is faster than building and walking a
# tree on the B200 (C1 32k: 0.4 vs 1.0 ms; 65k: 1.7 vs 2.5 ms; 1M: 362 vs 19 ms).
DIRECT_BELOW = 1 << 17


def auto_params(precision: float) -> tuple[int, float] | None:
    """(order, theta) for a precision, or None when only the exact kernel meets it."""
    for floor, order, theta in AUTO_PARAMS:
        if precision >= floor:
            return order, theta
    return None


def _to_dev(arr: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev)


def _sort(pos4: torch.Tensor, dims: int):
    n = pos4.shape[0]
    dev = pos4.device
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    skeys = torch.empty_like(keys)
    sidx = torch.empty_like(idx)
    st = _device.stream()
    _native.call("spk_tree_keys", pos4.data_ptr(), n, dims, keys.data_ptr(), idx.data_ptr(), st)
    ws = _device.workspace(_native.query("spk_tree_sort_workspace_bytes", n), "tree_sort")
    _native.call("spk_tree_sort", keys.data_ptr(), idx.data_ptr(), skeys.data_ptr(),
                 sidx.data_ptr(), n, dims, ws.data_ptr(), ws.numel(), st)
    return skeys, sidx


def _host_tree(lib, skeys: torch.Tensor, n: int, dims: int, leaf_cap: int):
    keys_h = skeys.cpu().numpy()  # synchronises the stream
    tree = lib.spk_tree_host_build(keys_h.ctypes.data, n, dims, leaf_cap)
    if not tree:
        raise _native.NativeError(lib.spk_last_error().decode())
    return tree


def _groups(lib, tree, cap: int):
    n_groups = int(lib.spk_tree_host_groups(tree, cap, None, None))
    gb = np.empty(n_groups, dtype=np.int64)
    ge = np.empty(n_groups, dtype=np.int64)
    lib.spk_tree_host_groups(tree, cap, gb.ctypes.data, ge.ctypes.data)
    return gb, ge


def _node_tables(lib, tree):
    sizes = np.zeros(2, dtype=np.int64)
    lib.spk_tree_host_sizes(tree, sizes.ctypes.data)
    n_nodes, n_leaves = int(sizes[0]), int(sizes[1])
    nb = np.empty(n_nodes, dtype=np.int64)
    ne = np.empty(n_nodes, dtype=np.int64)
    fc = np.empty(n_nodes, dtype=np.int32)
    nc = np.empty(n_nodes, dtype=np.int32)
    lib.spk_tree_host_nodes(tree, nb.ctypes.data, ne.ctypes.data, fc.ctypes.data,
                            nc.ctypes.data, None)
    leaves = np.empty(n_leaves, dtype=np.int32)
    lib.spk_tree_host_leaf_nodes(tree, leaves.ctypes.data)
    n_lv = int(lib.spk_tree_host_levels(tree, None))
    lv = np.empty(n_lv + 1, dtype=np.int64)
    lib.spk_tree_host_levels(tree, lv.ctypes.data)
    return dict(nb=nb, ne=ne, fc=fc, nc=nc, leaves=leaves, levels=lv)


def tree_sums_device(tgt4: torch.Tensor, src4: torch.Tensor, dims: int, eps2: float,
                     order: int, theta: float, *, leaf_cap: int = LEAF_CAP,
                     stats: dict | None = None, lists: dict | None = None):
    """Treecode approximation of ``direct_sums_device(tgt4, src4, ...)`` -> (val, grad)
    fp64 on the device, in the targets' original order.

    ``stats`` (optional dict) receives the tree / list sizes; with ``stats["timing"] =
    True`` also per-phase wall times (synchronising between phases).  ``lists``
    (optional dict) receives the device interaction lists and the host planner's lists
    for the same tree (tests)."""
    import time

    if not 2 <= order <= MAX_ORDER:
        raise ValueError(f"interp_order must be in [2, {MAX_ORDER}]")
    lib = _native.load()
    dev = src4.device
    st = _device.stream()
    n_s, n_t = src4.shape[0], tgt4.shape[0]
    same = tgt4.data_ptr() == src4.data_ptr() and n_t == n_s
    m = order ** dims
    group = lib.spk_tree_group_size()
    timing = stats is not None and stats.get("timing", False)
    marks = []

    def mark(name):
        if timing:
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))

    mark("start")
    # 1. sort sources (and targets), host octree(s) over the sorted keys
    skeys, sperm = _sort(src4, dims)
    tree = _host_tree(lib, skeys, n_s, dims, leaf_cap)
    ttree = None
    try:
        T = _node_tables(lib, tree)
        if same:
            gb, ge = _groups(lib, tree, group)
        else:
            tkeys, tperm = _sort(tgt4, dims)
            ttree = _host_tree(lib, tkeys, n_t, dims, group)
            gb, ge = _groups(lib, ttree, group)
        if lists is not None:
            lists["host_tree"] = (tree, T)
            tree = None  # the caller frees it
    finally:
        if tree:
            lib.spk_tree_host_free(tree)
        if ttree:
            lib.spk_tree_host_free(ttree)
    mark("build")
    n_nodes, n_leaves, n_groups = T["nb"].shape[0], T["leaves"].shape[0], gb.shape[0]
    d_nb, d_ne, d_fc, d_nc, d_leaves, d_gb, d_ge = (_to_dev(a, dev) for a in (
        T["nb"], T["ne"], T["fc"], T["nc"], T["leaves"], gb, ge))
    d_lb = d_nb[d_leaves.long()]
    d_le = d_ne[d_leaves.long()]
    # 2. sorted records; proxies go after the n_s particles (at most one slot per node)
    rec = torch.empty((n_s + n_nodes * m, 4), dtype=torch.float32, device=dev)
    _native.call("spk_tree_gather", src4.data_ptr(), sperm.data_ptr(), n_s, None,
                 rec.data_ptr(), st)
    if same:
        tperm, trec = sperm, rec
    else:
        trec = torch.empty((n_t, 4), dtype=torch.float32, device=dev)
        _native.call("spk_tree_gather", tgt4.data_ptr(), tperm.data_ptr(), n_t, None,
                     trec.data_ptr(), st)
    # 3. node boxes (leaves reduce, levels merge) and target group boxes
    node_box = torch.empty((n_nodes, 6), dtype=torch.float32, device=dev)
    lv = T["levels"]
    _native.call("spk_tree_node_boxes", rec.data_ptr(), n_nodes, d_fc.data_ptr(),
                 d_nc.data_ptr(), n_leaves, d_leaves.data_ptr(), d_lb.data_ptr(),
                 d_le.data_ptr(), lv.shape[0] - 1, lv.ctypes.data, dims, node_box.data_ptr(), st)
    _native.add_launches(int(np.count_nonzero(np.diff(lv))))
    group_box = torch.empty((n_groups, 6), dtype=torch.float32, device=dev)
    _native.call("spk_tree_boxes", trec.data_ptr(), n_groups, d_gb.data_ptr(), d_ge.data_ptr(),
                 dims, group_box.data_ptr(), st)
    mark("boxes")
    # 4. interaction lists on the device: count pass, sizes to the host, write pass
    slot_of = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    slot_node = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    slot_box = torch.empty((n_nodes, 6), dtype=torch.float32, device=dev)
    slot_unit_off = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    seg_off = torch.empty(n_groups + 1, dtype=torch.int64, device=dev)
    totals = torch.empty(3, dtype=torch.int64, device=dev)
    ws = _device.workspace(_native.query("spk_tree_plan_workspace_bytes", n_nodes, n_groups),
                           "tree_plan")
    _native.call("spk_tree_plan_count", d_nb.data_ptr(), d_ne.data_ptr(), d_fc.data_ptr(),
                 d_nc.data_ptr(), n_nodes, node_box.data_ptr(), group_box.data_ptr(), n_groups,
                 float(theta), order, dims, n_s, slot_of.data_ptr(), slot_node.data_ptr(),
                 slot_box.data_ptr(), slot_unit_off.data_ptr(), seg_off.data_ptr(),
                 totals.data_ptr(), ws.data_ptr(), ws.numel(), st)
    n_seg, n_slots, n_units = (int(x) for x in totals.cpu().numpy())
    seg_start = torch.empty(max(n_seg, 1), dtype=torch.int64, device=dev)
    seg_count = torch.empty(max(n_seg, 1), dtype=torch.int32, device=dev)
    unit_slot = torch.empty(max(n_units, 1), dtype=torch.int32, device=dev)
    unit_begin = torch.empty(max(n_units, 1), dtype=torch.int64, device=dev)
    unit_end = torch.empty(max(n_units, 1), dtype=torch.int64, device=dev)
    _native.call("spk_tree_plan_write", d_nb.data_ptr(), d_ne.data_ptr(), d_fc.data_ptr(),
                 d_nc.data_ptr(), n_nodes, node_box.data_ptr(), group_box.data_ptr(), n_groups,
                 float(theta), order, dims, n_s, slot_of.data_ptr(), slot_node.data_ptr(),
                 slot_unit_off.data_ptr(), n_slots, seg_off.data_ptr(), seg_start.data_ptr(),
                 seg_count.data_ptr(), unit_slot.data_ptr(), unit_begin.data_ptr(),
                 unit_end.data_ptr(), st)
    mark("plan")
    # 5. proxies (P2M) and the weighted sums
    if n_slots:
        ws2 = _device.workspace(_native.query("spk_tree_p2m_workspace_bytes", n_units, order,
                                              dims), "tree_p2m")
        _native.call("spk_tree_p2m", rec.data_ptr(), n_units, unit_slot.data_ptr(),
                     unit_begin.data_ptr(), unit_end.data_ptr(), n_slots,
                     slot_unit_off.data_ptr(), slot_box.data_ptr(), order, dims,
                     rec[n_s:].data_ptr(), ws2.data_ptr(), ws2.numel(), st)
    mark("p2m")
    val = torch.empty(n_t, dtype=torch.float64, device=dev)
    grad = torch.empty((n_t, dims), dtype=torch.float64, device=dev)
    _native.call("spk_tree_eval", trec.data_ptr(), tperm.data_ptr(), n_groups, d_gb.data_ptr(),
                 d_ge.data_ptr(), rec.data_ptr(), seg_off.data_ptr(), seg_start.data_ptr(),
                 seg_count.data_ptr(), dims, float(eps2), val.data_ptr(), grad.data_ptr(), st)
    mark("eval")
    if stats is not None:
        so = seg_off.cpu().numpy()
        sc = seg_count[:n_seg].cpu().numpy().astype(np.int64)
        per_group = np.add.reduceat(np.append(sc, 0), np.minimum(so[:-1], n_seg)) * (so[1:] > so[:-1])
        stats.update(nodes=n_nodes, leaves=n_leaves, groups=n_groups, segments=n_seg,
                     slots=n_slots, units=n_units, interp_order=order, opening_theta=theta,
                     pairs=int(np.dot(per_group, ge - gb)))
        if timing:
            stats["phases_ms"] = {marks[i][0]: 1e3 * (marks[i][1] - marks[i - 1][1])
                                  for i in range(1, len(marks))}
    if lists is not None:
        lists.update(seg_off=seg_off.cpu().numpy(), seg_start=seg_start[:n_seg].cpu().numpy(),
                     seg_count=seg_count[:n_seg].cpu().numpy(),
                     slot_node=slot_node[:n_slots].cpu().numpy(),
                     node_box=node_box.cpu().numpy(), group_box=group_box.cpu().numpy(),
                     n_groups=n_groups, n_src=n_s)
    return val, grad
