"""GPU treecode for the repulsion sums (``RepulsionConfig(backend="tree")``).

The reference's tree backend is a CPU dual-tree Chebyshev FMM
(/root/reference/pkg/src/vdtraj/repulsion.py:90-200, _treecode.py:77-471) whose contract
is ``tree_precision`` relative error on the cost and on the gradient l2 norm against
direct summation.  This module keeps the contract with a particle-cluster treecode laid
out for the B200 (csrc/tree.cu, csrc/tree_host.cpp):

  1. GPU: Morton keys of the float4 positions, CUB radix sort, gather sorted records.
  2. GPU: octree over the sorted keys, level by level (BFS, contiguous children,
     <= LEAF_CAP per leaf), and target groups (<= 64 consecutive targets forming sibling
     subtrees); the serial host builder (tree_host.cpp) is the reference it is tested
     against.
  3. GPU: tight node boxes (leaves reduce, levels merge bottom-up) and group boxes.
  4. GPU: one thread per target group walks the octree -> segments of near particles and
     of far-node proxies (q^d tensor Chebyshev points on the node's box); count pass,
     one 32-byte read-back of the totals, write pass.
  5. GPU: P2M proxy weights; one warp per target group (<= 64 targets) sums the weighted
     kernel over its segments (packed f32x2 FMA + MUFU.RSQ, fp64 accumulation per
     256-record batch).

The (order, theta) table was calibrated on the B200 against the exact K1 kernel on the
SPARKLING distributions (profiles/r01_tree_calibration.jsonl): every row meets its
precision with margin on radial-spoke, perturbed and uniform clouds.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import _device, _native

# (precision floor, interpolation order, opening threshold) -- same role as the
# reference's _AUTO_PARAMS (repulsion.py:24-30), calibrated for this scheme on the B200
# (profiles/r01_tree_calibration.jsonl, r01_tree_att_calibration.jsonl): the worst
# gradient error over the C1, C2, C4, 3D-radial and uniform clouds, repulsion and lattice
# attraction, is at least 2.5x below the floor.  Below 1e-6 the fp32 pair arithmetic
# itself (~3e-7 vs fp64) is the limit: such precisions run the exact kernels.
AUTO_PARAMS = (
    (1e-2, 3, 0.8),
    (1e-3, 4, 0.7),
    (1e-4, 5, 0.7),
    (1e-5, 6, 0.7),
    (1e-6, 6, 0.5),
)
MAX_ORDER = 8
SUB_FRONT = 64  # frontier slots per group walk (sparkling_b200.h SPK_TREE_FRONT)
LEAF_CAP = 256  # source particles per octree leaf
# At or below this many sources the exact kernel is faster than building and walking a
# tree on the B200 (C1 32k: 0.4 vs 1.0 ms; 65k: 1.7 vs 2.5 ms; 1M: 362 vs 19 ms).
DIRECT_BELOW = 1 << 17
# Auto-mode probe cadence inside optimize(): a table row validated by the 64-target probe
# is reused for this many calls with the same sizes, then probed again (starting from the
# validated row) because the points move and can cluster within a level.
REPROBE_EVERY = 10


def cached_row(row_cache, key):
    """(row, reprobe): the validated table row for ``key`` while it is fresh (row, False);
    (row, True) when the re-probe is due (start probing at that row); (None, False) when
    nothing is cached."""
    if row_cache is None:
        return None, False
    entry = row_cache.get(key)
    if entry is None:
        return None, False
    entry[1] += 1
    if entry[1] < REPROBE_EVERY:
        return entry[0], False
    return entry[0], True


def store_row(row_cache, key, row):
    if row_cache is not None:
        row_cache[key] = [row, 0]
# Target octrees are split down to at least this level (cells of 1/16 of the domain):
# sparse targets (coarse decimation levels) would otherwise form groups spanning whole
# spokes, whose near field against the dense lattice is huge (131k targets against the
# C4 lattice: 45 -> 24 ms; no effect at 524k targets and above).
TARGET_MIN_LEVEL = 5
# Far level (P2L/L2P on parents of <= FAR_PARENT_CAP targets), used for the repulsion
# from this many targets on: in the optimizer's call path at C4 it cuts the repulsion
# evaluation from 118 to 91 ms (1e-3) and 186 to 138 ms (1e-4), incl. the per-call P2M
# of every node (profiles/r01_far_level.txt).  The lattice attraction keeps the plain
# walk (its q5 far level is not faster).  SPK_FAR_LEVEL_MIN overrides.
FAR_LEVEL_MIN = int(os.environ.get("SPK_FAR_LEVEL_MIN", str(1 << 22)))
FAR_PARENT_CAP = 1024


def far_parent_cap(n_targets: int) -> int | None:
    """Parent capacity of the far level for this many targets (None: plain treecode)."""
    return FAR_PARENT_CAP if n_targets >= FAR_LEVEL_MIN else None


# 2D rows: a q^2 proxy is cheap, and dense-centre 2D clouds (radius ~ u^2) need higher
# orders than the 3D table gives -- (6, 0.7) reached 2.2e-5 on them for the 1e-5 row
# (scripts/tree_calib2d.py, profiles/r01_tree_calib2d.jsonl; found by tests/test_gpu_fuzz).
# Worst gradient error over dense-centre radial (150k, 1M), uniform, clustered and 2D
# spoke clouds: 1.5e-4 / 2.2e-5 / 8.1e-7 / 5.0e-7 for the 1e-3 .. 1e-6 rows.
AUTO_PARAMS_2D = (
    (1e-2, 3, 0.8),
    (1e-3, 4, 0.7),
    (1e-4, 6, 0.7),
    (1e-5, 7, 0.6),
    (1e-6, 8, 0.6),
)


def auto_params(precision: float, dims: int = 3) -> tuple[int, float] | None:
    """(order, theta) for a precision, or None when only the exact kernel meets it."""
    for floor, order, theta in (AUTO_PARAMS_2D if dims == 2 else AUTO_PARAMS):
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


def _host_tree(lib, skeys: torch.Tensor, n: int, dims: int, leaf_cap: int,
               min_level: int = 0):
    keys_h = skeys.cpu().numpy()  # synchronises the stream
    tree = lib.spk_tree_host_build(keys_h.ctypes.data, n, dims, leaf_cap, min_level)
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


class _DeviceOctree:
    """Octree over sorted keys built on the GPU (spk_tree_build): node tables on the
    device, BFS level offsets on the host.  Same nodes as the host builder."""

    def __init__(self, keys: torch.Tensor, n: int, dims: int, leaf_cap: int,
                 min_level: int = 0):
        dev = keys.device
        st = _device.stream()
        cap = 16 * n // max(leaf_cap, 1) + 1024
        while True:
            self.nb = torch.empty(cap, dtype=torch.int64, device=dev)
            self.ne = torch.empty(cap, dtype=torch.int64, device=dev)
            self.fc = torch.empty(cap, dtype=torch.int32, device=dev)
            self.nc = torch.empty(cap, dtype=torch.int32, device=dev)
            self.leaves = torch.empty(cap, dtype=torch.int32, device=dev)
            self.levels = np.zeros(64, dtype=np.int64)
            counts = np.zeros(3, dtype=np.int64)
            ws = _device.workspace(_native.query("spk_tree_build_workspace_bytes", n, cap),
                                   "tree_build")
            try:
                _native.call("spk_tree_build", keys.data_ptr(), n, dims, leaf_cap, min_level,
                             cap,
                             self.nb.data_ptr(), self.ne.data_ptr(), self.fc.data_ptr(),
                             self.nc.data_ptr(), self.leaves.data_ptr(), self.levels.ctypes.data,
                             counts.ctypes.data, ws.data_ptr(), ws.numel(), st)
                break
            except _native.NativeError as exc:
                if "capacity" not in str(exc):
                    raise
                cap *= 2
        self.n_nodes, self.n_leaves, n_lv = (int(c) for c in counts)
        self.levels = self.levels[:n_lv + 1].copy()
        _native.add_launches(4 * n_lv + 5)  # per level: split, scan (2), link; + leaves
        self.nb, self.ne = self.nb[:self.n_nodes], self.ne[:self.n_nodes]
        self.fc, self.nc = self.fc[:self.n_nodes], self.nc[:self.n_nodes]
        self.leaves = self.leaves[:self.n_leaves]

    def groups(self, cap: int, cut: torch.Tensor | None = None):
        """Target groups (spk_tree_groups) -> device (begin, end) sorted by begin; ``cut``
        (u8 per particle) marks particles that must start a group."""
        dev = self.nb.device
        gcap = max(self.n_nodes * 8, int(self.ne[:1].item() // cap) * 4 + 1024)
        gb = torch.empty(gcap, dtype=torch.int64, device=dev)
        ge = torch.empty(gcap, dtype=torch.int64, device=dev)
        n_groups = np.zeros(1, dtype=np.int64)
        ws = _device.workspace(_native.query("spk_tree_build_workspace_bytes", 0,
                                             max(self.n_nodes, gcap)), "tree_groups")
        _native.call("spk_tree_groups", self.nb.data_ptr(), self.ne.data_ptr(),
                     self.fc.data_ptr(), self.nc.data_ptr(), self.n_nodes, cap,
                     _device.ptr(cut), gcap,
                     gb.data_ptr(), ge.data_ptr(), n_groups.ctypes.data, ws.data_ptr(),
                     ws.numel(), _device.stream())
        k = int(n_groups[0])
        return gb[:k], ge[:k]


class SourceTree:
    """Sources sorted along the Morton curve, their octree and tight node boxes, resident
    on the device.  ``weights`` (fp32 device, per source in input order) makes a weighted
    source set (the density lattice); None means unit weights (repulsion).

    ``keep_host`` keeps the host octree handle (``self.host``) for the tests' cross-check
    of the GPU planner; call :meth:`close` to free it."""

    def __init__(self, src4: torch.Tensor, dims: int, leaf_cap: int = LEAF_CAP,
                 weights: torch.Tensor | None = None, proxy_orders=(), keep_host=False):
        lib = _native.load()
        dev = src4.device
        st = _device.stream()
        self.dims, self.n = dims, src4.shape[0]
        self.keys, self.perm = _sort(src4, dims)
        octree = _DeviceOctree(self.keys, self.n, dims, leaf_cap)
        self.octree = octree
        self.host = None
        if keep_host:  # the serial host builder, for the tests' cross-checks
            self.host = _host_tree(lib, self.keys, self.n, dims, leaf_cap)
            self.tables = _node_tables(lib, self.host)
        self.n_nodes, self.n_leaves = octree.n_nodes, octree.n_leaves
        self.d_nb, self.d_ne, self.d_fc, self.d_nc, self.d_leaves = (
            octree.nb, octree.ne, octree.fc, octree.nc, octree.leaves)
        self.levels = octree.levels
        self._groups = None
        self.rec = torch.empty((self.n, 4), dtype=torch.float32, device=dev)
        _native.call("spk_tree_gather", src4.data_ptr(), self.perm.data_ptr(), self.n,
                     _device.ptr(weights), self.rec.data_ptr(), st)
        self.node_box = torch.empty((self.n_nodes, 6), dtype=torch.float32, device=dev)
        lb = self.d_nb[self.d_leaves.long()]
        le = self.d_ne[self.d_leaves.long()]
        lv = self.levels
        _native.call("spk_tree_node_boxes", self.rec.data_ptr(), self.n_nodes,
                     self.d_fc.data_ptr(), self.d_nc.data_ptr(), self.n_leaves,
                     self.d_leaves.data_ptr(), lb.data_ptr(), le.data_ptr(), lv.shape[0] - 1,
                     lv.ctypes.data, dims, self.node_box.data_ptr(), st)
        _native.add_launches(int(np.count_nonzero(np.diff(lv))))
        self._static = {}
        for q in proxy_orders:
            self.static_proxies(q)

    def groups(self):
        """Target groups of these particles used as targets (device begin, end)."""
        if self._groups is None:
            self._groups = self.octree.groups(_native.load().spk_tree_group_size())
        return self._groups

    def close(self):
        if self.host:
            _native.load().spk_tree_host_free(self.host)
            self.host = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def static_proxies(self, order: int):
        """Proxies of EVERY node holding more than order^d sources, computed once (for
        source sets that do not move, e.g. the density lattice).  Returns (records
        [n + slots * m] with the proxies after the sources, slot_of [n_nodes] i32)."""
        hit = self._static.get(order)
        if hit is not None:
            return hit
        dev = self.rec.device
        st = _device.stream()
        m = order ** self.dims
        T = {"nb": self.d_nb.cpu().numpy(), "ne": self.d_ne.cpu().numpy()}
        cnt = T["ne"] - T["nb"]
        eligible = cnt > m
        slot_of = np.where(eligible, np.cumsum(eligible) - 1, -1).astype(np.int32)
        nodes = np.nonzero(eligible)[0].astype(np.int32)
        n_slots = nodes.shape[0]
        rec = torch.empty((self.n + n_slots * m, 4), dtype=torch.float32, device=dev)
        rec[:self.n].copy_(self.rec)
        if n_slots:
            units = (cnt[nodes] + 4095) // 4096
            suo = np.concatenate([[0], np.cumsum(units)]).astype(np.int64)
            n_units = int(suo[-1])
            us = np.repeat(np.arange(n_slots, dtype=np.int32), units)
            ub = T["nb"][nodes][us] + 4096 * (np.arange(n_units) - suo[us])
            ue = np.minimum(ub + 4096, T["ne"][nodes][us])
            # slot boxes (center, inflated half) from the device node boxes
            nbox = self.node_box.cpu().numpy()[nodes]
            c = 0.5 * (nbox[:, :3] + nbox[:, 3:])
            h = 0.5 * (nbox[:, 3:] - nbox[:, :3])
            hmax = h[:, :self.dims].max(axis=1, keepdims=True)
            h = np.maximum(h, np.float32(1e-6) * hmax + np.float32(1e-30))
            if self.dims == 2:
                h[:, 2] = 1.0
            sbox = np.ascontiguousarray(np.concatenate([c, h], axis=1), dtype=np.float32)
            d_us, d_ub, d_ue, d_suo, d_sb = (_to_dev(a, dev) for a in (
                us, ub.astype(np.int64), ue.astype(np.int64), suo, sbox))
            ws = _device.workspace(_native.query("spk_tree_p2m_workspace_bytes", n_units,
                                                 order, self.dims), "tree_p2m")
            _native.call("spk_tree_p2m", rec.data_ptr(), n_units, d_us.data_ptr(),
                         d_ub.data_ptr(), d_ue.data_ptr(), n_slots, d_suo.data_ptr(),
                         d_sb.data_ptr(), order, self.dims, rec[self.n:].data_ptr(),
                         ws.data_ptr(), ws.numel(), st)
        hit = (rec, _to_dev(slot_of, dev))
        self._static[order] = hit
        return hit


class TargetGroups:
    """Targets sorted along the Morton curve and cut into groups of <= TR_GROUP that
    follow their octree (sibling subtrees), with tight group boxes (device)."""

    def __init__(self, tgt4: torch.Tensor, dims: int, same_as: SourceTree | None = None,
                 min_level: int = TARGET_MIN_LEVEL, parent_cap: int | None = None):
        lib = _native.load()
        dev = tgt4.device
        st = _device.stream()
        self.n = tgt4.shape[0]
        self.dims = dims
        group = lib.spk_tree_group_size()
        if same_as is not None:
            self.perm, self.rec = same_as.perm, same_as.rec
            octree = same_as.octree
        else:
            keys, self.perm = _sort(tgt4, dims)
            self.rec = torch.empty((self.n, 4), dtype=torch.float32, device=dev)
            _native.call("spk_tree_gather", tgt4.data_ptr(), self.perm.data_ptr(), self.n,
                         None, self.rec.data_ptr(), st)
            octree = _DeviceOctree(keys, self.n, dims, group, min_level)
        self.parents = None
        if parent_cap:
            # far level: parents of <= parent_cap targets; every group lies in one parent
            pb, pe = octree.groups(parent_cap)
            cut = torch.zeros(self.n + 1, dtype=torch.uint8, device=dev)
            cut[pb] = 1
            self.d_gb, self.d_ge = octree.groups(group, cut)
            self.n_parents = pb.shape[0]
            self.pbox = torch.empty((self.n_parents, 6), dtype=torch.float32, device=dev)
            _native.call("spk_tree_boxes", self.rec.data_ptr(), self.n_parents, pb.data_ptr(),
                         pe.data_ptr(), dims, self.pbox.data_ptr(), st)
            self.pid = torch.empty(self.n, dtype=torch.int32, device=dev)
            _native.call("spk_tree_parent_ids", pb.data_ptr(), pe.data_ptr(), self.n_parents,
                         self.pid.data_ptr(), st)
            self.gparent = self.pid[self.d_gb].contiguous()
            self.parents = (pb, pe)
        elif same_as is not None:
            self.d_gb, self.d_ge = same_as.groups()
        else:
            self.d_gb, self.d_ge = octree.groups(group)
        self.n_groups = self.d_gb.shape[0]
        self.box = torch.empty((self.n_groups, 6), dtype=torch.float32, device=dev)
        _native.call("spk_tree_boxes", self.rec.data_ptr(), self.n_groups, self.d_gb.data_ptr(),
                     self.d_ge.data_ptr(), dims, self.box.data_ptr(), st)


def _check_overflow(n: int) -> None:
    """The traversal stack bound holds for the Morton key depth (static_assert in
    tree.cu); a nonzero count would mean dropped subtrees, so fail instead of summing."""
    if n:
        raise _native.NativeError(f"tree plan: traversal stack overflow in {n} walks")


# Sub-walks pay while one thread per group leaves the GPU idle (a rank's Morton block,
# the coarse levels); with many groups the serial walks already fill it and the sub-walks'
# ancestor tests and 64x longer scans cost more (full3d level 6, 8.4M targets: plan
# passes 6.1 ms serial vs 20.6 ms sub-walks; 2k groups: 6.1 -> 2.1 ms;
# profiles/r02_tree_subwalk_phases.jsonl).
SUBWALK_MAX_GROUPS = 16384


def _sub_offsets(n_groups: int, dev) -> torch.Tensor | None:
    """Per-(group, frontier slot) list offsets of the sub-walk traversal (tree.cu
    traverse_sub_kernel), or None for the one-thread-per-group walk: sub-walks below
    SUBWALK_MAX_GROUPS groups; SPK_TREE_SUBWALK=0/1 forces either."""
    env = os.environ.get("SPK_TREE_SUBWALK")
    if env == "0" or (env is None and n_groups > SUBWALK_MAX_GROUPS):
        return None
    return torch.empty(n_groups * SUB_FRONT + 1, dtype=torch.int64, device=dev)


def _static_plan(src: SourceTree, boxes: torch.Tensor, n_groups: int, theta: float,
                 order: int, slot_of: torch.Tensor, pbox=None, gparent=None, far_only=False):
    """Interaction lists against the source tree's static (all-node) proxies."""
    dev = src.rec.device
    st = _device.stream()
    n_nodes = src.n_nodes
    tmp_i = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    tmp_n = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    tmp_b = torch.empty((n_nodes, 6), dtype=torch.float32, device=dev)
    tmp_u = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    seg_off = torch.empty(n_groups + 1, dtype=torch.int64, device=dev)
    totals = torch.empty(4, dtype=torch.int64, device=dev)
    ws = _device.workspace(_native.query("spk_tree_plan_workspace_bytes", n_nodes, n_groups),
                           "tree_plan")
    args = (src.d_nb.data_ptr(), src.d_ne.data_ptr(), src.d_fc.data_ptr(), src.d_nc.data_ptr(),
            n_nodes, src.node_box.data_ptr(), boxes.data_ptr(), n_groups, float(theta), order,
            src.dims, src.n)
    sub_off = None if pbox is not None else _sub_offsets(n_groups, dev)
    _native.call("spk_tree_plan_count", *args, tmp_i.data_ptr(), tmp_n.data_ptr(),
                 tmp_b.data_ptr(), tmp_u.data_ptr(), seg_off.data_ptr(), totals.data_ptr(),
                 _device.ptr(pbox), _device.ptr(gparent), int(far_only), _device.ptr(sub_off),
                 ws.data_ptr(), ws.numel(), st)
    if sub_off is not None:
        _native.add_launches(1)
    n_seg, _, _, overflow = (int(x) for x in totals.cpu().numpy())
    _check_overflow(overflow)
    seg_start = torch.empty(max(n_seg, 1), dtype=torch.int64, device=dev)
    seg_count = torch.empty(max(n_seg, 1), dtype=torch.int32, device=dev)
    _native.call("spk_tree_plan_write", *args, slot_of.data_ptr(), tmp_n.data_ptr(),
                 tmp_u.data_ptr(), 0, seg_off.data_ptr(), seg_start.data_ptr(),
                 seg_count.data_ptr(), tmp_i.data_ptr(), seg_off.data_ptr(),
                 seg_off.data_ptr(), _device.ptr(pbox), _device.ptr(gparent), int(far_only),
                 _device.ptr(sub_off), st)
    return seg_off, seg_start, seg_count, n_seg


def _far_level(tg: TargetGroups, src: SourceTree, order: int, far_order: int, theta: float,
               eps2: float, rec: torch.Tensor, slot_of: torch.Tensor):
    """P2L: every parent's far list evaluated at the far_order^d Chebyshev points of its
    box -> (parent Chebyshev boxes, values [P * mt], gradients [P * mt, d])."""
    dev = src.rec.device
    st = _device.stream()
    dims = src.dims
    n_par = tg.n_parents
    so, ss, sc, _ = _static_plan(src, tg.pbox, n_par, theta, order, slot_of, far_only=True)
    mt = far_order ** dims
    pts = torch.empty((n_par * mt, 4), dtype=torch.float32, device=dev)
    pcb = torch.empty((n_par, 6), dtype=torch.float32, device=dev)
    _native.call("spk_tree_cheb_targets", tg.pbox.data_ptr(), n_par, far_order, dims,
                 pts.data_ptr(), pcb.data_ptr(), st)
    group = _native.load().spk_tree_group_size()
    per = (mt + group - 1) // group
    j = torch.arange(per, device=dev, dtype=torch.int64)
    base = torch.arange(n_par, device=dev, dtype=torch.int64)[:, None] * mt
    gb = (base + j[None, :] * group).reshape(-1)
    ge = torch.minimum(gb + group, (base + mt).expand(-1, per).reshape(-1))
    glist = torch.arange(n_par, device=dev, dtype=torch.int32).repeat_interleave(per)
    ident = torch.arange(n_par * mt, device=dev, dtype=torch.int32)
    pval = torch.empty(n_par * mt, dtype=torch.float64, device=dev)
    pgrad = torch.empty((n_par * mt, dims), dtype=torch.float64, device=dev)
    _native.call("spk_tree_eval", pts.data_ptr(), ident.data_ptr(), gb.shape[0], gb.data_ptr(),
                 ge.data_ptr(), glist.data_ptr(), rec.data_ptr(), so.data_ptr(), ss.data_ptr(),
                 sc.data_ptr(), dims, float(eps2), pval.data_ptr(), pgrad.data_ptr(), st)
    return pcb, pval, pgrad


def tree_eval(tg: TargetGroups, src: SourceTree, order: int, theta: float, eps2: float, *,
              static: bool = False, stats: dict | None = None, lists: dict | None = None,
              val: torch.Tensor | None = None, grad: torch.Tensor | None = None,
              far_order: int | None = None, far: bool = True):
    """Weighted treecode sums of the sources at the targets -> (val, grad) fp64, targets'
    original order.  ``static`` uses the source tree's cached all-node proxies (no P2M in
    the call); otherwise proxies are built for the nodes this traversal opens as far.
    With a far level (``tg`` built with ``parent_cap``), nodes far from a target's parent
    are evaluated at the parent's far_order^d Chebyshev points and interpolated (P2L/L2P);
    the groups' lists then hold only the remaining nodes (static proxies); ``far=False``
    ignores the parents (the groups are valid plain groups either way)."""
    if not 2 <= order <= MAX_ORDER:
        raise ValueError(f"interp_order must be in [2, {MAX_ORDER}]")
    if far and tg.parents is not None:
        return _tree_eval_far(tg, src, order, theta, eps2, far_order or order, val, grad)
    dev = src.rec.device
    st = _device.stream()
    dims, n_s, m = src.dims, src.n, order ** src.dims
    n_nodes, n_groups = src.n_nodes, tg.n_groups
    timing = stats is not None and stats.get("timing", False)
    marks = []

    def mark(name):
        if timing:
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))

    mark("start")
    slot_of = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    slot_node = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    slot_box = torch.empty((n_nodes, 6), dtype=torch.float32, device=dev)
    slot_unit_off = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    seg_off = torch.empty(n_groups + 1, dtype=torch.int64, device=dev)
    totals = torch.empty(4, dtype=torch.int64, device=dev)
    sub_off = _sub_offsets(n_groups, dev)
    ws = _device.workspace(_native.query("spk_tree_plan_workspace_bytes", n_nodes, n_groups),
                           "tree_plan")
    _native.call("spk_tree_plan_count", src.d_nb.data_ptr(), src.d_ne.data_ptr(),
                 src.d_fc.data_ptr(), src.d_nc.data_ptr(), n_nodes, src.node_box.data_ptr(),
                 tg.box.data_ptr(), n_groups, float(theta), order, dims, n_s,
                 slot_of.data_ptr(), slot_node.data_ptr(), slot_box.data_ptr(),
                 slot_unit_off.data_ptr(), seg_off.data_ptr(), totals.data_ptr(), None, None,
                 0, _device.ptr(sub_off), ws.data_ptr(), ws.numel(), st)
    if sub_off is not None:
        _native.add_launches(1)
    n_seg, n_slots, n_units, overflow = (int(x) for x in totals.cpu().numpy())
    _check_overflow(overflow)
    mark("plan_count")
    if static:
        rec, write_slot_of = src.static_proxies(order)
        n_units_w = 0
    else:
        rec = torch.empty((n_s + n_slots * m, 4), dtype=torch.float32, device=dev)
        rec[:n_s].copy_(src.rec)
        write_slot_of = slot_of
        n_units_w = n_units
    seg_start = torch.empty(max(n_seg, 1), dtype=torch.int64, device=dev)
    seg_count = torch.empty(max(n_seg, 1), dtype=torch.int32, device=dev)
    unit_slot = torch.empty(max(n_units_w, 1), dtype=torch.int32, device=dev)
    unit_begin = torch.empty(max(n_units_w, 1), dtype=torch.int64, device=dev)
    unit_end = torch.empty(max(n_units_w, 1), dtype=torch.int64, device=dev)
    _native.call("spk_tree_plan_write", src.d_nb.data_ptr(), src.d_ne.data_ptr(),
                 src.d_fc.data_ptr(), src.d_nc.data_ptr(), n_nodes, src.node_box.data_ptr(),
                 tg.box.data_ptr(), n_groups, float(theta), order, dims, n_s,
                 write_slot_of.data_ptr(), slot_node.data_ptr(), slot_unit_off.data_ptr(),
                 0 if static else n_slots, seg_off.data_ptr(), seg_start.data_ptr(),
                 seg_count.data_ptr(), unit_slot.data_ptr(), unit_begin.data_ptr(),
                 unit_end.data_ptr(), None, None, 0, _device.ptr(sub_off), st)
    mark("plan_write")
    if not static and n_slots:
        ws2 = _device.workspace(_native.query("spk_tree_p2m_workspace_bytes", n_units, order,
                                              dims), "tree_p2m")
        _native.call("spk_tree_p2m", rec.data_ptr(), n_units, unit_slot.data_ptr(),
                     unit_begin.data_ptr(), unit_end.data_ptr(), n_slots,
                     slot_unit_off.data_ptr(), slot_box.data_ptr(), order, dims,
                     rec[n_s:].data_ptr(), ws2.data_ptr(), ws2.numel(), st)
    mark("p2m")
    if val is None:
        val = torch.empty(tg.n, dtype=torch.float64, device=dev)
    if grad is None:
        grad = torch.empty((tg.n, dims), dtype=torch.float64, device=dev)
    _native.call("spk_tree_eval", tg.rec.data_ptr(), tg.perm.data_ptr(), n_groups,
                 tg.d_gb.data_ptr(), tg.d_ge.data_ptr(), None, rec.data_ptr(),
                 seg_off.data_ptr(), seg_start.data_ptr(), seg_count.data_ptr(), dims,
                 float(eps2), val.data_ptr(), grad.data_ptr(), st)
    mark("eval")
    if timing:
        stats["eval_phases_ms"] = {marks[i][0]: 1e3 * (marks[i][1] - marks[i - 1][1])
                                   for i in range(1, len(marks))}
    if stats is not None:
        so = seg_off.cpu().numpy()
        sc = seg_count[:n_seg].cpu().numpy().astype(np.int64)
        per_group = np.add.reduceat(np.append(sc, 0), np.minimum(so[:-1], n_seg)) * \
            (so[1:] > so[:-1])
        sizes = (tg.d_ge - tg.d_gb).cpu().numpy()
        ss = seg_start[:n_seg].cpu().numpy()
        near = np.add.reduceat(np.append(np.where(ss < n_s, sc, 0), 0),
                               np.minimum(so[:-1], n_seg)) * (so[1:] > so[:-1])
        stats.update(nodes=n_nodes, leaves=src.n_leaves, groups=n_groups, segments=n_seg,
                     slots=n_slots, units=n_units, interp_order=order, opening_theta=theta,
                     pairs=int(np.dot(per_group, sizes)),
                     near_pairs=int(np.dot(near, sizes)))
    if lists is not None:
        lists.update(seg_off=seg_off.cpu().numpy(), seg_start=seg_start[:n_seg].cpu().numpy(),
                     seg_count=seg_count[:n_seg].cpu().numpy(),
                     slot_node=slot_node[:n_slots].cpu().numpy(),
                     node_box=src.node_box.cpu().numpy(), group_box=tg.box.cpu().numpy(),
                     n_groups=n_groups, n_src=n_s)
    return val, grad


def _tree_eval_far(tg, src, order, theta, eps2, far_order, val, grad):
    dev = src.rec.device
    st = _device.stream()
    dims = src.dims
    rec, slot_of = src.static_proxies(order)
    pcb, pval, pgrad = _far_level(tg, src, order, far_order, theta, eps2, rec, slot_of)
    so, ss, sc, _ = _static_plan(src, tg.box, tg.n_groups, theta, order, slot_of,
                                 tg.pbox, tg.gparent)
    if val is None:
        val = torch.empty(tg.n, dtype=torch.float64, device=dev)
    if grad is None:
        grad = torch.empty((tg.n, dims), dtype=torch.float64, device=dev)
    _native.call("spk_tree_eval", tg.rec.data_ptr(), tg.perm.data_ptr(), tg.n_groups,
                 tg.d_gb.data_ptr(), tg.d_ge.data_ptr(), None, rec.data_ptr(), so.data_ptr(),
                 ss.data_ptr(), sc.data_ptr(), dims, float(eps2), val.data_ptr(),
                 grad.data_ptr(), st)
    _native.call("spk_tree_l2p", tg.rec.data_ptr(), tg.perm.data_ptr(), tg.n, tg.pid.data_ptr(),
                 pcb.data_ptr(), pval.data_ptr(), pgrad.data_ptr(), far_order, dims,
                 val.data_ptr(), grad.data_ptr(), st)
    return val, grad


def tree_sums_device(tgt4: torch.Tensor, src4: torch.Tensor, dims: int, eps2: float,
                     order: int, theta: float, *, leaf_cap: int = LEAF_CAP,
                     stats: dict | None = None, lists: dict | None = None):
    """Treecode approximation of ``direct_sums_device(tgt4, src4, ...)`` -> (val, grad)
    fp64 on the device, in the targets' original order (unit-weight sources, proxies
    built for this call).

    ``stats`` (optional dict) receives the tree / list sizes; with ``stats["timing"] =
    True`` also per-phase wall times (synchronising between phases).  ``lists``
    (optional dict) receives the device interaction lists and, under "host_tree", the
    host octree (handle, tables) for the tests' cross-check (caller frees the handle)."""
    if not 2 <= order <= MAX_ORDER:
        raise ValueError(f"interp_order must be in [2, {MAX_ORDER}]")
    timing = stats is not None and stats.get("timing", False)
    marks = []

    def mark(name):
        if timing:
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))

    same = tgt4.data_ptr() == src4.data_ptr() and tgt4.shape[0] == src4.shape[0]
    mark("start")
    src = SourceTree(src4, dims, leaf_cap, keep_host=lists is not None)
    mark("build")
    tg = TargetGroups(tgt4, dims, same_as=src if same else None)
    mark("boxes")
    val, grad = tree_eval(tg, src, order, theta, eps2, stats=stats, lists=lists)
    mark("eval")
    if lists is not None:
        lists["host_tree"] = (src.host, src.tables)
        src.host = None  # ownership passes to the caller
    if timing:
        stats["phases_ms"] = {marks[i][0]: 1e3 * (marks[i][1] - marks[i - 1][1])
                              for i in range(1, len(marks))}
    return val, grad
