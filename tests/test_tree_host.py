"""Host half of the treecode (csrc/tree_host.cpp), no GPU: octree over sorted Morton
keys, target groups and interaction lists.  Structural invariants: the nodes partition
the sorted range level by level, leaves respect the capacity, groups tile the targets
in order, and every group's list covers every source exactly once (near particle ranges
plus far nodes) -- the completeness property the reference's dual_traverse guarantees
(_treecode.py:173-244) -- and contiguous ranges merge only within a second-level
subtree, as the device's sub-walks do."""

import numpy as np
import pytest

from paper_2108_02991_b200 import _native


def spread(v, dims):
    x = v.astype(np.uint64)
    out = np.zeros_like(x)
    bits = 21 if dims == 3 else 31
    for b in range(bits):
        out |= ((x >> np.uint64(b)) & np.uint64(1)) << np.uint64(dims * b)
    return out


def morton(pts):
    dims = pts.shape[1]
    bits = 21 if dims == 3 else 31
    q = np.clip(np.floor((pts.astype(np.float64) + 1) * 0.5 * (1 << bits)), 0,
                (1 << bits) - 1).astype(np.uint64)
    key = np.zeros(len(pts), dtype=np.uint64)
    for a in range(dims):
        key |= spread(q[:, a], dims) << np.uint64(dims - 1 - a)
    return key


def boxes(sp, b, e):
    out = np.empty((len(b), 6), np.float32)
    for i, (x, y) in enumerate(zip(b, e)):
        out[i, :3] = 0
        out[i, 3:] = 0
        out[i, :sp.shape[1]] = sp[x:y].min(0)
        out[i, 3:3 + sp.shape[1]] = sp[x:y].max(0)
    return np.ascontiguousarray(out)


@pytest.mark.parametrize("dims", [2, 3])
def test_tree_groups_and_lists_cover_every_source_once(dims):
    lib = _native.load()
    rng = np.random.default_rng(dims)
    n = 40000
    pts = np.concatenate([rng.uniform(-1, 1, (n // 2, dims)),
                          rng.normal(0, 0.05, (n // 2, dims)).clip(-1, 1)]).astype(np.float32)
    pts[:50] = pts[50]  # duplicates
    keys = morton(pts)
    order = np.argsort(keys, kind="stable")
    sk = np.ascontiguousarray(keys[order])
    sp = pts[order]
    cap = 64
    tree = lib.spk_tree_host_build(sk.ctypes.data, n, dims, cap, 0)
    try:
        sizes = np.zeros(2, np.int64)
        lib.spk_tree_host_sizes(tree, sizes.ctypes.data)
        nn, nl = (int(x) for x in sizes)
        beg = np.empty(nn, np.int64)
        end = np.empty(nn, np.int64)
        fc = np.empty(nn, np.int32)
        nc = np.empty(nn, np.int32)
        lv = np.empty(nn, np.int32)
        lib.spk_tree_host_nodes(tree, beg.ctypes.data, end.ctypes.data, fc.ctypes.data,
                                nc.ctypes.data, lv.ctypes.data)
        assert beg[0] == 0 and end[0] == n
        for v in np.nonzero(nc)[0]:
            ch = np.arange(fc[v], fc[v] + nc[v])
            assert beg[ch[0]] == beg[v] and end[ch[-1]] == end[v]
            assert np.array_equal(end[ch[:-1]], beg[ch[1:]])
            assert np.all(lv[ch] == lv[v] + 1)
        leaves = np.nonzero(nc == 0)[0]
        assert len(leaves) == nl
        big = end[leaves] - beg[leaves] > cap
        assert np.all(lv[leaves][big] == (21 if dims == 3 else 31))  # only duplicates
        lb = np.empty(nl, np.int64)
        le = np.empty(nl, np.int64)
        lib.spk_tree_host_leaves(tree, lb.ctypes.data, le.ctypes.data)
        leaf_box = boxes(sp, lb, le)
        lib.spk_tree_host_set_leaf_boxes(tree, leaf_box.ctypes.data)
        group = 256
        ng = lib.spk_tree_host_groups(tree, group, None, None)
        gb = np.empty(ng, np.int64)
        ge = np.empty(ng, np.int64)
        lib.spk_tree_host_groups(tree, group, gb.ctypes.data, ge.ctypes.data)
        assert gb[0] == 0 and ge[-1] == n and np.array_equal(ge[:-1], gb[1:])
        assert np.all(ge - gb <= group) and np.all(ge > gb)
        order_q = 4
        m = order_q ** dims
        counts = np.zeros(5, np.int64)
        group_box = boxes(sp, gb, ge)
        assert lib.spk_tree_host_plan(tree, ng, group_box.ctypes.data, 0.6, order_q,
                                      n, counts.ctypes.data) == 0
        n_seg, n_slots, n_units = (int(c) for c in counts[:3])
        assert n_slots > 0
        seg_off = np.empty(ng + 1, np.int64)
        seg_start = np.empty(n_seg, np.int64)
        seg_count = np.empty(n_seg, np.int32)
        slot_box = np.empty((n_slots, 6), np.float32)
        us = np.empty(n_units, np.int32)
        ub = np.empty(n_units, np.int64)
        ue = np.empty(n_units, np.int64)
        suo = np.empty(n_slots + 1, np.int64)
        lib.spk_tree_host_export_plan(tree, seg_off.ctypes.data, seg_start.ctypes.data,
                                      seg_count.ctypes.data, slot_box.ctypes.data,
                                      us.ctypes.data, ub.ctypes.data, ue.ctypes.data,
                                      suo.ctypes.data)
        slot_node = np.empty(n_slots, np.int32)
        lib.spk_tree_host_slot_nodes(tree, slot_node.ctypes.data)
        # P2M units tile every proxy node's particle range
        for s in range(n_slots):
            u = np.arange(suo[s], suo[s + 1])
            v = slot_node[s]
            assert ub[u[0]] == beg[v] and ue[u[-1]] == end[v]
            assert np.all(us[u] == s)
        # every group's segments cover each source exactly once
        for g in range(0, ng, max(1, ng // 40)):
            cover = np.zeros(n, np.int32)
            for k in range(seg_off[g], seg_off[g + 1]):
                st, c = int(seg_start[k]), int(seg_count[k])
                if st < n:
                    assert st + c <= n
                    cover[st:st + c] += 1
                else:
                    first = (st - n) // m
                    assert (st - n) % m == 0 and c % m == 0
                    for s in range(first, first + c // m):
                        v = slot_node[s]
                        cover[beg[v]:end[v]] += 1
            assert np.all(cover == 1), g
        # merge rule of the device's sub-walks (tree.cu traverse_sub_kernel): a direct
        # range never spans two second-level subtrees (the frontier: level-2 nodes and
        # leaves above level 2, which partition the sources)
        front = np.nonzero((lv == 2) | ((nc == 0) & (lv < 2)))[0]
        fb = np.sort(beg[front])
        assert fb[0] == 0 and np.array_equal(np.sort(end[front])[:-1], fb[1:])
        direct = seg_start < n
        st, c = seg_start[direct], seg_count[direct].astype(np.int64)
        k = np.searchsorted(fb, st, side="right") - 1
        limit = np.append(fb[1:], n)[k]
        assert np.all(st + c <= limit)
    finally:
        lib.spk_tree_host_free(tree)
