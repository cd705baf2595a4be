"""Device-resident state of one optimisation run, sharded over ranks.

``ShardedRun`` owns the fp64 shot coordinates of this rank's contiguous block of shots,
the float4 positions of ALL samples (the K1 sources), and the gradient buffers.  Each
optimizer iteration is:

  evaluate()      fused K1 + K2 (or field interpolation + K1) -> combine kernel
                  -> 6 scalars -> all-gather, summed in rank order (deterministic)
  step_project()  K3 with the step k - eta*grad in its prologue; the polish epilogue
                  writes this rank's float4 positions straight into its slice of the
                  gather buffer; NCCL all-gather of positions over NVLink
  residual_max()  feasibility reduction -> all-gather max

The device operations come from an ``ops`` object; the product uses :class:`CudaOps`
(the sm_100a kernels).  Tests substitute CPU ops to exercise the multi-rank logic with
the gloo backend.
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _native
from .attraction import field_eval_device, grid_sums_device, tree_grid_sums_device
from .projection import project_device, project_overlap_device, residuals_device
from .repulsion import direct_sums_device, tree_sums_checked


class CudaOps:
    """The product device operations: every call is one of our sm_100a kernels."""

    def __init__(self):
        self.device = _device.device()
        # treecode auto-mode rows validated by the probe (repulsion and lattice), per run
        self._tree_rows = {}

    def empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def to_device(self, arr: np.ndarray) -> torch.Tensor:
        return _device.h2d(arr)

    def pack(self, coords, out):
        return _device.pack_positions(coords, out)

    def sums(self, tgt4, src4, coords_local, fld, cfg):
        """Raw attraction (val, grad) and repulsion (val, grad) sums for local targets."""
        n_t = tgt4.shape[0]
        d = cfg.dims
        eps2_rep = cfg.repulsion.kernel_eps ** 2
        att_tree = cfg.grad_mode == "exact" and cfg.attraction_tree_precision is not None
        if cfg.repulsion.backend == "tree" or att_tree:
            # treecode repulsion (tree.py) and/or treecode attraction; the targets'
            # sort is shared when both run
            tg = None
            if cfg.repulsion.backend == "tree":
                vr, gr, tg = tree_sums_checked(tgt4, src4, d, cfg.repulsion, return_groups=True,
                                               row_cache=self._tree_rows)
            else:
                vr, gr = direct_sums_device(tgt4, src4, d, eps2_rep)
            if att_tree:
                va, ga = tree_grid_sums_device(tgt4, fld, fld.kernel_eps ** 2,
                                               cfg.attraction_tree_precision, tg=tg,
                                               row_cache=self._tree_rows)
            elif cfg.grad_mode == "exact":
                va, ga = grid_sums_device(tgt4, fld, fld.kernel_eps ** 2)
            else:
                va, ga, _ = field_eval_device(coords_local.reshape(-1, d), fld, cfg.grad_mode)
            return va, ga, vr, gr
        vr = self.empty(n_t)
        gr = self.empty((n_t, d))
        if cfg.grad_mode == "exact":
            va = self.empty(n_t)
            ga = self.empty((n_t, d))
            w = fld.device_sources()
            sides = fld.sides
            n_cells = int(np.prod(sides))
            nbytes = _native.query("spk_nbody_workspace_bytes", n_t, n_cells, src4.shape[0])
            ws = _device.workspace(nbytes, "nbody")
            _native.call("spk_fused_sums", tgt4.data_ptr(), n_t, d, w.data_ptr(),
                         _native.i64_array(sides), float(fld.kernel_eps ** 2),
                         src4.data_ptr(), src4.shape[0],
                         float(eps2_rep), va.data_ptr(), ga.data_ptr(), vr.data_ptr(),
                         gr.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream())
        else:
            va, ga, _ = field_eval_device(coords_local.reshape(-1, d), fld, cfg.grad_mode)
            vr, gr = direct_sums_device(tgt4, src4, d, eps2_rep)
        return va, ga, vr, gr

    def combine(self, va, ga, vr, gr, p, coords, prev_c, prev_g, grad_out):
        n_t, d = ga.shape
        out = self.empty(6)
        ws = _device.workspace(_native.query("spk_combine_workspace_bytes", n_t), "combine")
        _native.call("spk_combine_gradient", n_t, d, va.data_ptr(), ga.data_ptr(), float(p),
                     vr.data_ptr(), gr.data_ptr(), float(p), coords.data_ptr(),
                     _device.ptr(prev_c), _device.ptr(prev_g), grad_out.data_ptr(),
                     out.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream())
        return out

    def project(self, coords, proj_cfg, grad, eta, out, pos4, nonfinite, sweeps=None,
                peers=None):
        return project_device(coords, proj_cfg, grad=grad, eta=eta, out=out, pos4=pos4,
                              nonfinite=nonfinite, sweeps=sweeps, peers=peers)

    def residuals(self, coords, proj_cfg):
        return residuals_device(coords, proj_cfg)

    # ---- K2-under-polish overlap (ShardedRun.overlap)
    OVERLAP_GROUPS = int(os.environ.get("SPK_OVERLAP_GROUPS", "8"))

    def overlap_capable(self, cfg) -> bool:
        """Eligible for the K2-under-polish schedule: exact lattice attraction and exact
        repulsion (the fused N-body splits into K2 per polish group + K1)."""
        return (cfg.grad_mode == "exact" and cfg.attraction_tree_precision is None
                and cfg.repulsion.backend == "direct")

    def _overlap_streams(self):
        if not hasattr(self, "_ostreams"):
            g = self.OVERLAP_GROUPS
            self._ostreams = ([torch.cuda.Stream(priority=-1) for _ in range(g)],
                              [torch.cuda.Stream(priority=0) for _ in range(g)])
        return self._ostreams

    def project_overlap(self, coords, proj_cfg, grad, eta, out, pos4, nonfinite, fld,
                        att_val, att_grad, sweeps, order, groups_out=None, polite=False,
                        peers=None):
        n_c = coords.shape[0]
        ps, ks = self._overlap_streams()
        g = max(1, min(len(ps), n_c // 8))
        busy = None
        if polite:
            if not hasattr(self, "_sm_busy"):
                # per-SM count of running polish CTAs (projection_overlap_device)
                self._sm_busy = torch.zeros(256, dtype=torch.int32, device=coords.device)
            busy = self._sm_busy
            busy.zero_()  # stream-ordered before this call's polish (no stale counts)
        return project_overlap_device(coords, proj_cfg, grad=grad, eta=eta, out=out,
                                      pos4=pos4, nonfinite=nonfinite, field=fld,
                                      att_val=att_val, att_grad=att_grad, sweeps=sweeps,
                                      order=order, polish_streams=ps[:g], k2_streams=ks[:g],
                                      groups_out=groups_out, sm_busy=busy, peers=peers)

    def repulsion_sums(self, tgt4, src4, cfg):
        return direct_sums_device(tgt4, src4, cfg.dims, cfg.repulsion.kernel_eps ** 2)

    def k1_streams(self):
        """(gather stream, K1 stream) of the pipelined K1 (ShardedRun._k1_pipelined)."""
        if not hasattr(self, "_k1s"):
            self._k1s = (torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0))
        return self._k1s

    def k1_workspace_bytes(self, shapes) -> int:
        return max(_native.query("spk_nbody_workspace_bytes", t, 0, s) for t, s in shapes)

    def repulsion_block(self, tgt4, src4, cfg, ws):
        """K1 of a target block against a source block, fresh fp64 outputs, caller-owned
        workspace (launches on a side stream must not share the cached one)."""
        n_t, n_s, d = tgt4.shape[0], src4.shape[0], cfg.dims
        val = torch.empty(n_t, dtype=torch.float64, device=tgt4.device)
        grad = torch.empty((n_t, d), dtype=torch.float64, device=tgt4.device)
        _native.call("spk_direct_sums", tgt4.data_ptr(), n_t, src4.data_ptr(), n_s, d,
                     float(cfg.repulsion.kernel_eps ** 2), val.data_ptr(), grad.data_ptr(),
                     ws.data_ptr(), ws.numel(), _device.stream())
        return val, grad

    # ---- spatial target partition for the treecodes (ShardedRun.spatial)
    def spatial_capable(self, cfg) -> bool:
        """Treecode sums cost per target depends on how densely a rank's targets fill
        space: a shot-sharded rank holds every 1/N-th spoke everywhere, so its target
        groups are sparse.  With the treecodes the N-body targets are therefore split by
        Morton order (compact blocks) instead of by shot."""
        return cfg.grad_mode == "exact" and (cfg.repulsion.backend == "tree"
                                             or cfg.attraction_tree_precision is not None)

    def spatial_order(self, pos4, dims):
        """Permutation of the samples along the Morton curve (device int64; the same on
        every rank for the same positions)."""
        from . import tree

        _, perm = tree._sort(pos4, dims)
        return perm.long()

    def upsample(self, coords):
        n_c, n_s, d = coords.shape
        out = self.empty((n_c, 2 * n_s, d))
        _native.call("spk_upsample_shots", coords.data_ptr(), out.data_ptr(), n_c, n_s, d,
                     _device.stream())
        return out


def k1_pipelined(ops, cfg, pos, groups, world, gather):
    """K1 (repulsion) of the next evaluation computed under the polish, as the polish
    groups finish (ShardedRun with the overlap schedule on several ranks; DESIGN.md
    section 7).

    ``pos``: this rank's position records [local shots, n_s, 4] as the projection writes
    them; ``groups``: (shot ids, polished event) per polish group in launch order, every
    rank with the same number of equally sized groups; ``gather(q, loc_q, src_q)`` fills
    ``src_q`` with every rank's q-th group block (``loc_q`` is this rank's; an NCCL
    all_gather_into_tensor across ranks).  Groups are taken in their expected finishing
    order (shortest first: the reverse of the longest-first launch order).  For the q-th
    group its block is gathered on a gather stream; then on a K1 stream the local targets
    of group q are summed against the gathered groups 0..q and the local targets of groups
    0..q-1 against gathered group q -- every (target group, source group) block runs
    once, as soon as both are final.  Sums accumulate per target group in a fixed block
    order (deterministic).  Returns (val, grad, [event]) in shot order, or None if the
    groups are unequal."""
    sizes = {int(ids.numel()) for ids, _ in groups}
    if len(sizes) != 1:
        return None
    G, n_g = len(groups), sizes.pop()
    local, n_s = pos.shape[0], pos.shape[1]
    d = cfg.dims
    ng_t = n_g * n_s
    cuda = pos.is_cuda
    dev = pos.device
    loc = ops.empty((G, ng_t, 4), torch.float32)
    src = ops.empty((G, world * ng_t, 4), torch.float32)
    acc_v = torch.zeros((G, ng_t), dtype=torch.float64, device=dev)
    acc_g = torch.zeros((G, ng_t, d), dtype=torch.float64, device=dev)
    proc = list(reversed(range(G)))
    ws = None
    if cuda:
        cs, ks = ops.k1_streams()
        shapes = [(ng_t, (q + 1) * world * ng_t) for q in range(G)]
        shapes += [(q * ng_t, world * ng_t) for q in range(1, G)]
        cs.wait_stream(torch.cuda.current_stream())
        ks.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(ks):
            ws = torch.empty(ops.k1_workspace_bytes(shapes), dtype=torch.uint8, device=dev)

    def on(stream):
        return torch.cuda.stream(stream) if cuda else contextlib.nullcontext()

    def block(tgt4, src4):
        if cuda:
            return ops.repulsion_block(tgt4, src4, cfg, ws)
        return ops.repulsion_sums(tgt4, src4, cfg)

    for q, g in enumerate(proc):
        ids, polished = groups[g]
        if cuda and polished is not None:
            cs.wait_event(polished)
        with on(cs if cuda else None):
            loc[q].copy_(pos.index_select(0, ids.long()).reshape(ng_t, 4))
            gather(q, loc[q], src[q])
        if cuda:
            ks.wait_stream(cs)
        with on(ks if cuda else None):
            v, gg = block(loc[q], src[:q + 1].reshape(-1, 4))
            acc_v[q] += v
            acc_g[q] += gg.view(ng_t, d)
            if q > 0:
                v, gg = block(loc[:q].reshape(-1, 4), src[q])
                acc_v[:q] += v.view(q, ng_t)
                acc_g[:q] += gg.view(q, ng_t, d)
    with on(ks if cuda else None):
        ids_all = torch.cat([groups[g][0] for g in proc]).long()
        vr = ops.empty(local * n_s)
        gr = ops.empty((local * n_s, d))
        vr.view(local, n_s)[ids_all] = acc_v.view(G * n_g, n_s)
        gr.view(local, n_s, d)[ids_all] = acc_g.view(G * n_g, n_s, d)
    events = []
    if cuda:
        ev = torch.cuda.Event()
        ev.record(ks)
        events.append(ev)
        for t in (loc, src, acc_v, acc_g, vr, gr, ws, ids_all):
            t.record_stream(ks)
        for t in (loc, src, pos):
            t.record_stream(cs)
        for ids, _ in groups:
            ids.record_stream(cs)
            ids.record_stream(ks)
    return vr, gr, events


class ShardedRun:
    """Per-rank device state for :func:`optimize` (see module docstring)."""

    def __init__(self, start: np.ndarray, cfg, fld, ops=None, group=None):
        self.cfg = cfg
        self.fld = fld
        self.ops = ops if ops is not None else CudaOps()
        if group is None and dist.is_available() and dist.is_initialized():
            group = dist.group.WORLD
        self.group = group
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        n_c, n_s, d = start.shape
        if n_c < self.world:
            # every rank must own at least one shot: the kernels need targets, and a rank
            # without any would fail while the others wait in the collectives
            raise ValueError(f"{n_c} shots cannot be sharded over {self.world} ranks; "
                             f"use at most {n_c} ranks")
        base, extra = divmod(n_c, self.world)
        self.counts = [base + (1 if r < extra else 0) for r in range(self.world)]
        self.offsets = [sum(self.counts[:r]) for r in range(self.world)]
        self.even = extra == 0
        self.n_c, self.d = n_c, d
        lo = self.offsets[self.rank]
        self.local = self.counts[self.rank]
        self.coords = self.ops.to_device(np.ascontiguousarray(start[lo:lo + self.local]))
        self._level_buffers(n_s)

    # ------------------------------------------------------------------ buffers
    def _level_buffers(self, n_s: int):
        ops, d = self.ops, self.d
        self.n_s = n_s
        self.p = self.n_c * n_s
        self.pos4_all = ops.empty((self.p, 4), torch.float32)
        if self.world == 1 or self.even:
            off = self.offsets[self.rank] * n_s
            self.pos4_local = self.pos4_all.narrow(0, off, self.local * n_s)
        else:
            self.pos4_local = ops.empty((max(self.counts) * n_s, 4), torch.float32)
        self.next = ops.empty((self.local, n_s, d))
        self.prev = ops.empty((self.local, n_s, d))
        self.grad = ops.empty((self.local, n_s, d))
        self.prev_grad = ops.empty((self.local, n_s, d))
        self.flag = ops.empty(1, torch.int32)
        self.have_prev = False
        self.host_prev = None
        # K2-under-polish overlap: the lattice sums of the positions the last projection
        # produced (att_pre), and the polish sweep counts that order the next one
        self.overlap = hasattr(ops, "overlap_capable") and ops.overlap_capable(self.cfg)
        env = os.environ.get("SPK_SPATIAL")
        self.spatial = (hasattr(ops, "spatial_capable") and ops.spatial_capable(self.cfg)
                        and (self.world > 1 if env is None else env == "1"))
        self.att_pre = None
        self.rep_pre = None
        self.sweeps_prev = None
        self._setup_peers()
        if self.overlap:
            self.att_val = ops.empty(self.local * n_s)
            self.att_grad = ops.empty((self.local * n_s, d))
            self.sweeps = ops.empty(self.local, torch.int32)

    # ------------------------------------------------------------ communication
    def _setup_peers(self):
        """Fused position all-gather (SPK_P2P_GATHER, default on with several ranks and
        even shards on CUDA): every rank maps the other ranks' position buffers (CUDA IPC,
        opened on this rank's device so its kernels write over NVLink) and the polish
        epilogue writes each new record into all of them (spk_polish_shots peer_pos4), so
        no separate all-gather runs.  Every rank must succeed or all use the all-gather;
        the first exchange of every level is also checked against an NCCL all-gather, and
        a mismatch falls back to the all-gather for the rest of the run."""
        for ptr in getattr(self, "_peer_ptrs", []):
            _native.call("spk_ipc_close", ctypes.c_void_p(ptr))
        self._peer_ptrs = []
        self.peers = None
        env = os.environ.get("SPK_P2P_GATHER")
        if (self.world == 1 or not self.even or not self.coords.is_cuda or env == "0"
                or getattr(self, "_p2p_failed", False)):
            return
        ok = 1.0
        mine = None
        try:
            info = self.pos4_all.untyped_storage()._share_cuda_()
            off = int(info[3]) + self.pos4_all.storage_offset() * self.pos4_all.element_size()
            raw = bytes(info[1])
            # torch's shareable handle: [version, b"c" (cudaMalloc block)] + the 64-byte
            # cudaIpcMemHandle_t; other kinds (expandable segments) are not IPC handles
            if len(raw) == 66 and raw[1:2] == b"c":
                raw = raw[2:]
            if len(raw) != 64:
                raise ValueError("not a cudaIpcMemHandle")
            mine = (raw, off)
        except Exception:  # noqa: BLE001 -- any failure means: use the all-gather
            ok = 0.0
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        addrs = []
        if ok and all(h is not None for h in allh):
            try:
                for r, (handle, off) in enumerate(allh):
                    if r == self.rank:
                        continue
                    ptr = ctypes.c_void_p()
                    _native.call("spk_ipc_open", handle, ctypes.byref(ptr))
                    self._peer_ptrs.append(ptr.value)
                    addrs.append(ptr.value + off)
            except Exception:  # noqa: BLE001
                ok = 0.0
        else:
            ok = 0.0
        flag = torch.tensor([ok], device=self.coords.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        if flag.item() != 1.0:
            for ptr in self._peer_ptrs:
                _native.call("spk_ipc_close", ctypes.c_void_p(ptr))
            self._peer_ptrs = []
            self._p2p_failed = True
            return
        table = torch.tensor(addrs, dtype=torch.int64, device=self.coords.device)
        self.peers = (table, len(addrs), self.offsets[self.rank] * self.n_s)
        self._p2p_verified = False

    def _exchanged(self):
        """Positions after a projection: with the fused gather only the first exchange of
        a level is verified (an NCCL all-gather compared on every rank); otherwise the
        all-gather."""
        if self.peers is None:
            self._gather_pos4()
            return
        if self._p2p_verified:
            return
        ref = self.ops.empty(self.pos4_all.shape, torch.float32)
        dist.all_gather_into_tensor(ref, self.pos4_local, group=self.group)
        ok = torch.tensor([1.0 if torch.equal(ref, self.pos4_all) else 0.0],
                          device=self.coords.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if ok.item() == 1.0:
            self._p2p_verified = True
            return
        import warnings

        warnings.warn("fused position all-gather (peer memory) did not match the NCCL "
                      "all-gather; using the all-gather for the rest of the run")
        self.pos4_all.copy_(ref)
        self.peers = None
        self._p2p_failed = True

    def _gather_pos4(self):
        if self.world == 1:
            return
        if self.even:
            dist.all_gather_into_tensor(self.pos4_all, self.pos4_local, group=self.group)
            return
        m = max(self.counts) * self.n_s
        pad = self.ops.empty((self.world * m, 4), torch.float32)
        dist.all_gather_into_tensor(pad, self.pos4_local, group=self.group)
        for r in range(self.world):
            n = self.counts[r] * self.n_s
            self.pos4_all[self.offsets[r] * self.n_s:self.offsets[r] * self.n_s + n] = \
                pad[r * m:r * m + n]

    def _all_scalars(self, t: torch.Tensor) -> np.ndarray:
        """(world, k) host array of every rank's scalar vector, rank order."""
        if self.world == 1:
            return t.detach().to("cpu").numpy()[None]
        buf = self.ops.empty((self.world, t.numel()), t.dtype)
        dist.all_gather_into_tensor(buf, t.reshape(1, -1), group=self.group)
        return buf.to("cpu").numpy()

    # --------------------------------------------------------------- iteration
    def project(self, proj_cfg):
        """Level-start projection (no step)."""
        kw = {"peers": self.peers} if self.peers is not None else {}
        out = self.ops.project(self.coords, proj_cfg, None, 0.0, self.next,
                               self._pos4_target(), None, **kw)
        self.coords, self.next = out, self.coords
        self._exchanged()
        self.have_prev = False
        self.host_prev = None
        self.att_pre = None
        self.rep_pre = None

    def _pos4_target(self):
        n = self.local * self.n_s
        return self.pos4_local if self.pos4_local.shape[0] == n else self.pos4_local[:n]

    def evaluate(self):
        """Fused device evaluation -> (att_cost, rep_cost, n_nonfinite, (dkdg, dgdg))."""
        tgt = self._pos4_target()
        if self.spatial:
            va, ga, vr, gr = self._spatial_sums()
        elif self.att_pre is not None:
            # K2 ran (or is still running) under the last polish; only K1 needs the
            # gathered sources, and it co-runs with the tail of K2
            va, ga, k2_events = self.att_pre
            self.att_pre = None
            if self.rep_pre is not None:
                # K1 too ran under the polish, block by block (_k1_pipelined)
                vr, gr, k1_events = self.rep_pre
                self.rep_pre = None
                k2_events = list(k2_events) + list(k1_events)
            else:
                vr, gr = self.ops.repulsion_sums(tgt, self.pos4_all, self.cfg)
            if k2_events:
                cur = torch.cuda.current_stream()
                for ev in k2_events:
                    cur.wait_event(ev)
        else:
            va, ga, vr, gr = self.ops.sums(tgt, self.pos4_all, self.coords, self.fld,
                                           self.cfg)
        prev_c = self.prev if self.have_prev else None
        prev_g = self.prev_grad if self.have_prev else None
        scal = self.ops.combine(va, ga, vr, gr, self.p, self.coords, prev_c, prev_g,
                                self.grad.view(-1, self.d))
        allv = self._all_scalars(scal)
        tot = np.zeros(allv.shape[1])
        for r in range(allv.shape[0]):
            tot = tot + allv[r]
        p = self.p
        att_cost = float(tot[0] / p)
        rep_cost = float(tot[1] / (2.0 * p * p))
        return att_cost, rep_cost, int(tot[4]), (float(tot[2]), float(tot[3]))

    def _spatial_sums(self):
        """N-body sums with the targets split by Morton order: rank r evaluates the r-th
        contiguous block of the sorted samples against all sources, the blocks' results
        are all-gathered (p x (2 + 2d) fp64, rank order) and every rank keeps the rows of
        its own shots.  Deterministic for a given world size."""
        d, p = self.d, self.p
        perm = self.ops.spatial_order(self.pos4_all, d)
        bounds = [p * r // self.world for r in range(self.world + 1)]
        lo, hi = bounds[self.rank], bounds[self.rank + 1]
        tgt = self.pos4_all[perm[lo:hi]].contiguous()
        va, ga, vr, gr = self.ops.sums(tgt, self.pos4_all, None, self.fld, self.cfg)
        w = 2 + 2 * d
        pack = torch.cat([va.reshape(-1, 1), ga.reshape(-1, d), vr.reshape(-1, 1),
                          gr.reshape(-1, d)], dim=1)
        if self.world > 1:
            m = max(bounds[r + 1] - bounds[r] for r in range(self.world))
            pad = self.ops.empty((m, w))
            pad[:hi - lo] = pack
            buf = self.ops.empty((self.world * m, w))
            dist.all_gather_into_tensor(buf, pad, group=self.group)
            pack = torch.cat([buf[r * m:r * m + bounds[r + 1] - bounds[r]]
                              for r in range(self.world)])
        full = self.ops.empty((p, w))
        full.index_copy_(0, perm, pack)
        n_s = self.n_s
        mine = full[self.offsets[self.rank] * n_s:(self.offsets[self.rank] + self.local) * n_s]
        return (mine[:, 0].contiguous(), mine[:, 1:1 + d].contiguous(),
                mine[:, 1 + d].contiguous(), mine[:, 2 + d:].contiguous())

    def set_host_gradient(self, grad: np.ndarray):
        """Patched-evaluator path: install a host gradient of ALL shots (every rank
        evaluates the same gathered pattern), keep this rank's rows, and return the BB
        dot products computed with numpy over the whole pattern exactly as step_size
        does (identical on every rank)."""
        coords = self.gather_coords()
        dots = (0.0, 0.0)
        if self.host_prev is not None:
            pc, pg = self.host_prev
            dk = coords - pc
            dg = grad - pg
            dots = (float(np.vdot(dk, dg)), float(np.vdot(dg, dg)))
        self.host_prev = (coords.copy(), grad)
        lo = self.offsets[self.rank]
        mine = np.ascontiguousarray(grad[lo:lo + self.local], dtype=np.float64)
        self.grad.copy_(torch.from_numpy(mine))
        return dots

    # Overlap pays when the polish is heavy next to the N-body: splitting the fused launch
    # into K1 + per-group K2 costs ~6 % of the N-body (the pipes no longer mix), the K2
    # hidden under the polish is ~40 % of the polish time (C2, profiles/
    # r02_rank_share_c2.jsonl).  Polish time per sample ~1.5e-11 s per sweep, N-body time
    # per target ~2.6e-13 s per source: overlap iff mean sweeps >= 2.7e-3 (G + p).  The
    # rule uses the previous projection's sweep counts, so it is deterministic.
    OVERLAP_MIN_SWEEPS_PER_SOURCE = 2.7e-3

    def _use_overlap(self) -> bool:
        env = os.environ.get("SPK_OVERLAP")
        if env is not None:
            return env == "1"
        if self.sweeps_prev is None:
            return False
        n_src = self.p + int(np.prod(self.fld.sides))
        mean = float(self.sweeps_prev.to(torch.float64).mean().item())
        return mean >= self.OVERLAP_MIN_SWEEPS_PER_SOURCE * n_src

    def _use_polite_k2(self) -> bool:
        """K2 CTAs only on SMs without polish CTAs (project_overlap_device sm_busy):
        SPK_POLITE_K2=0/1 forces it; by default on when this rank's shots fit one polish
        CTA per SM, so the polish holds a minority of the GPU and idle SMs appear as its
        shots finish (a rank's share at N >= 8 at C2)."""
        env = os.environ.get("SPK_POLITE_K2")
        if env is not None:
            return env == "1"
        if not self.coords.is_cuda:
            return False
        props = torch.cuda.get_device_properties(self.coords.device)
        return self.local <= props.multi_processor_count

    def _use_k1_pipeline(self) -> bool:
        """K1 block by block under the polish (_k1_pipelined), opt-in with SPK_K1_PIPE=1
        (even shards only).  Off by default: the per-rank-share projection measured it
        within +-3 % of the plain overlap schedule at N = 2 / 4 / 8 (the K1 blocks take
        issue slots from the latency-bound polish on the same SMs)."""
        return os.environ.get("SPK_K1_PIPE") == "1" and self.even

    def _k1_pipelined(self, groups):
        """K1 of the next evaluation, block by block under the polish (k1_pipelined)."""
        def gather(q, loc_q, src_q):
            if self.world > 1:
                dist.all_gather_into_tensor(src_q, loc_q, group=self.group)
            else:
                src_q.copy_(loc_q)

        pos = self._pos4_target().view(self.local, self.n_s, 4)
        return k1_pipelined(self.ops, self.cfg, pos, groups, self.world, gather)

    def step_project(self, proj_cfg, eta: float) -> bool:
        """coords <- P(coords - eta * grad); returns False if the step was non-finite."""
        self.flag.zero_()
        if self.overlap and self._use_overlap():
            order = None
            if self.sweeps_prev is not None:
                order = torch.argsort(self.sweeps_prev, descending=True,
                                      stable=True).to(torch.int32)
            groups = [] if self._use_k1_pipeline() else None
            kw = {"peers": self.peers} if self.peers is not None else {}
            out, k2_events = self.ops.project_overlap(
                self.coords, proj_cfg, self.grad, float(eta), self.next, self._pos4_target(),
                self.flag, self.fld, self.att_val, self.att_grad, self.sweeps, order,
                groups_out=groups, polite=self._use_polite_k2(), **kw)
            self.att_pre = (self.att_val, self.att_grad, k2_events)
            self.rep_pre = self._k1_pipelined(groups) if groups else None
            self.sweeps_prev = self.sweeps.clone()
        elif self.overlap:
            # plain schedule, but keep the sweep counts that decide and order the overlap
            kw = {"peers": self.peers} if self.peers is not None else {}
            out = self.ops.project(self.coords, proj_cfg, self.grad, float(eta), self.next,
                                   self._pos4_target(), self.flag, self.sweeps, **kw)
            self.sweeps_prev = self.sweeps.clone()
        else:
            kw = {"peers": self.peers} if self.peers is not None else {}
            out = self.ops.project(self.coords, proj_cfg, self.grad, float(eta), self.next,
                                   self._pos4_target(), self.flag, **kw)
        # rotate: prev <- coords, coords <- out, next <- old prev
        self.prev, self.coords, self.next = self.coords, out, self.prev
        self.prev_grad, self.grad = self.grad, self.prev_grad
        self.have_prev = True
        # the flag all-gather completes only after every rank's projection (and so its
        # peer writes, with the fused gather) has finished
        bad = self._all_scalars(self.flag.to(torch.float64))
        self._exchanged()
        return not bool(bad.max() > 0)

    def residual_max(self, proj_cfg) -> float:
        r = self.ops.residuals(self.coords, proj_cfg)
        allv = self._all_scalars(r)
        return float(allv[:, 4].max())

    def upsample(self):
        self.coords = self.ops.upsample(self.coords)
        self._level_buffers(self.coords.shape[1])

    def gather_coords(self) -> np.ndarray:
        """All ranks' fp64 coordinates, global shot order, on the host."""
        if self.world == 1:
            return self.coords.detach().to("cpu").numpy().copy()
        m = max(self.counts)
        loc = self.ops.empty((m, self.n_s, self.d))
        loc[:self.local] = self.coords
        buf = self.ops.empty((self.world * m, self.n_s, self.d))
        dist.all_gather_into_tensor(buf, loc, group=self.group)
        host = buf.to("cpu").numpy()
        parts = [host[r * m:r * m + self.counts[r]] for r in range(self.world)]
        return np.ascontiguousarray(np.concatenate(parts, axis=0))
