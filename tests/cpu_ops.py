"""CPU stand-in for paper_2108_02991_b200.engine.CudaOps, built on the oracle.  TEST ONLY:
lets the multi-rank engine (sharding, all-gathers, rank-ordered reductions, guards) run
under the gloo backend in a GPU-less container.  Mirrors the kernels' semantics: float32
positions for the N-body, fp64 everything else."""

import numpy as np
import torch

from oracle import oracle as orc
from paper_2108_02991_b200.projection import stacked_operator_norm


class OracleOps:
    def __init__(self):
        self.device = torch.device("cpu")

    def empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype)

    def to_device(self, arr):
        return torch.from_numpy(np.array(arr, dtype=np.float64, copy=True))

    @staticmethod
    def _fill_pos4(coords, pos4):
        d = coords.shape[-1]
        flat = coords.reshape(-1, d)
        pos4.zero_()
        pos4[:, :d] = flat.to(torch.float32)
        pos4[:, 3] = 1.0

    def pack(self, coords, out):
        self._fill_pos4(coords, out)
        return out

    def sums(self, tgt4, src4, coords_local, fld, cfg):
        d = cfg.dims
        assert cfg.grad_mode == "exact", "OracleOps covers the exact (north-star) mode"
        t = tgt4[:, :d].double().numpy()
        s = src4[:, :d].double().numpy()
        va, ga = orc.grid_sums(t, fld.density.grid, fld.kernel_eps ** 2)
        vr, gr = orc.cross_sums(t, s, cfg.repulsion.kernel_eps ** 2)
        return tuple(torch.from_numpy(x) for x in (va, ga, vr, gr))

    def spatial_capable(self, cfg):
        # the spatial target partition (engine.ShardedRun.spatial) only when a test asks
        import os

        return os.environ.get("SPK_SPATIAL") == "1"

    def spatial_order(self, pos4, dims):
        """Morton order of the samples (21 bits per axis), deterministic, like the
        device sort."""
        q = np.clip(((pos4[:, :dims].double().numpy() + 1.0) * 0.5 * (1 << 21)).astype(np.int64),
                    0, (1 << 21) - 1)
        key = np.zeros(q.shape[0], dtype=np.int64)
        for bit in range(21):
            for a in range(dims):
                key |= ((q[:, a] >> bit) & 1) << (bit * dims + a)
        return torch.from_numpy(np.argsort(key, kind="stable"))

    def combine(self, va, ga, vr, gr, p, coords, prev_c, prev_g, grad_out):
        g = ga.numpy() / float(p) - gr.numpy() / (float(p) * float(p))
        grad_out.copy_(torch.from_numpy(g))
        out = np.zeros(6)
        out[0] = va.numpy().sum()
        out[1] = vr.numpy().sum()
        if prev_c is not None:
            dk = coords.numpy().reshape(g.shape) - prev_c.numpy().reshape(g.shape)
            dg = g - prev_g.numpy().reshape(g.shape)
            out[2] = np.vdot(dk, dg)
            out[3] = np.vdot(dg, dg)
        out[4] = np.count_nonzero(~np.isfinite(g))
        return torch.from_numpy(out)

    def project(self, coords, cfg, grad, eta, out, pos4, nonfinite, sweeps=None):
        k = coords.numpy()
        if grad is not None:
            k = k - eta * grad.numpy()
        if nonfinite is not None and not np.isfinite(k).all():
            nonfinite.fill_(1)
        n_c, n_s, d = k.shape
        pin = -1 if cfg.pin is None else cfg.pin.pinned_index
        pv = np.zeros(d) if cfg.pin is None else cfg.pin.pinned_value
        tau = 1.0 / stacked_operator_norm(n_s, pin)
        res, sw = orc.project_all(k, cfg.speed_bound, cfg.accel_bound, pin, pv, cfg.n_pit,
                                  tau, 0.1 * cfg.feas_tol, monotone=cfg.monotone)
        out.copy_(torch.from_numpy(res))
        if pos4 is not None:
            self._fill_pos4(out, pos4)
        if sweeps is not None:
            sweeps.copy_(torch.from_numpy(sw.astype(np.int32)))
        return out


    def residuals(self, coords, cfg):
        c = coords.numpy()
        amp = max(np.abs(c).max() - 1.0, 0.0)
        d1 = np.linalg.norm(np.diff(c, axis=1), axis=2)
        d2 = np.linalg.norm(np.diff(c, 2, axis=1), axis=2)
        sp = max(d1.max() - cfg.speed_bound, 0.0) if d1.size else 0.0
        ac = max(d2.max() - cfg.accel_bound, 0.0) if d2.size else 0.0
        pe = 0.0
        if cfg.pin is not None:
            pe = float(np.abs(c[:, cfg.pin.pinned_index, :] - cfg.pin.pinned_value).max())
        return torch.tensor([amp, sp, ac, pe, max(amp, sp, ac, pe)], dtype=torch.float64)

    def upsample(self, coords):
        c = coords.numpy()
        n_c, n_s, d = c.shape
        up = np.empty((n_c, 2 * n_s, d))
        up[:, 0::2] = c
        up[:, 1:-1:2] = 0.5 * (c[:, :-1] + c[:, 1:])
        up[:, -1] = c[:, -1] + 0.5 * (c[:, -1] - c[:, -2])
        return torch.from_numpy(np.clip(up, -1.0, 1.0))


class OverlapOracleOps(OracleOps):
    """OracleOps with the engine's K2-under-polish schedule (engine.ShardedRun.overlap):
    the projection of each polish group (shots in ``order``) followed by that group's
    lattice sums, synchronously -- exercises the schedule's bookkeeping (shot order from
    the previous sweeps, per-rank K2 rows, K1 alone afterwards) on the CPU."""

    OVERLAP_GROUPS = 3

    def overlap_capable(self, cfg):
        return cfg.grad_mode == "exact"

    def project_overlap(self, coords, cfg, grad, eta, out, pos4, nonfinite, fld, att_val,
                        att_grad, sweeps, order, groups_out=None, polite=False):
        self.overlap_calls = getattr(self, "overlap_calls", 0) + 1
        self.project(coords, cfg, grad, eta, out, pos4, nonfinite, sweeps)
        n_c, n_s, d = coords.shape
        ids = np.arange(n_c) if order is None else order.numpy()
        assert sorted(ids.tolist()) == list(range(n_c))
        for grp in np.array_split(ids, self.OVERLAP_GROUPS):
            if groups_out is not None:
                groups_out.append((torch.from_numpy(grp.astype(np.int32)), None))
            for c in grp:
                t = pos4[c * n_s:(c + 1) * n_s, :d].double().numpy()
                va, ga = orc.grid_sums(t, fld.density.grid, fld.kernel_eps ** 2)
                att_val[c * n_s:(c + 1) * n_s] = torch.from_numpy(va)
                att_grad[c * n_s:(c + 1) * n_s] = torch.from_numpy(ga)
        return out, []

    def repulsion_sums(self, tgt4, src4, cfg):
        d = cfg.dims
        vr, gr = orc.cross_sums(tgt4[:, :d].double().numpy(), src4[:, :d].double().numpy(),
                                cfg.repulsion.kernel_eps ** 2)
        return torch.from_numpy(vr), torch.from_numpy(gr)
