"""Constraint projection K3 on the B200 (fp64; one CTA per shot for FISTA, a systolic
ring of sweeps per shot for the polish).

Projects each shot onto {|s| <= 1, ||s[n+1]-s[n]|| <= alpha dt, ||s[n+2]-2s[n+1]+s[n]||
<= beta dt^2, s[pin] = v} with the reference's algorithm
(/root/reference/pkg/src/vdtraj/projection.py): dual FISTA with gradient restart
(:169-284) then the over-relaxed cyclic feasibility polish (:287-373).  The kernels are
bit-identical to the reference on the same inputs and step size tau (csrc/project.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .core import FEAS_TOL, LinearConstraint, NormalizedLimits, SamplingPattern

MAX_POLISH_SWEEPS = 50000
_LAMBDA_CACHE: dict = {}


@dataclass
class ProjectionConfig:
    """Same fields, defaults and validation as the reference (projection.py:28-68)."""

    alpha: float
    beta: float
    raster_dt: float
    n_pit: int = 100
    feas_tol: float = FEAS_TOL
    pin: LinearConstraint | None = None
    monotone: bool = False

    def __post_init__(self):
        if self.n_pit < 1:
            raise ValueError("n_pit must be >= 1")
        if self.feas_tol <= 0:
            raise ValueError("feas_tol must be positive")
        if self.raster_dt <= 0:
            raise ValueError("raster_dt must be positive")
        if self.alpha < 0 or self.beta < 0:
            raise ValueError("alpha and beta must be non-negative")

    @classmethod
    def from_limits(cls, limits: NormalizedLimits, raster_dt: float, **kw):
        return cls(alpha=limits.alpha, beta=limits.beta, raster_dt=raster_dt, **kw)

    @property
    def speed_bound(self) -> float:
        return self.alpha * self.raster_dt

    @property
    def accel_bound(self) -> float:
        return self.beta * self.raster_dt**2


def _gram_apply(x: np.ndarray, pin_idx: int) -> np.ndarray:
    """(I + D1^T D1 + D2^T D2) x with the pinned coordinate removed, evaluated with the
    same elementwise sequence as projection.py:86-95 (so lambda is bit-identical)."""
    n = x.shape[0]
    first = np.diff(x)
    second = np.diff(x, 2)
    out = x.copy()
    out[:-1] -= first
    out[1:] += first
    out[: n - 2] += second
    out[1 : n - 1] -= 2 * second
    out[2:] += second
    if pin_idx >= 0:
        out[pin_idx] = 0.0
    return out


def stacked_operator_norm(n_s: int, pin_idx: int) -> float:
    """lambda_max of the stacked constraint operator by 50 power iterations from
    default_rng(12345) (projection.py:71-100); cached per (n_s, pin_idx).  tau = 1/lambda."""
    key = (int(n_s), int(pin_idx))
    hit = _LAMBDA_CACHE.get(key)
    if hit is not None:
        return hit
    x = np.random.default_rng(12345).standard_normal(n_s)
    if pin_idx >= 0:
        x[pin_idx] = 0.0
    for _ in range(50):
        x /= np.linalg.norm(x)
        x = _gram_apply(x, pin_idx)
    lam = float(np.linalg.norm(x))
    _LAMBDA_CACHE[key] = lam
    return lam


_stacked_operator_norm = stacked_operator_norm  # reference-private name


def _pin_arrays(cfg: ProjectionConfig, dims: int):
    if cfg.pin is None:
        return -1, np.zeros(dims)
    value = np.asarray(cfg.pin.pinned_value, dtype=np.float64)
    if value.shape != (dims,):
        raise ValueError(f"pinned_value must have {dims} components")
    return int(cfg.pin.pinned_index), value


def project_device(coords: torch.Tensor, cfg: ProjectionConfig, *, grad=None, eta=0.0,
                   out: torch.Tensor | None = None, pos4=None, sweeps=None, trace=None,
                   nonfinite=None, tau: float | None = None,
                   max_sweeps: int = MAX_POLISH_SWEEPS, eta_per_shot=None,
                   peers=None) -> torch.Tensor:
    """K3 on device buffers: out = P(coords - eta * grad) for every shot.

    ``coords``/``grad``/``out``: (n_shots, n_s, d) fp64 CUDA tensors.  ``pos4`` (optional)
    receives the float4 positions of the result (the next N-body's sources);
    ``eta_per_shot`` (optional device f64 [n_shots]) replaces ``eta`` shot by shot.
    ``peers`` (optional ``(device int64 table of peer buffer addresses, count, record
    offset)``): the polish epilogue also writes the positions into the other ranks'
    buffers (spk_polish_shots; the engine's fused position all-gather)."""
    n_c, n_s, dims = coords.shape
    pin_idx, pin_val = _pin_arrays(cfg, dims)
    if pin_idx >= n_s:
        raise ValueError(f"pinned_index {pin_idx} out of range for N_s={n_s}")
    if n_s < 2:
        raise ValueError("projection needs at least 2 samples per shot")
    if tau is None:
        tau = 1.0 / stacked_operator_norm(n_s, pin_idx)
    if out is None:
        out = torch.empty_like(coords)
    nbytes = _native.query("spk_project_workspace_bytes", n_c, n_s, dims, int(trace is not None))
    ws = _device.workspace(nbytes, "project")
    pv = _native.f64_array(list(pin_val) + [0.0] * (3 - dims))
    if peers is not None:
        # FISTA, then the polish of every shot with the peer-writing epilogue
        table, n_peers, offset = peers
        _native.call("spk_project_fista", coords.data_ptr(), _device.ptr(grad), float(eta),
                     _device.ptr(eta_per_shot), out.data_ptr(), n_c, n_s, dims,
                     cfg.speed_bound, cfg.accel_bound, pin_idx, pv, cfg.n_pit, float(tau),
                     int(bool(cfg.monotone)), _device.ptr(trace), _device.ptr(nonfinite),
                     ws.data_ptr(), ws.numel(), _device.stream())
        _native.call("spk_polish_shots", out.data_ptr(), None, n_c, n_c, n_s, dims,
                     cfg.speed_bound, cfg.accel_bound, pin_idx, pv, 0.1 * cfg.feas_tol,
                     int(max_sweeps), _device.ptr(pos4), _device.ptr(sweeps), None,
                     table.data_ptr(), int(n_peers), int(offset), ws.data_ptr(), ws.numel(),
                     _device.stream())
        return out
    _native.call("spk_project_all", coords.data_ptr(), _device.ptr(grad), float(eta),
                 _device.ptr(eta_per_shot), out.data_ptr(), n_c, n_s, dims, cfg.speed_bound,
                 cfg.accel_bound, pin_idx, pv, cfg.n_pit, float(tau), int(bool(cfg.monotone)), 0.1 * cfg.feas_tol,
                 int(max_sweeps), _device.ptr(pos4), _device.ptr(sweeps), _device.ptr(trace),
                 _device.ptr(nonfinite), ws.data_ptr(), ws.numel(), _device.stream())
    return out


def project_shot(shot: np.ndarray, cfg: ProjectionConfig, return_trace: bool = False):
    """Project one (N_s, d) shot (projection.py:394-418); optionally the dual objective
    after every FISTA iteration."""
    shot = np.ascontiguousarray(shot, dtype=np.float64)
    if shot.ndim != 2:
        raise ValueError("shot must be (N_s, d)")
    dev_in = _device.h2d(shot[None])
    trace = None
    if return_trace:
        trace = torch.empty(cfg.n_pit, dtype=torch.float64, device=dev_in.device)
    out = project_device(dev_in, cfg, trace=trace)
    res = _device.d2h(out)[0]
    if return_trace:
        return res, _device.d2h(trace)
    return res


def project_pattern(k: SamplingPattern, cfg: ProjectionConfig) -> SamplingPattern:
    """Project every shot independently (projection.py:421-432); bit-exact shot
    independence holds because each shot is one CTA / one warp with no cross-shot
    state."""
    coords = np.ascontiguousarray(k.coords)
    out = project_device(_device.h2d(coords), cfg)
    return SamplingPattern(_device.d2h(out))


def residuals_device(coords: torch.Tensor, cfg: ProjectionConfig,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Device feasibility residuals -> tensor [amplitude, speed, accel, pin, max]."""
    n_c, n_s, dims = coords.shape
    pin_idx, pin_val = _pin_arrays(cfg, dims)
    if out is None:
        out = torch.empty(5, dtype=torch.float64, device=coords.device)
    ws = _device.workspace(_native.query("spk_residuals_workspace_bytes", n_c), "resid")
    pv = _native.f64_array(list(pin_val) + [0.0] * (3 - dims))
    _native.call("spk_feasibility_residuals", coords.data_ptr(), n_c, n_s, dims,
                 cfg.speed_bound, cfg.accel_bound, pin_idx, pv, out.data_ptr(),
                 ws.data_ptr(), ws.numel(), _device.stream())
    return out


def feasibility_residuals(k: SamplingPattern, cfg: ProjectionConfig) -> dict:
    """Max violation per constraint (projection.py:435-452)."""
    vals = _device.d2h(residuals_device(_device.h2d(k.coords), cfg))
    res = {"amplitude": float(vals[0]), "speed": float(vals[1]),
           "acceleration": float(vals[2])}
    if cfg.pin is not None:
        res["pin"] = float(vals[3])
    res["max"] = max(res.values())
    return res


def project_overlap_device(coords: torch.Tensor, cfg: ProjectionConfig, *, grad, eta,
                           out: torch.Tensor, pos4: torch.Tensor, nonfinite, field,
                           att_val: torch.Tensor, att_grad: torch.Tensor,
                           sweeps: torch.Tensor, order: torch.Tensor | None,
                           polish_streams, k2_streams, eta_per_shot=None, groups_out=None,
                           sm_busy=None, peers=None):
    """K3 with the lattice attraction (K2) of every shot started as soon as its polish
    group is done, so that K2 runs under the polish of the slower shots.

    The polish time of a shot varies by ~3x between shots and the iteration waits for the
    slowest, so SMs idle during that tail -- most of them on a rank with few shots
    (multi-GPU), the last waves' worth on one GPU.  Shots are
    polished in groups, longest first by the previous iteration's sweep counts
    (``order``, device int32; None = shot order), each group on its own high-priority
    stream, and each group's K2 (spk_grid_sums_shots) follows on a
    low-priority stream.  The projection itself is unchanged (bit-identical per shot);
    K2 writes ``att_val`` [n_shots * n_s] / ``att_grad`` [n_shots * n_s, d] for the NEW
    positions ``pos4``.  Returns ``(out, k2_events)``: the caller's stream has waited for
    the projection; wait on ``k2_events`` before reading ``att_val`` / ``att_grad``.
    ``sweeps`` receives this call's sweep counts.  ``groups_out`` (a list) receives
    ``(shot ids, polished event)`` per group in launch order, for work that may start as
    soon as a group's positions are final (the engine's pipelined K1).
    ``sm_busy`` (device int32 [256] of zeros, or None): the polish CTAs count themselves
    per SM and the K2 CTAs wait for an SM without polish CTAs, so K2 takes only the SMs
    the polish has left instead of sharing issue slots with it."""
    n_c, n_s, dims = coords.shape
    pin_idx, pin_val = _pin_arrays(cfg, dims)
    peer_table, n_peers, peer_offset = peers if peers is not None else (None, 0, 0)
    tau = 1.0 / stacked_operator_norm(n_s, pin_idx)
    nbytes = _native.query("spk_project_workspace_bytes", n_c, n_s, dims, 0)
    ws = _device.workspace(nbytes, "project")
    pv = _native.f64_array(list(pin_val) + [0.0] * (3 - dims))
    main = torch.cuda.current_stream()
    _native.call("spk_project_fista", coords.data_ptr(), _device.ptr(grad), float(eta),
                 _device.ptr(eta_per_shot), out.data_ptr(), n_c, n_s, dims, cfg.speed_bound,
                 cfg.accel_bound, pin_idx, pv, cfg.n_pit, float(tau), int(bool(cfg.monotone)),
                 None, _device.ptr(nonfinite), ws.data_ptr(), ws.numel(), main.cuda_stream)
    if order is None:
        order = torch.arange(n_c, dtype=torch.int32, device=coords.device)
    G = len(polish_streams)
    bounds = [n_c * g // G for g in range(G + 1)]
    fista_done = torch.cuda.Event()
    fista_done.record(main)
    w = field.device_sources()
    sides = field.sides
    n_cells = int(np.prod(sides))
    eps2 = float(field.kernel_eps ** 2)
    side_arr = _native.i64_array(sides)
    done = []
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        if hi <= lo:
            continue
        ids = order[lo:hi]
        ps, ks = polish_streams[g], k2_streams[g]
        ps.wait_event(fista_done)
        _native.call("spk_polish_shots", out.data_ptr(), ids.data_ptr(), hi - lo, n_c, n_s,
                     dims, cfg.speed_bound, cfg.accel_bound, pin_idx, pv, 0.1 * cfg.feas_tol,
                     MAX_POLISH_SWEEPS, pos4.data_ptr(), sweeps.data_ptr(),
                     _device.ptr(sm_busy), _device.ptr(peer_table), n_peers, peer_offset,
                     ws.data_ptr(), ws.numel(), ps.cuda_stream)
        polished = torch.cuda.Event()
        polished.record(ps)
        ks.wait_event(polished)
        if groups_out is not None:
            groups_out.append((ids, polished))
        kb = _native.query("spk_grid_sums_shots_workspace_bytes", hi - lo, n_s, n_cells)
        kws = _device.workspace(kb, f"k2_overlap_{g}")
        _native.call("spk_grid_sums_shots", pos4.data_ptr(), ids.data_ptr(), hi - lo, n_s,
                     w.data_ptr(), side_arr, dims, eps2, att_val.data_ptr(),
                     att_grad.data_ptr(), _device.ptr(sm_busy), kws.data_ptr(), kws.numel(),
                     ks.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(ks)
        # buffers used on the side streams stay reserved until that work completes, even
        # if the caller drops them first (caching-allocator stream semantics)
        for t, st in ((ids, ps), (ids, ks), (out, ps), (sweeps, ps), (pos4, ps), (pos4, ks),
                      (att_val, ks), (att_grad, ks)):
            t.record_stream(st)
        done.append((ps, ev))
    # the caller's stream waits for the polish only: K1 (which needs the gathered
    # positions, not K2) can then co-run with the tail of the SFU-bound K2 launches; the
    # returned events must be waited on before the K2 results are read
    k2_events = []
    for ps, ev in done:
        main.wait_stream(ps)
        k2_events.append(ev)
    return out, k2_events
