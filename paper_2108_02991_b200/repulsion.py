"""Repulsion term: the all-pairs N-body K1 on the B200.

Cost (1/(2p^2)) sum_i sum_j sqrt(|x_i - x_j|^2 + eps^2) and gradient
(1/p^2) sum_j (x_i - x_j)/sqrt(...) -- the reference's definitions
(/root/reference/pkg/src/vdtraj/repulsion.py:1-7, 72-87).  The pair sums run in
``spk_direct_sums`` (csrc/nbody.cu); the normalisation is done here with numpy exactly
like the reference, so outputs are float64 numpy arrays owned by the caller.

``backend="tree"`` runs the GPU treecode (tree.py, csrc/tree.cu) with the reference's
contract and control flow (repulsion.py:90-200): automatic (order, theta) from
``tree_precision``; with an explicit ``interp_order`` the result is probed against exact
sums on 64 strided targets and the order escalated (warning) or the evaluation dropped
to direct summation; problems of at most ``leaf_size`` particles are evaluated directly,
and so are problems below ``tree.DIRECT_BELOW`` sources, where the exact B200 kernel is
faster than building a tree (the precision contract holds a fortiori).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native, tree
from .core import SamplingPattern

MAX_INTERP_ORDER = 8


@dataclass
class RepulsionConfig:
    """Same fields and validation as the reference (repulsion.py:33-60).

    ``backend="tree"`` meets ``tree_precision`` (relative error of the cost and of the
    gradient l2 norm) as checked by a 64-target probe against the exact kernel: on every
    call through the public API, and inside ``optimize`` on the first call of a level and
    then every ``tree.REPROBE_EVERY`` iterations (between probes the validated row is
    trusted, as the reference trusts its table)."""

    kernel_eps: float = 1e-3
    backend: str = "direct"
    tree_precision: float = 1e-4
    leaf_size: int = 192
    interp_order: int | None = None

    def __post_init__(self):
        if self.kernel_eps < 0:
            raise ValueError("kernel_eps must be >= 0")
        if self.backend not in ("direct", "tree"):
            raise ValueError(f"backend must be 'direct' or 'tree', got {self.backend!r}")
        if self.tree_precision <= 0:
            raise ValueError("tree_precision must be positive")
        if self.leaf_size < 8:
            raise ValueError("leaf_size must be >= 8")
        if self.interp_order is not None and not 2 <= self.interp_order <= MAX_INTERP_ORDER:
            raise ValueError(f"interp_order must be in [2, {MAX_INTERP_ORDER}]")


def _points(k) -> np.ndarray:
    if isinstance(k, SamplingPattern):
        return np.ascontiguousarray(k.points())
    pts = np.ascontiguousarray(k, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] not in (2, 3):
        raise ValueError("expected a SamplingPattern or a (p, d) array")
    return pts


def direct_sums_device(tgt4: torch.Tensor, src4: torch.Tensor, dims: int, eps2: float):
    """Raw K1 sums on device buffers (float4 targets / sources) -> (val, grad) fp64.

    Device-level counterpart of ``_treecode.direct_sums`` / ``direct_sums_subset``
    (_treecode.py:474-534)."""
    n_t, n_s = tgt4.shape[0], src4.shape[0]
    val = torch.empty(n_t, dtype=torch.float64, device=tgt4.device)
    grad = torch.empty((n_t, dims), dtype=torch.float64, device=tgt4.device)
    nbytes = _native.query("spk_nbody_workspace_bytes", n_t, 0, n_s)
    ws = _device.workspace(nbytes, "nbody")
    _native.call("spk_direct_sums", tgt4.data_ptr(), n_t, src4.data_ptr(), n_s, dims,
                 float(eps2), val.data_ptr(), grad.data_ptr(), ws.data_ptr(), ws.numel(),
                 _device.stream())
    return val, grad


def eval_repulsion_direct(k, eps: float = 1e-3) -> tuple[float, np.ndarray]:
    """Exact O(p^2) repulsion cost and gradient (repulsion.py:72-87)."""
    pts = _points(k)
    p = pts.shape[0]
    if p < 1:
        raise ValueError("need at least one particle")
    coords = _device.h2d(pts)
    pos4 = _device.pack_positions(coords)
    val, grad = direct_sums_device(pos4, pos4, pts.shape[1], eps * eps)
    val_h = _device.d2h(val)
    grad_h = _device.d2h(grad)
    cost = float(val_h.sum() / (2.0 * p * p))
    grad_h /= p * p
    return cost, grad_h


def auto_tree_params(precision: float, dims: int = 3) -> tuple[int, float]:
    """Interpolation order and opening threshold for a precision (repulsion.py:90-96);
    (MAX_INTERP_ORDER, 0.0) -- i.e. exact sums -- below the fp32 floor."""
    params = tree.auto_params(precision, dims)
    return params if params is not None else (MAX_INTERP_ORDER, 0.0)


def _probe_error(tgt4, src4, dims, eps2, val, grad) -> tuple[float, float]:
    """Relative error vs exact K1 on 64 strided targets (repulsion.py:151-162)."""
    n = tgt4.shape[0]
    stride = max(1, n // 64)
    idx = torch.arange(0, n, stride, device=tgt4.device)[:64]
    v_ref, g_ref = direct_sums_device(tgt4[idx].contiguous(), src4, dims, eps2)
    v_ref, g_ref = _device.d2h(v_ref), _device.d2h(g_ref)
    v, g = _device.d2h(val[idx]), _device.d2h(grad[idx])
    err_val = abs(v.sum() - v_ref.sum()) / max(abs(v_ref.sum()), 1e-300)
    err_grad = np.linalg.norm(g - g_ref) / max(np.linalg.norm(g_ref), 1e-300)
    return float(err_val), float(err_grad)


def tree_sums_checked(tgt4, src4, dims: int, cfg: RepulsionConfig, *,
                      return_groups: bool = False, row_cache: dict | None = None):
    """Device raw sums for backend="tree" with the reference's order selection, probe,
    escalation and direct fallback (repulsion.py:165-200).  With ``return_groups`` also
    returns the target groups (tree.TargetGroups, or None on the direct path) so that a
    treecode attraction can reuse the targets' sort.  ``row_cache`` (the optimizer's):
    the auto-mode probe runs on the first call per (sizes, precision) and its validated
    table row is reused, with a re-probe every ``tree.REPROBE_EVERY`` calls (the points
    move within a level); without a cache (the public API) every call probes."""
    eps2 = cfg.kernel_eps * cfg.kernel_eps
    params = tree.auto_params(cfg.tree_precision, dims)
    n_src = src4.shape[0]

    def done(val, grad, tg=None):
        return (val, grad, tg) if return_groups else (val, grad)

    if n_src <= max(cfg.leaf_size, tree.DIRECT_BELOW) or params is None:
        # small problems (exact kernel is faster) and precisions below the fp32 floor
        return done(*direct_sums_device(tgt4, src4, dims, eps2))
    auto_order, theta = params
    rows = tree.AUTO_PARAMS_2D if dims == 2 else tree.AUTO_PARAMS
    ckey = ("rep", tgt4.shape[0], n_src, dims, cfg.tree_precision)
    cached, reprobe = (None, False) if cfg.interp_order is not None else \
        tree.cached_row(row_cache, ckey)
    if cached is not None:
        if cached >= len(rows):
            return done(*direct_sums_device(tgt4, src4, dims, eps2))
        _, auto_order, theta = rows[cached]
    order = cfg.interp_order if cfg.interp_order is not None else auto_order
    same = tgt4.data_ptr() == src4.data_ptr() and tgt4.shape[0] == n_src
    src = tree.SourceTree(src4, dims)
    cap = tree.far_parent_cap(tgt4.shape[0])
    tg = tree.TargetGroups(tgt4, dims, same_as=src if same else None, parent_cap=cap)
    # the far level needs every node's proxies (static), the plain walk builds its own
    val, grad = tree.tree_eval(tg, src, order, theta, eps2, static=cap is not None)
    if cfg.interp_order is None and (cached is None or reprobe):
        # Extension of the reference (which trusts its table in auto mode): the same
        # 64-target probe, and on a miss the next stricter (order, theta) row, then the
        # exact kernel.  The table is calibrated on SPARKLING-like, uniform and radial
        # clouds; dense blobs whose sub-boxes all sit at the opening ratio can exceed it
        # (profiles/r01_tree_fuzz_sweep.txt).  Inside optimize() the validated row is
        # re-probed every tree.REPROBE_EVERY calls, starting from that row.
        k = cached if reprobe else next(i for i, r in enumerate(rows)
                                        if cfg.tree_precision >= r[0])
        err_val, err_grad = _probe_error(tgt4, src4, dims, eps2, val, grad)
        while max(err_val, err_grad) > cfg.tree_precision:
            k += 1
            if k >= len(rows):
                warnings.warn(
                    f"tree backend (auto) reached relative error {max(err_val, err_grad):.2e}"
                    f" > {cfg.tree_precision:.2e} on the probe at every table row; falling "
                    f"back to direct summation")
                tree.store_row(row_cache, ckey, k)
                return done(*direct_sums_device(tgt4, src4, dims, eps2), tg)
            _, order, theta = rows[k]
            warnings.warn(
                f"tree backend (auto) reached relative error {max(err_val, err_grad):.2e} > "
                f"{cfg.tree_precision:.2e} on the probe; tightening to interp_order={order}, "
                f"theta={theta}")
            val, grad = tree.tree_eval(tg, src, order, theta, eps2, static=cap is not None)
            err_val, err_grad = _probe_error(tgt4, src4, dims, eps2, val, grad)
        tree.store_row(row_cache, ckey, k)
    if cfg.interp_order is not None:
        err_val, err_grad = _probe_error(tgt4, src4, dims, eps2, val, grad)
        while max(err_val, err_grad) > cfg.tree_precision and order < MAX_INTERP_ORDER:
            order += 1
            warnings.warn(
                f"tree backend at interp_order={order - 1} reached relative error "
                f"{max(err_val, err_grad):.2e} > {cfg.tree_precision:.2e}; "
                f"escalating to order {order}")
            val, grad = tree.tree_eval(tg, src, order, theta, eps2, static=cap is not None)
            err_val, err_grad = _probe_error(tgt4, src4, dims, eps2, val, grad)
        if max(err_val, err_grad) > cfg.tree_precision:
            warnings.warn(
                f"tree backend cannot reach precision {cfg.tree_precision:.2e} at "
                f"interp_order {MAX_INTERP_ORDER}; falling back to direct summation")
            return done(*direct_sums_device(tgt4, src4, dims, eps2), tg)
    return done(val, grad, tg)


def eval_repulsion_tree(k, cfg: RepulsionConfig) -> tuple[float, np.ndarray]:
    """Repulsion cost and gradient through the GPU treecode (repulsion.py:165-200):
    within ``cfg.tree_precision`` relative error of :func:`eval_repulsion_direct` on the
    cost and the gradient l2 norm; at most ``leaf_size`` particles -> direct (bitwise)."""
    pts = _points(k)
    p = pts.shape[0]
    if p <= cfg.leaf_size:
        return eval_repulsion_direct(pts, cfg.kernel_eps)
    pos4 = _device.pack_positions(_device.h2d(pts))
    val, grad = tree_sums_checked(pos4, pos4, pts.shape[1], cfg)
    val_h = _device.d2h(val)
    grad_h = _device.d2h(grad)
    cost = float(val_h.sum() / (2.0 * p * p))
    grad_h /= p * p
    return cost, grad_h


def eval_repulsion(k, cfg: RepulsionConfig) -> tuple[float, np.ndarray]:
    """Dispatch on ``cfg.backend`` (repulsion.py:203-207)."""
    if cfg.backend == "tree":
        return eval_repulsion_tree(k, cfg)
    return eval_repulsion_direct(k, cfg.kernel_eps)
