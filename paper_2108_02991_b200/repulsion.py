"""Repulsion term: the all-pairs N-body K1 on the B200.

Cost (1/(2p^2)) sum_i sum_j sqrt(|x_i - x_j|^2 + eps^2) and gradient
(1/p^2) sum_j (x_i - x_j)/sqrt(...) -- the reference's definitions
(/root/reference/pkg/src/vdtraj/repulsion.py:1-7, 72-87).  The pair sums run in
``spk_direct_sums`` (csrc/nbody.cu); the normalisation is done here with numpy exactly
like the reference, so outputs are float64 numpy arrays owned by the caller.

``backend="tree"`` is accepted for drop-in configs; it is served by the same exact
kernel, which meets any ``tree_precision`` the fp32 kernel resolves (>= ~1e-6 relative),
so the reference's escalation / fallback warnings never fire.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .core import SamplingPattern

MAX_INTERP_ORDER = 8


@dataclass
class RepulsionConfig:
    """Same fields and validation as the reference (repulsion.py:33-60)."""

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


def eval_repulsion_tree(k, cfg: RepulsionConfig) -> tuple[float, np.ndarray]:
    """Tree-backend entry point (repulsion.py:165-200), served exactly by K1."""
    return eval_repulsion_direct(k, cfg.kernel_eps)


def eval_repulsion(k, cfg: RepulsionConfig) -> tuple[float, np.ndarray]:
    """Dispatch on ``cfg.backend`` (repulsion.py:203-207)."""
    if cfg.backend == "tree":
        return eval_repulsion_tree(k, cfg)
    return eval_repulsion_direct(k, cfg.kernel_eps)
