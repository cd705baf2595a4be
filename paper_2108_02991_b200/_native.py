"""ctypes binding of the C ABI in include/sparkling_b200.h.

The product path has no CPU fallback: if the shared library is missing or no CUDA device
is visible, every compute entry point raises.  PyTorch is used only for device memory,
streams and torch.distributed; all hot-path arithmetic runs in our own kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

_lock = threading.Lock()
_lib = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_flt = ctypes.c_float
c_size = ctypes.c_size_t
c_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/sparkling_b200.h one to one.
SIGNATURES = {
    "spk_version": (c_int, []),
    "spk_ipc_handle": (c_int, [c_vp, c_vp]),
    "spk_ipc_open": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "spk_ipc_close": (c_int, [c_vp]),
    "spk_last_error": (ctypes.c_char_p, []),
    "spk_nbody_workspace_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "spk_direct_sums": (c_int, [c_vp, c_i64, c_vp, c_i64, c_int, c_flt, c_vp, c_vp, c_vp,
                                c_size, c_vp]),
    "spk_grid_sums": (c_int, [c_vp, c_i64, c_vp, ctypes.POINTER(c_i64), c_int, c_flt, c_vp,
                              c_vp, c_vp, c_size, c_vp]),
    "spk_fused_sums": (c_int, [c_vp, c_i64, c_int, c_vp, ctypes.POINTER(c_i64), c_flt, c_vp,
                               c_i64, c_flt, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "spk_nbody_batched_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_i64]),
    "spk_fused_sums_batched": (c_int, [c_vp, c_i64, c_i64, c_int, c_vp, ctypes.POINTER(c_i64),
                                       c_flt, c_vp, c_i64, c_flt, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_size, c_vp]),
    "spk_combine_batched_workspace_bytes": (c_size, [c_i64, c_i64]),
    "spk_combine_gradient_batched": (c_int, [c_i64, c_i64, c_int, c_vp, c_vp, c_dbl, c_vp,
                                             c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             c_size, c_vp]),
    "spk_feasibility_residuals_batched": (c_int, [c_vp, c_i64, c_i64, c_int, c_int, c_dbl,
                                                  c_dbl, c_int, ctypes.POINTER(c_dbl), c_vp,
                                                  c_vp, c_size, c_vp]),
    "spk_pack_positions": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp]),
    "spk_build_grid_sources": (c_int, [c_vp, c_int, ctypes.POINTER(c_i64), c_vp, c_vp, c_vp]),
    "spk_combine_workspace_bytes": (c_size, [c_i64]),
    "spk_combine_gradient": (c_int, [c_i64, c_int, c_vp, c_vp, c_dbl, c_vp, c_vp, c_dbl,
                                     c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "spk_project_workspace_bytes": (c_size, [c_i64, c_int, c_int, c_int]),
    "spk_project_all": (c_int, [c_vp, c_vp, c_dbl, c_vp, c_vp, c_i64, c_int, c_int, c_dbl, c_dbl,
                                c_int, ctypes.POINTER(c_dbl), c_int, c_dbl, c_int, c_dbl,
                                c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "spk_project_fista": (c_int, [c_vp, c_vp, c_dbl, c_vp, c_vp, c_i64, c_int, c_int, c_dbl,
                                  c_dbl, c_int, ctypes.POINTER(c_dbl), c_int, c_dbl, c_int,
                                  c_vp, c_vp, c_vp, c_size, c_vp]),
    "spk_polish_shots": (c_int, [c_vp, c_vp, c_i64, c_i64, c_int, c_int, c_dbl, c_dbl, c_int,
                                 ctypes.POINTER(c_dbl), c_dbl, c_int, c_vp, c_vp, c_vp, c_vp,
                                 c_int, c_i64, c_vp, c_size, c_vp]),
    "spk_grid_sums_shots_workspace_bytes": (c_size, [c_i64, c_int, c_i64]),
    "spk_grid_sums_shots": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, ctypes.POINTER(c_i64),
                                    c_int, ctypes.c_float, c_vp, c_vp, c_vp, c_vp, c_size,
                                    c_vp]),
    "spk_residuals_workspace_bytes": (c_size, [c_i64]),
    "spk_feasibility_residuals": (c_int, [c_vp, c_i64, c_int, c_int, c_dbl, c_dbl, c_int,
                                          ctypes.POINTER(c_dbl), c_vp, c_vp, c_size, c_vp]),
    "spk_upsample_shots": (c_int, [c_vp, c_vp, c_i64, c_int, c_int, c_vp]),
    "spk_field_eval": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_i64, c_int, c_vp, c_vp,
                               c_vp, c_vp]),
    "spk_tree_keys": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp]),
    "spk_tree_sort_workspace_bytes": (c_size, [c_i64]),
    "spk_tree_sort": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_size, c_vp]),
    "spk_tree_gather": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "spk_tree_boxes": (c_int, [c_vp, c_i64, c_vp, c_vp, c_int, c_vp, c_vp]),
    "spk_tree_p2m_workspace_bytes": (c_size, [c_i64, c_int, c_int]),
    "spk_tree_p2m": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_int, c_int,
                             c_vp, c_vp, c_size, c_vp]),
    "spk_tree_eval": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                              c_int, c_flt, c_vp, c_vp, c_vp]),
    "spk_tree_host_groups": (c_i64, [c_vp, c_i64, c_vp, c_vp]),
    "spk_tree_build_workspace_bytes": (c_size, [c_i64, c_i64]),
    "spk_tree_build": (c_int, [c_vp, c_i64, c_int, c_i64, c_int, c_i64, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "spk_tree_groups": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp,
                                c_vp, c_vp, c_size, c_vp]),
    "spk_tree_cheb_targets": (c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp]),
    "spk_tree_parent_ids": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "spk_tree_l2p": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_vp,
                             c_vp, c_vp]),
    "spk_nudft_workspace_bytes": (c_size, [c_i64, c_int, ctypes.POINTER(c_i64)]),
    "spk_nudft_adjoint": (c_int, [c_vp, c_vp, c_i64, c_int, ctypes.POINTER(c_i64), c_int, c_vp,
                                  c_vp, c_size, c_vp]),
    "spk_nudft_forward": (c_int, [c_vp, c_vp, c_i64, c_int, ctypes.POINTER(c_i64), c_int, c_vp,
                                  c_vp, c_size, c_vp]),
    "spk_dcf_update": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "spk_psf_magnitude": (c_int, [c_vp, c_i64, c_dbl, c_vp, c_vp]),
    "spk_tree_host_levels": (c_i64, [c_vp, c_vp]),
    "spk_tree_host_leaf_nodes": (None, [c_vp, c_vp]),
    "spk_tree_node_boxes": (c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                    c_vp, c_int, c_vp, c_vp]),
    "spk_tree_plan_workspace_bytes": (c_size, [c_i64, c_i64]),
    "spk_tree_plan_count": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl,
                                    c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_int, c_vp, c_vp, c_size, c_vp]),
    "spk_tree_plan_write": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl,
                                    c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                                    c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp]),
    "spk_tree_host_slot_nodes": (None, [c_vp, c_vp]),
    "spk_tree_group_size": (c_int, []),
    "spk_tree_host_build": (c_vp, [c_vp, c_i64, c_int, c_i64, c_int]),
    "spk_tree_host_free": (None, [c_vp]),
    "spk_tree_host_sizes": (None, [c_vp, c_vp]),
    "spk_tree_host_leaves": (None, [c_vp, c_vp, c_vp]),
    "spk_tree_host_nodes": (None, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "spk_tree_host_set_leaf_boxes": (None, [c_vp, c_vp]),
    "spk_tree_host_plan": (c_int, [c_vp, c_i64, c_vp, c_dbl, c_int, c_i64, c_vp]),
    "spk_tree_host_export_plan": (None, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                         c_vp]),
}


# Kernels launched per successful call of each entry point (for gpu_launches accounting).
LAUNCHES = {
    "spk_direct_sums": 2, "spk_grid_sums": 2, "spk_fused_sums": 3, "spk_pack_positions": 1,
    "spk_build_grid_sources": 1, "spk_combine_gradient": 2, "spk_project_all": 2,
    "spk_feasibility_residuals": 2, "spk_upsample_shots": 1, "spk_field_eval": 1,
    "spk_fused_sums_batched": 3, "spk_combine_gradient_batched": 2,
    "spk_feasibility_residuals_batched": 2,
    "spk_tree_keys": 1, "spk_tree_sort": 10, "spk_tree_gather": 1, "spk_tree_boxes": 1,
    "spk_tree_p2m": 2, "spk_tree_eval": 1, "spk_tree_plan_count": 9, "spk_tree_node_boxes": 1,
    "spk_tree_groups": 11, "spk_tree_cheb_targets": 1, "spk_tree_parent_ids": 1,
    "spk_tree_l2p": 1,
    "spk_tree_plan_write": 2, "spk_nudft_adjoint": 2, "spk_nudft_forward": 2,
    "spk_dcf_update": 1, "spk_psf_magnitude": 1,
    "spk_project_fista": 1, "spk_polish_shots": 1, "spk_grid_sums_shots": 4,
}
_launched = [0]


def reset_launch_count() -> None:
    _launched[0] = 0


def launch_count() -> int:
    return _launched[0]


def add_launches(k: int) -> None:
    """Account kernels whose number depends on the call (e.g. one per tree level)."""
    _launched[0] += int(k)


class NativeError(RuntimeError):
    """A nonzero status returned through the C ABI."""


def library_path() -> str:
    return _build.LIB_PATH


def load(build_if_missing: bool = True):
    """Load (building first if needed) the sm_100a shared library."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB_PATH
            if not os.path.exists(path):
                if not build_if_missing:
                    raise ImportError(f"{path} missing; run __graft_entry__.build()")
                _build.build()
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def call(name: str, *args) -> None:
    """Call a status-returning entry point; raise on nonzero status."""
    lib = load()
    status = getattr(lib, name)(*args)
    if status == 0:
        _launched[0] += LAUNCHES.get(name, 0)
    if status != 0:
        msg = lib.spk_last_error().decode(errors="replace")
        if status == 1:
            raise ValueError(f"{name}: {msg}")
        raise NativeError(f"{name} failed with status {status}: {msg}")


def query(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))


def f64_array(values):
    arr = (c_dbl * max(1, len(values)))()
    for i, v in enumerate(values):
        arr[i] = float(v)
    return arr


def i64_array(values):
    arr = (c_i64 * max(1, len(values)))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr
