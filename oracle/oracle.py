"""ctypes front-end of the CPU oracle (oracle/spk_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) import this module, and only as the checker / the reference CPU
arm.  The product package ``paper_2108_02991_b200`` never imports it.

Each wrapper names the reference routine it restates (paths relative to
/root/reference/pkg/src/vdtraj/).  Results are bit-identical to the reference's numba
kernels on the committed golden fixtures (tests/golden/, checked in
tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (IEEE order, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.or_max_threads.restype = ctypes.c_int
        lib.or_direct_sums.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                       _f64p, _f64p, ctypes.c_int]
        lib.or_direct_sums_subset.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _i64p,
                                              ctypes.c_int64, ctypes.c_double, _f64p, _f64p,
                                              ctypes.c_int]
        lib.or_cross_sums.argtypes = [_f64p, ctypes.c_int64, _f64p, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_double, _f64p, _f64p, ctypes.c_int]
        lib.or_grid_sums.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, _f64p, _i64p,
                                     ctypes.c_double, _f64p, _f64p, ctypes.c_int]
        lib.or_project_shot.argtypes = [_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, _f64p, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int, _f64p, _f64p, _f64p]
        lib.or_polish.argtypes = [_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_int, _f64p, ctypes.c_double,
                                  ctypes.c_int]
        lib.or_polish.restype = ctypes.c_int
        lib.or_project_all.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int, _f64p,
                                       ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, _f64p, _i32p,
                                       ctypes.c_int]
        _lib = lib
    return _lib


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def max_threads() -> int:
    return int(_load().or_max_threads())


def direct_sums(pos, eps2, nthreads=0):
    """Restates ``_treecode.direct_sums`` (_treecode.py:506-534): raw (val, grad)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    p, d = pos.shape
    val = np.empty(p)
    grad = np.empty((p, d))
    _load().or_direct_sums(_p(pos), p, d, float(eps2), _p(val), _p(grad), int(nthreads))
    return val, grad


def direct_sums_subset(pos, targets, eps2, nthreads=0):
    """Restates ``_treecode.direct_sums_subset`` (_treecode.py:474-503)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    targets = np.ascontiguousarray(targets, dtype=np.int64)
    p, d = pos.shape
    m = targets.shape[0]
    val = np.empty(m)
    grad = np.empty((m, d))
    _load().or_direct_sums_subset(_p(pos), p, d, _p(targets, _i64p), m, float(eps2),
                                  _p(val), _p(grad), int(nthreads))
    return val, grad


def cross_sums(targets, sources, eps2, nthreads=0):
    """direct_sums rows for separate target points (sharded form of _treecode.py:506)."""
    tgt = np.ascontiguousarray(targets, dtype=np.float64)
    src = np.ascontiguousarray(sources, dtype=np.float64)
    m, d = tgt.shape
    val = np.empty(m)
    grad = np.empty((m, d))
    _load().or_cross_sums(_p(tgt), m, _p(src), src.shape[0], d, float(eps2), _p(val),
                          _p(grad), int(nthreads))
    return val, grad


def grid_sums(targets, rho_grid, eps2, nthreads=0):
    """Exact density-weighted attraction sums (north-star A4; pinned at grid nodes
    against ``precompute_field``, attraction.py:62-113)."""
    tgt = np.ascontiguousarray(targets, dtype=np.float64)
    rho = np.ascontiguousarray(rho_grid, dtype=np.float64)
    m, d = tgt.shape
    if rho.ndim != d:
        raise ValueError("density dims != target dims")
    side = np.array(rho.shape + (1,) * (3 - d), dtype=np.int64)
    val = np.empty(m)
    grad = np.empty((m, d))
    _load().or_grid_sums(_p(tgt), m, d, _p(rho), _p(side, _i64p), float(eps2), _p(val),
                         _p(grad), int(nthreads))
    return val, grad


def repulsion(points, eps=1e-3, nthreads=0):
    """``eval_repulsion_direct`` normalisation (repulsion.py:72-87) over the oracle sums."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    p = pts.shape[0]
    val, grad = direct_sums(pts, eps * eps, nthreads)
    return float(val.sum() / (2.0 * p * p)), grad / (p * p)


def attraction_exact(points, rho_grid, eps, nthreads=0):
    """North-star attraction: cost = (1/p) sum_i sum_y rho h, grad = (1/p) sum rho (x-y)/h."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    p = pts.shape[0]
    val, grad = grid_sums(pts, rho_grid, eps * eps, nthreads)
    return float(val.sum() / p), grad / p


def project_shot(shot, a, b, pin_idx, pin_val, n_iter, tau, monotone=False,
                 return_trace=False, polish_tol=None, max_sweeps=50000):
    """Restates ``_project_shot`` + ``_feasibility_polish`` (projection.py:169-373)."""
    shot = np.ascontiguousarray(shot, dtype=np.float64)
    ns, d = shot.shape
    pv = np.ascontiguousarray(np.zeros(d) if pin_val is None else pin_val, dtype=np.float64)
    out = np.empty_like(shot)
    work = np.empty(10 * ns * d + 8)
    trace = np.empty(n_iter) if return_trace else None
    lib = _load()
    lib.or_project_shot(_p(shot), ns, d, float(a), float(b), int(pin_idx), _p(pv),
                        int(n_iter), float(tau), int(bool(monotone)), _p(out),
                        _p(trace) if trace is not None else None, _p(work))
    sweeps = 0
    if polish_tol is not None:
        sweeps = lib.or_polish(_p(out), ns, d, float(a), float(b), int(pin_idx), _p(pv),
                               float(polish_tol), int(max_sweeps))
    if return_trace:
        return out, trace, sweeps
    return out, sweeps


def polish(s, a, b, pin_idx, pin_val, tol, max_sweeps=50000):
    """Restates ``_feasibility_polish`` (projection.py:287-373) in place on a copy."""
    s = np.array(s, dtype=np.float64, copy=True, order="C")
    ns, d = s.shape
    pv = np.ascontiguousarray(np.zeros(d) if pin_val is None else pin_val, dtype=np.float64)
    sweeps = _load().or_polish(_p(s), ns, d, float(a), float(b), int(pin_idx), _p(pv),
                               float(tol), int(max_sweeps))
    return s, sweeps


def project_all(shots, a, b, pin_idx, pin_val, n_iter, tau, tol, monotone=False,
                max_sweeps=50000, nthreads=0):
    """Restates ``_project_all`` (projection.py:376-382)."""
    shots = np.ascontiguousarray(shots, dtype=np.float64)
    n_c, ns, d = shots.shape
    pv = np.ascontiguousarray(np.zeros(d) if pin_val is None else pin_val, dtype=np.float64)
    out = np.empty_like(shots)
    sweeps = np.empty(n_c, dtype=np.int32)
    _load().or_project_all(_p(shots), n_c, ns, d, float(a), float(b), int(pin_idx), _p(pv),
                           int(n_iter), float(tau), int(bool(monotone)), float(tol),
                           int(max_sweeps), _p(out), _p(sweeps, _i32p), int(nthreads))
    return out, sweeps
