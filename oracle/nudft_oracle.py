"""numpy restatement of the reference's direct NUDFT and density compensation.
TEST INFRASTRUCTURE ONLY (imported by tests/ as the checker, never by the product).

Reference: /root/reference/pkg/src/vdtraj/analysis.py -- nudft_adjoint (:41-55),
nudft_forward (:58-69), density_compensation (:72-96), compute_psf magnitudes
(:112-137).  Written as one dense phase matrix exp(i pi K R^T) over every voxel offset
R (r_a = 0..n_a-1 minus n_a // 2), not as the reference's per-axis tables; it agrees
with the reference to ~1e-13 relative on the golden fixtures (tests/golden/analysis.npz,
checked in tests/test_analysis_host.py).  Intended for p x voxels up to ~1e7.
"""

from __future__ import annotations

import numpy as np


def _offsets(grid_shape) -> np.ndarray:
    axes = [np.arange(n) - n // 2 for n in grid_shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1).astype(np.float64)


def phase_matrix(points: np.ndarray, grid_shape) -> np.ndarray:
    """E[i, r] = exp(i pi k_i . r) for every sample and voxel offset."""
    return np.exp(1j * np.pi * (np.asarray(points, np.float64) @ _offsets(grid_shape).T))


def nudft_adjoint(points, weights, grid_shape) -> np.ndarray:
    e = phase_matrix(points, grid_shape)
    return (np.asarray(weights, np.complex128) @ e).reshape(tuple(grid_shape))


def nudft_forward(points, image) -> np.ndarray:
    e = phase_matrix(points, image.shape)
    return e.conj() @ np.asarray(image, np.complex128).ravel()


def density_compensation(points, grid_shape, iters) -> np.ndarray:
    e = phase_matrix(points, grid_shape)
    w = np.ones(e.shape[0])
    for _ in range(iters):
        back = e.conj() @ (w @ e)
        w = w / np.maximum(np.abs(back), 1e-12)
    return w


def psf_values(points, grid_shape, weights=None) -> np.ndarray:
    w = np.ones(len(points)) if weights is None else np.asarray(weights)
    return np.abs(nudft_adjoint(points, w, grid_shape) / np.sum(w))
