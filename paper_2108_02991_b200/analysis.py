"""Pattern analysis on the B200: density compensation, point spread function, metrics.

Mirrors /root/reference/pkg/src/vdtraj/analysis.py (same names, arguments, budget guard
and exceptions).  The nonuniform DFTs -- the only O(p x voxels) work -- run in our
kernels (csrc/nudft.cu: generated-operand complex products).  ``precision="fp64"`` (the
default) computes in fp64 like the reference's complex128 numpy; ``"mixed"`` uses fp32
products with fp64 phases and accumulation (~1e-6 relative, about twice as fast) -- not
suitable for density_compensation, whose fixed-point iteration amplifies that noise by
~1e6.  The metrics are O(voxels) host code on the returned magnitudes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .core import HardwareSpec, SamplingPattern, resample_to_dwell
from .density import TargetDensity

DB_CAP = 300.0
PRECISIONS = {"fp64": 0, "mixed": 1}  # SPK_NUDFT_FP64 / SPK_NUDFT_MIXED
# p * grid-voxel budget of the direct DFT before allow_slow is required (analysis.py:18-19)
DFT_BUDGET = 1 << 31


def _check_budget(p: int, grid_shape, allow_slow: bool) -> None:
    voxels = int(np.prod(grid_shape))
    if p * voxels > DFT_BUDGET and not allow_slow:
        raise ValueError(
            f"direct DFT of {p} samples on a {tuple(grid_shape)} grid "
            f"({p * voxels:.2e} sample-voxel products) exceeds the budget; "
            f"pass allow_slow=True (CLI: --allow-slow) to run anyway")


def _grid(grid_shape, dims: int):
    shape = tuple(int(n) for n in grid_shape)
    if len(shape) != dims:
        raise ValueError(f"grid_shape {shape} does not match {dims}-D points")
    if min(shape) < 1:
        raise ValueError("grid sizes must be positive")
    return shape


def _complex_dev(values, n: int) -> torch.Tensor:
    """Host complex (or real) array -> device interleaved fp64 [n, 2]."""
    c = np.asarray(values, dtype=np.complex128).reshape(-1)
    if c.shape[0] != n:
        raise ValueError(f"expected {n} values, got {c.shape[0]}")
    return _device.h2d(np.ascontiguousarray(c.view(np.float64).reshape(n, 2)))


def _to_complex(t: torch.Tensor, shape) -> np.ndarray:
    return np.ascontiguousarray(_device.d2h(t)).view(np.complex128).reshape(shape)


def _mode(precision: str) -> int:
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {tuple(PRECISIONS)}, got {precision!r}")
    return PRECISIONS[precision]


def nudft_adjoint_device(pts: torch.Tensor, w: torch.Tensor, grid_shape,
                         precision: str = "fp64") -> torch.Tensor:
    """Device adjoint NUDFT: pts [p, d] f64, w [p, 2] f64 (complex) -> [prod(grid), 2]."""
    mode = _mode(precision)
    p, dims = pts.shape
    shape = _grid(grid_shape, dims)
    g = _native.i64_array(shape)
    out = torch.empty((int(np.prod(shape)), 2), dtype=torch.float64, device=pts.device)
    ws = _device.workspace(_native.query("spk_nudft_workspace_bytes", p, dims, g), "nudft")
    _native.call("spk_nudft_adjoint", pts.data_ptr(), w.data_ptr(), p, dims, g, mode,
                 out.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream())
    return out


def nudft_forward_device(pts: torch.Tensor, img: torch.Tensor, grid_shape,
                         precision: str = "fp64") -> torch.Tensor:
    """Device forward NUDFT: img [prod(grid), 2] f64 (complex) -> [p, 2]."""
    mode = _mode(precision)
    p, dims = pts.shape
    shape = _grid(grid_shape, dims)
    g = _native.i64_array(shape)
    out = torch.empty((p, 2), dtype=torch.float64, device=pts.device)
    ws = _device.workspace(_native.query("spk_nudft_workspace_bytes", p, dims, g), "nudft")
    _native.call("spk_nudft_forward", pts.data_ptr(), img.data_ptr(), p, dims, g, mode,
                 out.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream())
    return out


def _points(points) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] not in (2, 3):
        raise ValueError("points must be (p, 2) or (p, 3)")
    return pts


def nudft_adjoint(points: np.ndarray, weights: np.ndarray, grid_shape,
                  allow_slow: bool = False, precision: str = "fp64") -> np.ndarray:
    """Grid weighted samples onto the image grid (analysis.py:41-55):
    out[r] = sum_i w_i exp(i pi k_i . r), r_a = 0..n_a-1 minus n_a // 2."""
    pts = _points(points)
    p, dims = pts.shape
    _check_budget(p, grid_shape, allow_slow)
    shape = _grid(grid_shape, dims)
    out = nudft_adjoint_device(_device.h2d(pts), _complex_dev(weights, p), shape, precision)
    return _to_complex(out, shape)


def nudft_forward(points: np.ndarray, image: np.ndarray, allow_slow: bool = False,
                  precision: str = "fp64") -> np.ndarray:
    """Sample an image-grid function at the trajectory points (analysis.py:58-69):
    f_i = sum_r image[r] exp(-i pi k_i . r)."""
    pts = _points(points)
    p, dims = pts.shape
    image = np.asarray(image)
    _check_budget(p, image.shape, allow_slow)
    shape = _grid(image.shape, dims)
    out = nudft_forward_device(_device.h2d(pts), _complex_dev(image, int(np.prod(shape))),
                               shape, precision)
    return _to_complex(out, (p,))


def density_compensation(k: SamplingPattern, grid_shape, iters: int = 10,
                         allow_slow: bool = False, precision: str = "fp64") -> np.ndarray:
    """Iterative density-compensation weights (analysis.py:72-96): start from ones, then
    w <- w / max(|forward(adjoint(w))|, 1e-12), ``iters`` times; device-resident."""
    if iters < 1:
        raise ValueError("iters must be >= 1")
    _mode(precision)
    pts = k.points()
    if pts.shape[0] == 0:
        raise ValueError("empty sampling pattern")
    p, dims = pts.shape
    _check_budget(p, grid_shape, allow_slow)
    shape = _grid(grid_shape, dims)
    d_pts = _device.h2d(np.ascontiguousarray(pts))
    w = torch.zeros((p, 2), dtype=torch.float64, device=d_pts.device)
    w[:, 0] = 1.0
    for _ in range(iters):
        gridded = nudft_adjoint_device(d_pts, w, shape, precision)
        back = nudft_forward_device(d_pts, gridded, shape, precision)
        _native.call("spk_dcf_update", w.data_ptr(), back.data_ptr(), p, _device.stream())
    return np.ascontiguousarray(_device.d2h(w[:, 0]))


@dataclass
class PsfVolume:
    """Point spread function magnitudes on the image grid (analysis.py:99-109)."""

    values: np.ndarray
    peak_index: tuple
    peak_value: float

    @property
    def dims(self) -> int:
        return self.values.ndim


def compute_psf(k: SamplingPattern, grid_shape, weights: np.ndarray | None = None,
                hw: HardwareSpec | None = None, allow_slow: bool = False,
                precision: str = "fp64") -> PsfVolume:
    """Density-compensated adjoint response to unit measurements (analysis.py:112-137);
    with ``hw`` the pattern is first resampled to the ADC dwell grid."""
    if hw is not None:
        k = resample_to_dwell(k, hw)
    pts = k.points()
    p, dims = pts.shape
    if weights is None:
        weights = np.ones(p)
    weights = np.asarray(weights)
    if len(weights) != p:
        raise ValueError(f"weights length {len(weights)} != sample count {p}")
    _check_budget(p, grid_shape, allow_slow)
    shape = _grid(grid_shape, dims)
    vol = nudft_adjoint_device(_device.h2d(np.ascontiguousarray(pts)),
                               _complex_dev(weights, p), shape, precision)
    total = np.sum(weights)
    mag = torch.empty(vol.shape[0], dtype=torch.float64, device=vol.device)
    if np.iscomplexobj(total):
        # complex weight sum: divide on the host path of the magnitudes' definition
        vals = np.abs(_to_complex(vol, shape) / total)
    else:
        _native.call("spk_psf_magnitude", vol.data_ptr(), vol.shape[0], float(total),
                     mag.data_ptr(), _device.stream())
        vals = _device.d2h(mag).reshape(shape)
    peak = tuple(int(i) for i in np.unravel_index(int(np.argmax(vals)), vals.shape))
    return PsfVolume(values=vals, peak_index=peak, peak_value=float(vals[peak]))


@dataclass
class PsfMetrics:
    """Width, sidelobe and noise-floor metrics (analysis.py:140-153)."""

    fwhm: tuple
    psl_db: float
    pnl_db: float
    fwhm_bounded: bool

    def as_dict(self) -> dict:
        return {"fwhm_voxels": list(self.fwhm), "psl_db": self.psl_db,
                "pnl_db": self.pnl_db, "fwhm_bounded": self.fwhm_bounded}


def _sub_voxel(v_hi: float, v_lo: float, v_next: float, half: float) -> float:
    """Where the profile crosses ``half`` between two samples, in [0, 1]: the root of the
    parabola through (0, v_hi), (1, v_lo), (2, v_next) when it lies in [0, 1], the linear
    crossing otherwise (analysis.py:156-181)."""
    linear = (v_hi - half) / (v_hi - v_lo)
    curv = 0.5 * (v_next - 2.0 * v_lo + v_hi)
    slope = v_lo - v_hi - curv
    off = v_hi - half
    if abs(curv) < 1e-14 * max(abs(v_hi), 1e-300):
        return linear
    disc = slope * slope - 4.0 * curv * off
    if disc < 0:
        return linear
    root = np.sqrt(disc)
    for x in ((-slope - root) / (2 * curv), (-slope + root) / (2 * curv)):
        if 0.0 <= x <= 1.0:
            return x
    return linear


def _fwhm_1d(profile: np.ndarray, c: int) -> float:
    """Full width at half maximum around index c (analysis.py:184-203); inf when a side
    never falls below half."""
    half = profile[c] / 2.0
    n = len(profile)
    widths = []
    for step in (1, -1):
        width = np.inf
        j = c + step
        while 0 <= j < n:
            if profile[j] < half:
                beyond = j + step
                v_next = profile[beyond] if 0 <= beyond < n else profile[j]
                frac = _sub_voxel(profile[j - step], profile[j], v_next, half)
                width = abs((j - step) + step * frac - c)
                break
            j += step
        widths.append(width)
    return widths[0] + widths[1]


def _lobe(profile: np.ndarray, c: int) -> tuple[int, int]:
    """First local minimum on each side of c (analysis.py:206-215)."""
    hi = c
    while hi < len(profile) - 1 and profile[hi + 1] <= profile[hi]:
        hi += 1
    lo = c
    while lo > 0 and profile[lo - 1] <= profile[lo]:
        lo -= 1
    return lo, hi


def psf_metrics(psf: PsfVolume, noise_shell: float = 0.75) -> PsfMetrics:
    """FWHM per axis through the peak, peak-to-sidelobe level outside the main-lobe box
    and peak-to-noise level over the outer shell, in dB capped at 300
    (analysis.py:218-273)."""
    vals = psf.values
    peak = psf.peak_value
    if peak <= 0:
        raise ValueError("PSF peak must be strictly positive")
    c = psf.peak_index
    fwhm, lobes = [], []
    for ax in range(vals.ndim):
        idx = list(c)
        idx[ax] = slice(None)
        prof = vals[tuple(idx)]
        fwhm.append(float(_fwhm_1d(prof, c[ax])))
        lobes.append(_lobe(prof, c[ax]))
    bounded = all(np.isfinite(f) for f in fwhm)

    main = np.zeros(vals.shape, dtype=bool)
    main[tuple(slice(lo, hi + 1) for lo, hi in lobes)] = True
    is_max = np.ones(vals.shape, dtype=bool)
    for ax in range(vals.ndim):  # periodic neighbours, as np.roll
        is_max &= (vals >= np.roll(vals, -1, axis=ax)) & (vals >= np.roll(vals, 1, axis=ax))
    side = vals[is_max & ~main]
    psl = 20.0 * np.log10(peak / side.max()) if side.size and side.max() > 0 else DB_CAP

    r2 = np.zeros(vals.shape)
    for ax, n in enumerate(vals.shape):
        shp = [1] * vals.ndim
        shp[ax] = n
        r2 = r2 + (((np.arange(n) - c[ax]) / (n / 2.0)) ** 2).reshape(shp)
    shell = vals[np.sqrt(r2) > noise_shell]
    if shell.size and np.any(shell > 0):
        pnl = 20.0 * np.log10(peak / np.sqrt(np.mean(shell ** 2)))
    else:
        pnl = DB_CAP
    return PsfMetrics(fwhm=tuple(fwhm), psl_db=float(min(psl, DB_CAP)),
                      pnl_db=float(min(pnl, DB_CAP)), fwhm_bounded=bounded)


def _bin_index(coord: np.ndarray, bins: int) -> np.ndarray:
    return np.clip(((coord + 1.0) * 0.5 * bins).astype(np.int64), 0, bins - 1)


def bin_samples(points: np.ndarray, bins: int) -> np.ndarray:
    """Normalised sample histogram on a uniform grid over the cube (analysis.py:276-286)."""
    dims = points.shape[1]
    idx = _bin_index(points, bins)
    flat = np.ravel_multi_index(tuple(idx[:, a] for a in range(dims)), (bins,) * dims)
    hist = np.bincount(flat, minlength=bins ** dims).astype(np.float64)
    return (hist / len(points)).reshape((bins,) * dims)


def bin_density(rho: TargetDensity, bins: int) -> np.ndarray:
    """The density grid aggregated into the same bins (analysis.py:289-301)."""
    n, dims = rho.grid_n, rho.dims
    idx = _bin_index(np.arange(-n, n + 1) / n, bins)
    mesh = np.meshgrid(*([idx] * dims), indexing="ij")
    flat = np.ravel_multi_index(tuple(m.ravel() for m in mesh), (bins,) * dims)
    out = np.zeros(bins ** dims)
    np.add.at(out, flat, rho.grid.ravel())
    return out.reshape((bins,) * dims)


def density_compliance(k: SamplingPattern, rho: TargetDensity,
                       bins: int = 8) -> tuple[float, np.ndarray, np.ndarray]:
    """L1 distance between the binned samples and the binned target (analysis.py:304-321)."""
    if bins < 4:
        raise ValueError("bins must be >= 4 per axis")
    if k.dims != rho.dims:
        raise ValueError(f"pattern dims {k.dims} != density dims {rho.dims}")
    h_samples = bin_samples(k.points(), bins)
    h_rho = bin_density(rho, bins)
    return float(np.abs(h_samples - h_rho).sum()), h_samples, h_rho
