"""Analysis path on the GPU (csrc/nudft.cu) vs the reference's outputs
(tests/golden/analysis.npz) and the numpy oracle (oracle/nudft_oracle.py).

Tolerance: fp32 products with fp64 phases and accumulation -> relative error ~1e-6 of
the output norm; tested at 2e-5 (max abs error / max |reference|)."""

import numpy as np
import pytest

from oracle import nudft_oracle as no
from spk_golden import golden

pytestmark = pytest.mark.gpu
TOL = 2e-5


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_nudft_golden(spk):
    from paper_2108_02991_b200 import analysis as an

    g = golden("analysis")
    for name in ("a2", "a3"):
        grid = tuple(int(x) for x in g[f"{name}_grid"])
        adj = an.nudft_adjoint(g[f"{name}_pts"], g[f"{name}_w"], grid)
        assert adj.shape == grid and adj.dtype == np.complex128
        assert rel(adj, g[f"{name}_adj"]) < TOL, name
        fwd = an.nudft_forward(g[f"{name}_pts"], g[f"{name}_img"])
        assert fwd.shape == (g[f"{name}_pts"].shape[0],)
        assert rel(fwd, g[f"{name}_fwd"]) < TOL, name


@pytest.mark.parametrize("dims,p,grid", [(2, 5000, (64, 48)), (3, 3000, (20, 17, 33)),
                                         (3, 700, (9, 64, 5)), (2, 129, (1, 7))])
def test_nudft_random_vs_oracle(spk, dims, p, grid):
    from paper_2108_02991_b200 import analysis as an

    rng = np.random.default_rng(p)
    pts = rng.uniform(-1, 1, (p, dims))
    w = rng.normal(size=p) + 1j * rng.normal(size=p)
    img = rng.normal(size=grid) + 1j * rng.normal(size=grid)
    assert rel(an.nudft_adjoint(pts, w, grid), no.nudft_adjoint(pts, w, grid)) < TOL
    assert rel(an.nudft_forward(pts, img), no.nudft_forward(pts, img)) < TOL


def test_density_compensation_golden(spk):
    g = golden("analysis")
    w2 = spk.density_compensation(spk.SamplingPattern(g["dcf2_coords"]), (16, 16), iters=3)
    assert rel(w2, g["dcf2"]) < TOL
    w3 = spk.density_compensation(spk.SamplingPattern(g["dcf3_coords"]), (8, 8, 8), iters=2)
    assert rel(w3, g["dcf3"]) < TOL


def test_compute_psf_golden(spk):
    g = golden("analysis")
    k2 = spk.SamplingPattern(g["dcf2_coords"])
    psf = spk.compute_psf(k2, (32, 32), weights=g["dcf2"])
    assert rel(psf.values, g["psf2"]) < TOL
    assert psf.peak_index == tuple(int(i) for i in g["psf2_peak"])
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=2e-6, fov=0.192, matrix=32, dims=2)
    assert rel(spk.compute_psf(k2, (24, 24), hw=hw).values, g["psf2h"]) < TOL
    k3 = spk.SamplingPattern(g["dcf3_coords"])
    psf3 = spk.compute_psf(k3, (12, 12, 12))
    assert rel(psf3.values, g["psf3"]) < TOL
    m = spk.psf_metrics(psf3)
    ref = g["psf3_metrics"]
    assert np.allclose(list(m.fwhm) + [m.psl_db, m.pnl_db], ref[:-1], rtol=1e-4)
    with pytest.raises(ValueError, match="weights length"):
        spk.compute_psf(k3, (8, 8, 8), weights=np.ones(3))


def test_linearity_and_adjointness(spk):
    """<adjoint(w), img> == <w, forward(img)> (size-independent property)."""
    from paper_2108_02991_b200 import analysis as an

    rng = np.random.default_rng(8)
    pts = rng.uniform(-1, 1, (20000, 3))
    grid = (32, 32, 24)
    w = rng.normal(size=20000) + 1j * rng.normal(size=20000)
    img = rng.normal(size=grid) + 1j * rng.normal(size=grid)
    lhs = np.vdot(img, an.nudft_adjoint(pts, w, grid))
    rhs = np.vdot(an.nudft_forward(pts, img), w)
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
    a1 = an.nudft_adjoint(pts, w, grid)
    a2 = an.nudft_adjoint(pts, 2.0 * w, grid)
    assert rel(a2, 2.0 * a1) < 1e-12
