"""Analysis path on the GPU (csrc/nudft.cu) vs the reference's outputs
(tests/golden/analysis.npz) and the numpy oracle (oracle/nudft_oracle.py).

Tolerances (max abs error / max |reference|): precision="fp64" (the default) computes
like the reference's complex128 numpy, tested at 1e-12; "mixed" (fp32 products, fp64
phases and accumulation) at 2e-5.  The density-compensation fixed point amplifies
relative noise by ~1e6 (test_dcf_radial_acceptance_fixture), so it is asserted in fp64."""

import numpy as np
import pytest

from oracle import nudft_oracle as no
from spk_golden import golden

pytestmark = pytest.mark.gpu
TOL = 1e-12
TOLS = {"fp64": 1e-12, "mixed": 2e-5}


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_nudft_golden(spk, precision):
    from paper_2108_02991_b200 import analysis as an

    g = golden("analysis")
    for name in ("a2", "a3"):
        grid = tuple(int(x) for x in g[f"{name}_grid"])
        adj = an.nudft_adjoint(g[f"{name}_pts"], g[f"{name}_w"], grid, precision=precision)
        assert adj.shape == grid and adj.dtype == np.complex128
        assert rel(adj, g[f"{name}_adj"]) < TOLS[precision], name
        fwd = an.nudft_forward(g[f"{name}_pts"], g[f"{name}_img"], precision=precision)
        assert fwd.shape == (g[f"{name}_pts"].shape[0],)
        assert rel(fwd, g[f"{name}_fwd"]) < TOLS[precision], name


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
@pytest.mark.parametrize("dims,p,grid", [(2, 5000, (64, 48)), (3, 3000, (20, 17, 33)),
                                         (3, 700, (9, 64, 5)), (2, 129, (1, 7)),
                                         (3, 1, (4, 4, 4)), (2, 77, (130, 3))])
def test_nudft_random_vs_oracle(spk, dims, p, grid, precision):
    from paper_2108_02991_b200 import analysis as an

    rng = np.random.default_rng(p)
    pts = rng.uniform(-1, 1, (p, dims))
    w = rng.normal(size=p) + 1j * rng.normal(size=p)
    img = rng.normal(size=grid) + 1j * rng.normal(size=grid)
    tol = TOLS[precision]
    assert rel(an.nudft_adjoint(pts, w, grid, precision=precision),
               no.nudft_adjoint(pts, w, grid)) < tol
    assert rel(an.nudft_forward(pts, img, precision=precision), no.nudft_forward(pts, img)) < tol


def test_precision_argument(spk):
    from paper_2108_02991_b200 import analysis as an

    with pytest.raises(ValueError, match="precision"):
        an.nudft_adjoint(np.zeros((3, 2)), np.ones(3), (4, 4), precision="fp16")


def test_dcf_radial_acceptance_fixture(spk):
    """The acceptance gate's PSF leg on the 3D radial init (64 x 128 on 32^3, 10
    iterations): weights and PSF metrics vs the reference's.  The fixed point amplifies
    relative noise ~1e6-fold, so this pins fp64 accuracy end to end."""
    g = golden("analysis")
    kr = spk.init_radial(64, 128, 3)
    w = spk.density_compensation(kr, (32, 32, 32), iters=10)
    assert rel(w, g["dcfr3"]) < 1e-7
    m = spk.psf_metrics(spk.compute_psf(kr, (32, 32, 32), w))
    got = np.array(list(m.fwhm) + [m.psl_db, m.pnl_db, float(m.fwhm_bounded)])
    assert np.allclose(got, g["dcfr3_metrics"], rtol=1e-7, atol=1e-7), (got, g["dcfr3_metrics"])


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
    assert abs(lhs - rhs) / abs(lhs) < 1e-10
    lhs = np.vdot(img, an.nudft_adjoint(pts, w, grid, precision="mixed"))
    rhs = np.vdot(an.nudft_forward(pts, img, precision="mixed"), w)
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
    a1 = an.nudft_adjoint(pts, w, grid)
    a2 = an.nudft_adjoint(pts, 2.0 * w, grid)
    assert rel(a2, 2.0 * a1) < 1e-12
