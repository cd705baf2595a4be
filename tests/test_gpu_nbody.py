"""K1 / K2 N-body kernels vs the oracle and the reference's golden vectors (GPU).

Tolerance (north star): relative L2 error of the gradient <= 1e-4; the fp32 pair math with
fp64 tile accumulation lands near 1e-6.  Exact-zero cases (coincident points, eps = 0)
hold exactly."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from spk_golden import golden

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-4
VAL_TOL = 1e-5


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


@pytest.fixture(scope="module")
def rep():
    return golden("repulsion")


def raw_direct(spk, tgt, src, eps2):
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.repulsion import direct_sums_device

    t4 = _device.pack_positions(_device.h2d(tgt))
    s4 = _device.pack_positions(_device.h2d(src))
    val, grad = direct_sums_device(t4, s4, tgt.shape[1], eps2)
    return _device.d2h(val), _device.d2h(grad)


def test_golden_direct_sums(spk, rep):
    for name in rep["names"]:
        pos = rep[f"{name}_pos"]
        eps2 = float(rep[f"{name}_eps2"])
        val, grad = raw_direct(spk, pos, pos, eps2)
        assert rel_l2(val, rep[f"{name}_val"]) <= VAL_TOL, name
        gref = rep[f"{name}_grad"]
        if np.linalg.norm(gref) > 0:
            assert rel_l2(grad, gref) <= GRAD_TOL, name
        else:
            assert np.all(grad == 0.0), name


def test_public_api_matches_golden(spk, rep):
    for name in rep["names"]:
        eps = float(np.sqrt(rep[f"{name}_eps2"]))
        cost, grad = spk.eval_repulsion_direct(rep[f"{name}_pos"], eps)
        assert isinstance(cost, float) and grad.dtype == np.float64
        assert abs(cost - float(rep[f"{name}_cost"])) <= VAL_TOL * abs(float(rep[f"{name}_cost"]))
        gref = rep[f"{name}_gnorm"]
        if np.linalg.norm(gref) > 0:
            assert rel_l2(grad, gref) <= GRAD_TOL, name


def test_two_particles_and_self_term(spk):
    # reference tests/test_repulsion.py:23-36
    cost, grad = spk.eval_repulsion_direct(np.array([[0.0, 0, 0], [1.0, 0, 0]]), eps=0.0)
    assert abs(cost - 0.25) < 1e-7
    assert np.abs(grad - np.array([[-0.25, 0, 0], [0.25, 0, 0]])).max() < 1e-7
    cost, grad = spk.eval_repulsion_direct(np.zeros((3, 2)), eps=0.1)
    assert cost == pytest.approx(0.1 / 2.0, rel=1e-6)
    assert np.all(grad == 0.0)


def test_subset_targets(spk, rep):
    pos = rep["spokes3d_pos"]
    tg = rep["subset_targets"]
    val, grad = raw_direct(spk, pos[tg], pos, 1e-6)
    assert rel_l2(val, rep["subset_val"]) <= VAL_TOL
    assert rel_l2(grad, rep["subset_grad"]) <= GRAD_TOL


@pytest.mark.parametrize("d,p", [(2, 32768), (3, 20000), (3, 4099), (2, 1)])
def test_vs_oracle_random(spk, d, p):
    rng = np.random.default_rng(p + d)
    pts = rng.uniform(-1, 1, (p, d))
    val, grad = raw_direct(spk, pts, pts, 1e-6)
    vref, gref = orc.direct_sums(pts, 1e-6)
    assert rel_l2(val, vref) <= VAL_TOL
    if p > 1:
        assert rel_l2(grad, gref) <= GRAD_TOL


def test_c2_scale_row_subset(spk):
    """Config C2 (3D 1024 x 1024, p = 2^20): all targets on the GPU, strided 2048-row
    subset of the fp64 oracle (direct_sums_subset, _treecode.py:474)."""
    from paper_2108_02991_b200 import optimizer as om

    pts = om.perturb(om.init_radial(1024, 1024, 3), 0.25, 0).points().copy()
    val, grad = raw_direct(spk, pts, pts, 1e-6)
    rows = np.arange(0, pts.shape[0], pts.shape[0] // 2048, dtype=np.int64)
    vref, gref = orc.direct_sums_subset(pts, rows, 1e-6)
    assert rel_l2(val[rows], vref) <= VAL_TOL
    assert rel_l2(grad[rows], gref) <= GRAD_TOL
    # size-independent property: forces sum to ~0 (antisymmetry)
    assert np.linalg.norm(grad.sum(0)) <= 1e-6 * np.abs(grad).sum()


def test_deterministic(spk):
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (50000, 3))
    a = raw_direct(spk, pts, pts, 1e-6)
    b = raw_direct(spk, pts, pts, 1e-6)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_exact_attraction_vs_oracle(spk):
    rng = np.random.default_rng(11)
    for d, n in ((2, 32), (3, 10)):
        rho = spk.discretize(spk.DensityParams(0.25, 2.0), n, d)
        fld = spk.precompute_field(rho)
        pts = rng.uniform(-1, 1, (3000, d))
        res = spk.eval_attraction(spk.SamplingPattern(pts[None]), fld, "exact")
        cref, gref = orc.attraction_exact(pts, rho.grid, fld.kernel_eps)
        assert abs(res.cost - cref) <= VAL_TOL * abs(cref)
        assert rel_l2(res.grad, gref) <= GRAD_TOL


def test_field_grids_match_reference_precompute(spk):
    att = golden("attraction")
    for name in att["names"]:
        rho = spk.TargetDensity(att[f"{name}_rho"], int(att[f"{name}_n"]))
        fld = spk.precompute_field(rho, kernel_eps=float(att[f"{name}_eps"]))
        pot = att[f"{name}_potential"]
        # same fp64 FFT convolution as the reference (cuFFT vs pocketfft round-off)
        assert np.abs(fld.potential - pot).max() <= 1e-13 * np.abs(pot).max(), name
        force = att[f"{name}_force"]
        assert np.abs(fld.force - force).max() <= 1e-12 * np.abs(force).max(), name


def test_fused_equals_separate(spk):
    """spk_fused_sums (one launch, two segments) == two separate launches."""
    from paper_2108_02991_b200 import _device, _native
    from paper_2108_02991_b200.attraction import grid_sums_device
    from paper_2108_02991_b200.repulsion import direct_sums_device

    rng = np.random.default_rng(5)
    rho = spk.discretize(spk.DensityParams(0.25, 2.0), 12, 3)
    fld = spk.precompute_field(rho)
    pts = rng.uniform(-1, 1, (7000, 3))
    p4 = _device.pack_positions(_device.h2d(pts))
    w = fld.device_sources()
    va, ga = grid_sums_device(p4, fld, fld.kernel_eps ** 2)
    vr, gr = direct_sums_device(p4, p4, 3, 1e-6)
    bufs = [torch.empty_like(t) for t in (va, ga, vr, gr)]
    nb = _native.query("spk_nbody_workspace_bytes", 7000, 25 ** 3, 7000)
    ws = _device.workspace(nb, "nbody")
    _native.call("spk_fused_sums", p4.data_ptr(), 7000, 3, w.data_ptr(),
                 _native.i64_array(fld.sides), float(fld.kernel_eps ** 2), p4.data_ptr(), 7000,
                 1e-6,
                 *[b.data_ptr() for b in bufs], ws.data_ptr(), ws.numel(), _device.stream())
    for x, y in zip(bufs, (va, ga, vr, gr)):
        assert rel_l2(_device.d2h(x), _device.d2h(y)) <= 1e-6


def test_exact_attraction_anisotropic_grid(spk):
    """Non-cubic density grid (full3d's 384 x 384 x 208 matrix shape, scaled down):
    K2 vs the oracle's anisotropic weighted sum."""
    rng = np.random.default_rng(12)
    rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (12, 12, 7), 3)
    fld = spk.precompute_field(rho)
    pts = rng.uniform(-1, 1, (2500, 3))
    res = spk.eval_attraction(spk.SamplingPattern(pts[None]), fld, "exact")
    cref, gref = orc.attraction_exact(pts, rho.grid, fld.kernel_eps)
    assert abs(res.cost - cref) <= VAL_TOL * abs(cref)
    assert rel_l2(res.grad, gref) <= GRAD_TOL
    with pytest.raises(ValueError, match="cubic"):
        spk.eval_attraction(spk.SamplingPattern(pts[None]), fld, "consistent")


def _subset_sums(spk, pts, rows, fld):
    """GPU K1 (rows vs all positions) and K2 (rows vs the lattice) for a row subset."""
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.attraction import grid_sums_device
    from paper_2108_02991_b200.repulsion import direct_sums_device

    t4 = _device.pack_positions(_device.h2d(pts[rows]))
    s4 = _device.pack_positions(_device.h2d(pts))
    vr, gr = direct_sums_device(t4, s4, pts.shape[1], 1e-6)
    va, ga = grid_sums_device(t4, fld, fld.kernel_eps ** 2)
    return [_device.d2h(x) for x in (vr, gr, va, ga)]


def test_c2_scale_attraction_row_subset(spk):
    """C2 (p = 2^20, 129^3 lattice): K2 on a 1024-row strided subset vs the fp64 oracle."""
    from paper_2108_02991_b200 import optimizer as om

    pts = om.perturb(om.init_radial(1024, 1024, 3), 0.25, 0).points().copy()
    rho = spk.discretize(spk.DensityParams(0.25, 2.0), 64, 3)
    fld = spk.precompute_field(rho)
    rows = np.arange(0, pts.shape[0], pts.shape[0] // 1024, dtype=np.int64)
    _, _, va, ga = _subset_sums(spk, pts, rows, fld)
    vref, gref = orc.grid_sums(pts[rows], rho.grid, fld.kernel_eps ** 2)
    assert rel_l2(va, vref) <= VAL_TOL
    assert rel_l2(ga, gref) <= GRAD_TOL


def test_c4_scale_row_subset(spk):
    """C4 (4096 x 2048 = 8.4M samples, 385 x 385 x 209 lattice): K1 and K2 on a 512-row
    strided subset of targets against all sources, vs the fp64 oracle."""
    from paper_2108_02991_b200 import optimizer as om

    pts = om.perturb(om.init_radial(4096, 2048, 3), 0.75, 0).points().copy()
    rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
    fld = spk.precompute_field(rho)
    rows = np.arange(0, pts.shape[0], pts.shape[0] // 512, dtype=np.int64)
    vr, gr, va, ga = _subset_sums(spk, pts, rows, fld)
    vref, gref = orc.direct_sums_subset(pts, rows, 1e-6)
    assert rel_l2(vr, vref) <= VAL_TOL
    assert rel_l2(gr, gref) <= GRAD_TOL
    aref, agref = orc.grid_sums(pts[rows], rho.grid, fld.kernel_eps ** 2)
    assert rel_l2(va, aref) <= VAL_TOL
    assert rel_l2(ga, agref) <= GRAD_TOL


def test_subnormal_eps_squared_stays_finite(spk):
    """eps below 1.1e-19 has a subnormal fp32 square, which the rsqrt.approx.ftz flushes:
    the guard must drop those coincident pairs (as for eps = 0) instead of producing
    inf / NaN (found by scripts/nbody_extreme.py)."""
    rng = np.random.default_rng(4)
    for d in (2, 3):
        pts = rng.uniform(-1, 1, (500, d))
        cost, grad = spk.eval_repulsion_direct(pts, eps=1e-20)
        assert np.isfinite(cost) and np.all(np.isfinite(grad))
        cref, gref = orc.repulsion(pts, 1e-20)
        assert abs(cost - cref) <= VAL_TOL * abs(cref)
        assert rel_l2(grad, gref) <= GRAD_TOL
        c1, g1 = spk.eval_repulsion_direct(pts[:1], eps=1e-20)
        assert np.isfinite(c1) and abs(c1) <= 1e-19 and np.all(g1 == 0.0)

