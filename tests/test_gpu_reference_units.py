"""The reference's unit-test properties (pkg/tests/test_repulsion.py, test_projection.py,
test_attraction.py, test_analysis.py), asserted through this package's public API on
the GPU.  Tolerances are the reference's except where this build's arithmetic differs
by design, each stated at the check:

* repulsion pair sums are fp32 with fp64 accumulation (north star: gradient rel l2
  <= 1e-4), so the reference's machine-precision invariances (1e-10 .. 1e-12) are
  asserted at 1e-6;
* the reference's small clouds (2000-4000 points) fall under the exact-kernel threshold
  here (2^17 sources, as the reference itself goes direct below ``leaf_size``), so the
  treecode properties are checked on clouds of 2^18 points, where the tree runs;
* the QP oracle is scipy's SLSQP instead of cvxpy (absent in this image).
"""

import numpy as np
import pytest

from qp_ref import qp_reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


def _radial_cloud(rng, p, d):
    r = rng.uniform(0, 1, p) ** 2
    v = rng.normal(size=(p, d))
    return np.ascontiguousarray(r[:, None] * v / np.linalg.norm(v, axis=1, keepdims=True))


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


# ------------------------------------------------------------------ repulsion (test_repulsion.py)
class TestRepulsion:
    def test_self_term_only(self, spk):
        """All pairs coincident: every kernel value is eps, gradients exactly 0."""
        cost, grad = spk.eval_repulsion_direct(np.zeros((3, 2)), eps=0.1)
        assert cost == pytest.approx(0.05, rel=1e-6)  # fp32 sqrt(eps^2)
        assert np.all(grad == 0.0)

    def test_rigid_motions(self, spk, rng):
        """Translation (2D/3D) and rotation (3D) invariance, at fp32 pair precision."""
        pts = rng.uniform(-0.5, 0.5, (64, 3))
        c0, g0 = spk.eval_repulsion_direct(pts, 1e-3)
        c1, g1 = spk.eval_repulsion_direct(pts + np.array([0.3, -0.2, 0.1]), 1e-3)
        assert abs(c1 - c0) <= 1e-6 * abs(c0)
        assert np.abs(g1 - g0).max() <= 1e-6 * np.abs(g0).max()
        th = 0.7
        rot = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
        c2, g2 = spk.eval_repulsion_direct(pts @ rot.T, 1e-3)
        assert abs(c2 - c0) <= 1e-6 * abs(c0)
        assert np.abs(g2 - g0 @ rot.T).max() <= 1e-6 * np.abs(g0).max()

    def test_forces_sum_to_zero(self, spk, rng):
        _, grad = spk.eval_repulsion_direct(rng.uniform(-1, 1, (200, 2)), 1e-3)
        assert np.linalg.norm(grad.sum(axis=0)) <= 1e-6 * np.abs(grad).sum()

    def test_tree_meets_default_precision(self, spk, rng):
        for d in (2, 3):
            pts = _radial_cloud(rng, 1 << 18, d)
            cfg = spk.RepulsionConfig(backend="tree", kernel_eps=1e-3)
            c0, g0 = spk.eval_repulsion_direct(pts, 1e-3)  # fp32 pairs: ~1e-6 << 1e-4
            c1, g1 = spk.eval_repulsion_tree(pts, cfg)
            assert abs(c1 - c0) / abs(c0) <= cfg.tree_precision
            assert _rel(g1, g0) <= cfg.tree_precision

    def test_tiny_pattern_is_the_direct_result(self, spk, rng):
        pts = rng.uniform(-1, 1, (2, 3))
        cfg = spk.RepulsionConfig(backend="tree")
        c_t, g_t = spk.eval_repulsion_tree(pts, cfg)
        c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
        assert c_t == c_d and np.array_equal(g_t, g_d)

    def test_error_falls_with_interpolation_order(self, spk, rng):
        from paper_2108_02991_b200 import _device
        from paper_2108_02991_b200.repulsion import direct_sums_device
        from paper_2108_02991_b200.tree import tree_sums_device

        pts = _radial_cloud(rng, 1 << 18, 2)
        p4 = _device.pack_positions(_device.h2d(pts))
        _, g_ref = direct_sums_device(p4, p4, 2, 1e-6)
        g_ref = _device.d2h(g_ref)
        errs = []
        for order in range(2, 7):
            _, g = tree_sums_device(p4, p4, 2, 1e-6, order, 0.55)
            errs.append(_rel(_device.d2h(g), g_ref))
        assert all(lo <= hi * 1.05 for lo, hi in zip(errs[1:], errs[:-1])), errs

    def test_dispatcher(self, spk, rng):
        pts = rng.uniform(-1, 1, (300, 2))
        c1, _ = spk.eval_repulsion(pts, spk.RepulsionConfig(backend="direct"))
        c2, _ = spk.eval_repulsion(pts, spk.RepulsionConfig(backend="tree"))
        assert c2 == pytest.approx(c1, rel=1e-4)

    def test_degenerate_distributions(self, spk, rng):
        """Coincident points (octree depth cap), a near-degenerate needle and two point
        masses, all large enough to run the treecode."""
        cfg = spk.RepulsionConfig(backend="tree")
        n = 200_000
        pts = np.tile(np.array([[0.3, -0.2, 0.1]]), (n, 1))
        c_t, g_t = spk.eval_repulsion_tree(pts, cfg)
        assert c_t == pytest.approx(cfg.kernel_eps / 2, rel=1e-5)  # every pair is eps
        assert np.abs(g_t).max() == 0.0
        t = rng.uniform(-1, 1, n)
        needle = np.stack([t, 1e-6 * rng.normal(size=n), np.zeros(n)], axis=1)
        two = np.concatenate([np.tile([[0.5, 0.5, 0.5]], (n // 2, 1)),
                              np.tile([[-0.5, 0.1, 0.0]], (n // 2, 1))])
        for cloud in (needle, two):
            c_t, g_t = spk.eval_repulsion_tree(cloud, cfg)
            c_d, g_d = spk.eval_repulsion_direct(cloud, cfg.kernel_eps)
            assert abs(c_t - c_d) / abs(c_d) <= cfg.tree_precision
            assert _rel(g_t, g_d) <= cfg.tree_precision

    def test_tree_translation_invariance(self, spk, rng):
        """The tree geometry moves with the cloud: invariance to the precision."""
        pts = rng.uniform(-0.4, 0.4, (1 << 18, 2))
        cfg = spk.RepulsionConfig(backend="tree")
        c1, _ = spk.eval_repulsion_tree(pts, cfg)
        c2, _ = spk.eval_repulsion_tree(pts + 0.25, cfg)
        assert abs(c1 - c2) <= 2 * cfg.tree_precision * abs(c1)

    def test_config_validation(self, spk):
        for kw in (dict(backend="gpu"), dict(tree_precision=0.0), dict(leaf_size=4),
                   dict(interp_order=1), dict(kernel_eps=-1.0)):
            with pytest.raises(ValueError):
                spk.RepulsionConfig(**kw)


# ---------------------------------------------------------------- projection (test_projection.py)
def _desk(spk, **kw):
    return spk.ProjectionConfig(alpha=10216.0, beta=4.6e7, raster_dt=1e-5, **kw)


class TestProjection:
    def test_feasible_input_unchanged(self, spk):
        cfg = spk.ProjectionConfig(alpha=0.5, beta=0.3, raster_dt=1.0, n_pit=50)
        t = np.linspace(-0.1, 0.1, 16)
        shot = np.stack([t, t ** 2], axis=1)
        assert np.abs(spk.project_shot(shot, cfg) - shot).max() <= cfg.feas_tol

    def test_box_only_clamp(self, spk):
        cfg = spk.ProjectionConfig(alpha=1e9, beta=1e12, raster_dt=1.0, n_pit=200)
        assert np.abs(spk.project_shot(np.full((12, 2), 1.5), cfg) - 1.0).max() <= 1e-6

    def test_pinned_sample_is_exact(self, spk, rng):
        pin = spk.LinearConstraint(pinned_index=4, pinned_value=np.array([0.1, -0.2]))
        cfg = spk.ProjectionConfig(alpha=0.4, beta=0.2, raster_dt=1.0, n_pit=200, pin=pin)
        out = spk.project_shot(rng.uniform(-1, 1, (9, 2)), cfg)
        assert np.array_equal(out[4], pin.pinned_value)

    def test_pinned_qp(self, spk, rng):
        """With a pin the projection still solves the QP (SLSQP with the pin as an
        equality), reference tolerance 1e-4."""
        from scipy.optimize import minimize

        a, b = 0.4, 0.2
        pin = spk.LinearConstraint(pinned_index=3, pinned_value=np.zeros(2))
        cfg = spk.ProjectionConfig(alpha=a, beta=b, raster_dt=1.0, n_pit=1500, pin=pin)
        shot = rng.uniform(-1.2, 1.2, (8, 2))
        out = spk.project_shot(shot, cfg)

        def cons(x):
            s = x.reshape(8, 2)
            d1, d2 = s[1:] - s[:-1], s[2:] - 2 * s[1:-1] + s[:-2]
            return np.concatenate([a * a - (d1 * d1).sum(1), b * b - (d2 * d2).sum(1)])

        res = minimize(lambda x: np.sum((x - shot.ravel()) ** 2), np.clip(shot, -1, 1).ravel(),
                       jac=lambda x: 2 * (x - shot.ravel()), method="SLSQP",
                       bounds=[(-1.0, 1.0)] * 16, options={"ftol": 1e-15, "maxiter": 1000},
                       constraints=[{"type": "ineq", "fun": cons},
                                    {"type": "eq", "fun": lambda x: x.reshape(8, 2)[3]}])
        assert cons(res.x).min() >= -1e-9
        assert np.abs(out - res.x.reshape(8, 2)).max() <= 1e-4

    def test_qp_unpinned(self, spk, rng):
        a, b = 0.3, 0.15
        cfg = spk.ProjectionConfig(alpha=a, beta=b, raster_dt=1.0, n_pit=1000)
        for _ in range(5):
            shot = rng.uniform(-1.5, 1.5, (8, 2))
            assert np.abs(spk.project_shot(shot, cfg) - qp_reference(shot, a, b)).max() <= 1e-4

    def test_pin_outside_omega_rejected(self, spk):
        with pytest.raises(ValueError, match="Omega"):
            spk.LinearConstraint(pinned_index=0, pinned_value=np.array([1.5, 0.0]))

    def test_monotone_dual_objective_never_increases(self, spk, rng):
        cfg = spk.ProjectionConfig(alpha=0.3, beta=0.15, raster_dt=1.0, n_pit=150, monotone=True)
        _, trace = spk.project_shot(rng.uniform(-1.4, 1.4, (32, 2)), cfg, return_trace=True)
        assert np.all(np.diff(trace) <= 1e-12)

    def test_pattern_of_one_shot_equals_project_shot(self, spk, rng):
        cfg = _desk(spk, n_pit=80)
        shot = rng.uniform(-1.1, 1.1, (32, 2))
        out = spk.project_pattern(spk.SamplingPattern(shot[None]), cfg)
        assert np.array_equal(out.coords[0], spk.project_shot(shot, cfg))

    def test_shots_are_independent_under_permutation(self, spk, rng):
        cfg = _desk(spk, n_pit=60)
        coords = rng.uniform(-1.1, 1.1, (6, 24, 2))
        out = spk.project_pattern(spk.SamplingPattern(coords), cfg)
        perm = rng.permutation(6)
        assert np.array_equal(spk.project_pattern(spk.SamplingPattern(coords[perm]), cfg).coords,
                              out.coords[perm])

    def test_gradient_step_returns_to_feasibility(self, spk, rng):
        pin = spk.LinearConstraint(pinned_index=64, pinned_value=np.zeros(2))
        base = np.cumsum(rng.normal(0, 0.004, (4, 128, 2)), axis=1)
        base -= base[:, 64:65, :]
        feasible = spk.project_pattern(spk.SamplingPattern(base), _desk(spk, n_pit=800, pin=pin))
        stepped = spk.SamplingPattern(feasible.coords
                                      + rng.uniform(-0.02, 0.02, feasible.coords.shape))
        cfg = _desk(spk, n_pit=100, pin=pin)
        assert spk.feasibility_residuals(spk.project_pattern(stepped, cfg), cfg)["max"] \
            <= cfg.feas_tol

    def test_idempotent_and_non_expansive(self, spk, rng):
        cfg = _desk(spk, n_pit=100)
        once = spk.project_pattern(spk.SamplingPattern(rng.uniform(-1.2, 1.2, (3, 16, 2))), cfg)
        twice = spk.project_pattern(once, cfg)
        assert np.linalg.norm(twice.coords - once.coords) <= cfg.feas_tol * np.sqrt(32)
        cfg = _desk(spk, n_pit=300)
        a = rng.uniform(-1.2, 1.2, (2, 16, 2))
        b = rng.uniform(-1.2, 1.2, (2, 16, 2))
        pa = spk.project_pattern(spk.SamplingPattern(a), cfg).coords
        pb = spk.project_pattern(spk.SamplingPattern(b), cfg).coords
        assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) + 2 * cfg.feas_tol

    def test_config_validation(self, spk):
        for kw in (dict(alpha=1.0, beta=1.0, raster_dt=1.0, n_pit=0),
                   dict(alpha=-1.0, beta=1.0, raster_dt=1.0),
                   dict(alpha=1.0, beta=1.0, raster_dt=0.0)):
            with pytest.raises(ValueError):
                spk.ProjectionConfig(**kw)


# ---------------------------------------------------------------- attraction (test_attraction.py)
def _point_mass(spk, n, d):
    g = np.zeros((2 * n + 1,) * d)
    g[(n,) * d] = 1.0
    return spk.TargetDensity(grid=g, grid_n=n)


class TestAttractionField:
    """precompute_field runs the reference's fp64 FFT convolution on the device (cuFFT)."""

    def test_point_mass_gives_the_kernel(self, spk):
        eps, n = 0.05, 8
        fld = spk.precompute_field(_point_mass(spk, n, 2), kernel_eps=eps)
        ax = np.arange(-n, n + 1) / n
        h = np.sqrt(ax[:, None] ** 2 + ax[None, :] ** 2 + eps ** 2)
        assert np.abs(fld.potential - h).max() <= 1e-12 * h.max()

    def test_force_is_odd(self, spk):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 12, 2),
                                   kernel_eps=0.02)
        fx = fld.force[0]
        assert np.abs(fx + fx[::-1, :]).max() <= 1e-12

    def test_brute_force_convolution(self, spk, rng):
        n, eps = 8, 0.1
        rho = spk.TargetDensity(grid=rng.uniform(0, 1, (2 * n + 1, 2 * n + 1)), grid_n=n)
        fld = spk.precompute_field(rho, kernel_eps=eps)
        ax = np.arange(-n, n + 1) / n
        x = np.stack(np.meshgrid(ax, ax, indexing="ij"), -1).reshape(-1, 2)
        h = np.sqrt(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1) + eps ** 2)
        ref = (h @ rho.grid.reshape(-1)).reshape(2 * n + 1, 2 * n + 1)
        assert np.abs(fld.potential - ref).max() / np.abs(ref).max() <= 1e-10

    def test_linear_in_the_density(self, spk, rng):
        g1 = spk.TargetDensity(rng.uniform(0, 1, (17, 17)), 8).grid
        g2 = spk.TargetDensity(rng.uniform(0, 1, (17, 17)), 8).grid
        f1 = spk.precompute_field(spk.TargetDensity(g1, 8), kernel_eps=0.05).potential
        f2 = spk.precompute_field(spk.TargetDensity(g2, 8), kernel_eps=0.05).potential
        mix = 0.25 * f1 + 0.75 * f2
        fm = spk.precompute_field(spk.TargetDensity(0.25 * g1 + 0.75 * g2, 8),
                                  kernel_eps=0.05).potential
        assert np.abs(fm - mix).max() <= 1e-12 * np.abs(mix).max()

    def test_defaults_and_memory_guidance(self, spk):
        from paper_2108_02991_b200.attraction import field_workspace_bytes

        assert spk.precompute_field(_point_mass(spk, 10, 2)).kernel_eps == pytest.approx(0.05)
        with pytest.raises(MemoryError, match="grid"):
            spk.precompute_field(_point_mass(spk, 4, 3), kernel_eps=0.1, mem_cap_bytes=1024)
        assert field_workspace_bytes(768, 3) > 1e10

    def test_interpolation_exact_at_nodes(self, spk):
        from paper_2108_02991_b200.attraction import interpolate

        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 8, 2),
                                   kernel_eps=0.05)
        nodes = np.array([[i / 8, j / 8] for i in (-8, -3, 0, 5) for j in (-8, 2, 8)])
        idx = np.round((nodes + 1) * 8).astype(int)
        assert np.array_equal(interpolate(fld.potential, nodes, 8),
                              fld.potential[idx[:, 0], idx[:, 1]])

    def test_origin_gradient_vanishes(self, spk):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 16, 2),
                                   kernel_eps=0.05)
        for mode in ("consistent", "smooth"):
            res = spk.eval_attraction(spk.SamplingPattern(np.zeros((1, 1, 2))), fld, mode)
            assert np.abs(res.grad).max() <= 1e-10

    def test_gradient_is_the_cost_derivative(self, spk, rng):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 32, 2),
                                   kernel_eps=1e-3)
        u = (rng.uniform(-0.9, 0.9, (40, 2)) + 1.0) * 32
        frac = u - np.floor(u)
        u = u + np.where(frac < 0.2, 0.2 - frac, 0.0) - np.where(frac > 0.8, frac - 0.8, 0.0)
        pts = u / 32 - 1.0
        grad = spk.eval_attraction(spk.SamplingPattern(pts[None]), fld, "consistent").grad
        h = 1e-6
        fd = np.zeros_like(grad)
        for i in range(40):
            for ax in range(2):
                q1, q2 = pts.copy(), pts.copy()
                q1[i, ax] += h
                q2[i, ax] -= h
                fd[i, ax] = (spk.eval_attraction(spk.SamplingPattern(q1[None]), fld).cost
                             - spk.eval_attraction(spk.SamplingPattern(q2[None]), fld).cost) / (2 * h)
        assert np.abs(grad - fd).max() / np.abs(fd).max() <= 1e-5

    def test_order_of_samples_is_irrelevant(self, spk, rng):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 16, 3))
        pts = rng.uniform(-1, 1, (50, 3))
        perm = rng.permutation(50)
        r1 = spk.eval_attraction(spk.SamplingPattern(pts[None]), fld)
        r2 = spk.eval_attraction(spk.SamplingPattern(pts[perm][None]), fld)
        assert r1.cost == pytest.approx(r2.cost, rel=1e-14)
        assert np.allclose(r1.grad[perm], r2.grad, atol=1e-15)

    def test_out_of_domain_clamped_and_counted(self, spk):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 8, 2))
        res = spk.eval_attraction(
            spk.SamplingPattern(np.array([[[1.5, 0.0], [0.0, 0.0], [-1.0, -2.0]]])), fld)
        assert res.n_clamped == 2 and np.isfinite(res.cost)

    def test_dims_must_match(self, spk):
        fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), 8, 2))
        with pytest.raises(ValueError, match="dims"):
            spk.eval_attraction(spk.SamplingPattern(np.zeros((1, 2, 3))), fld)


# ---------------------------------------------------------------- analysis (test_analysis.py)
def _cartesian(spk, n, d):
    axes = [(2.0 / n) * (np.arange(n) - n // 2)] * d
    pts = np.stack([m.ravel() for m in np.meshgrid(*axes, indexing="ij")], axis=1)
    return spk.SamplingPattern(pts.reshape(1, -1, d))


class TestAnalysis:
    def test_full_cartesian_sampling_has_flat_weights(self, spk):
        w = spk.density_compensation(_cartesian(spk, 8, 2), (8, 8), iters=10)
        assert w.std() / w.mean() <= 1e-6 and np.all(w > 0)

    def test_radial_weights_grow_with_radius(self, spk):
        pat = spk.init_radial(48, 33, 2)
        w = spk.density_compensation(pat, (16, 16), iters=10)
        r = np.linalg.norm(pat.points(), axis=1)
        keep = r < 0.9
        edges = np.linspace(0, 0.9, 7)
        means = [w[keep][(r[keep] >= lo) & (r[keep] < hi)].mean()
                 for lo, hi in zip(edges, edges[1:])]
        assert np.all(np.diff(means) > 0)

    def test_empty_pattern_and_defaults(self, spk):
        import inspect

        pat = spk.SamplingPattern(np.zeros((1, 1, 2)))
        pat.coords = pat.coords[:, :0, :]
        with pytest.raises(ValueError, match="empty"):
            spk.density_compensation(pat, (8, 8))
        assert inspect.signature(spk.density_compensation).parameters["iters"].default == 10

    def test_psf_special_patterns(self, spk):
        psf = spk.compute_psf(spk.SamplingPattern(np.zeros((1, 1, 2))), (16, 16))
        assert psf.values.max() / psf.values.mean() == pytest.approx(1.0, rel=1e-12)
        psf = spk.compute_psf(_cartesian(spk, 16, 2), (16, 16))
        assert psf.peak_index == (8, 8)
        off = psf.values.copy()
        off[8, 8] = 0.0
        assert off.max() <= 1e-10 * psf.peak_value

    def test_adjoint_linear_and_hermitian_symmetric(self, spk, rng):
        from paper_2108_02991_b200.analysis import nudft_adjoint

        pts = rng.uniform(-1, 1, (40, 2))
        w1, w2 = rng.uniform(0.5, 1.5, 40), rng.uniform(0.5, 1.5, 40)
        g12 = nudft_adjoint(pts, w1 + 2 * w2, (12, 12))
        g = nudft_adjoint(pts, w1, (12, 12)) + 2 * nudft_adjoint(pts, w2, (12, 12))
        assert np.abs(g12 - g).max() <= 1e-10 * np.abs(g12).max()
        half = rng.uniform(-1, 1, (30, 2))
        grid = nudft_adjoint(np.concatenate([half, -half]), np.ones(60), (16, 16))
        assert np.abs(grid.imag).max() <= 1e-10 * np.abs(grid.real).max()

    def test_psf_arguments(self, spk, rng):
        with pytest.raises(ValueError, match="length"):
            spk.compute_psf(spk.SamplingPattern(np.zeros((1, 4, 2))), (8, 8), weights=np.ones(3))
        hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.57e6, raster_dt=1e-5,
                              dwell_dt=5e-6, fov=0.2, matrix=16, dims=2)
        pat = spk.SamplingPattern(rng.uniform(-1, 1, (2, 16, 2)))
        assert np.array_equal(spk.compute_psf(pat, (16, 16), hw=hw).values,
                              spk.compute_psf(spk.resample_to_dwell(pat, hw), (16, 16)).values)
        with pytest.raises(ValueError, match="allow_slow"):
            spk.compute_psf(spk.SamplingPattern(np.zeros((1, 100000, 3))), (64, 64, 64))

    def test_psf_metrics_properties(self, spk, rng):
        vals = np.zeros((16, 16, 16))
        vals[8, 8, 8] = 1.0
        m = spk.psf_metrics(spk.PsfVolume(values=vals, peak_index=(8, 8, 8), peak_value=1.0))
        assert all(f <= 1.0 for f in m.fwhm) and m.psl_db == 300.0 and m.pnl_db == 300.0
        vals = rng.uniform(0.01, 0.2, (21, 21))
        vals[10, 10] = 1.0
        m1 = spk.psf_metrics(spk.PsfVolume(vals, (10, 10), 1.0))
        m2 = spk.psf_metrics(spk.PsfVolume(7.5 * vals, (10, 10), 7.5))
        assert m1.fwhm == m2.fwhm
        assert m1.psl_db == pytest.approx(m2.psl_db, rel=1e-12)
        assert m1.pnl_db == pytest.approx(m2.pnl_db, rel=1e-12)
        assert not spk.psf_metrics(spk.PsfVolume(np.ones((9, 9)), (4, 4), 1.0)).fwhm_bounded

    def test_density_compliance(self, spk, rng):
        from paper_2108_02991_b200.analysis import bin_density

        rho = spk.discretize(spk.DensityParams(0.25, 2.0), 32, 3)
        h = bin_density(rho, 8).ravel()
        cells = rng.choice(h.size, size=10 ** 6, p=h / h.sum())
        idx = np.stack(np.unravel_index(cells, (8, 8, 8)), axis=1)
        pts = (idx + rng.uniform(0, 1, idx.shape)) * 0.25 - 1.0
        l1, _, _ = spk.density_compliance(spk.SamplingPattern(pts.reshape(1, -1, 3)), rho, bins=8)
        assert l1 <= 0.02
        flat = spk.discretize(spk.DensityParams(0.5, 0.0), 16, 2)
        l1, _, _ = spk.density_compliance(spk.SamplingPattern(np.zeros((1, 5000, 2))), flat, bins=8)
        assert l1 == pytest.approx(2.0 * (1.0 - 1.0 / 64), rel=0.01)
        rho2 = spk.discretize(spk.DensityParams(0.25, 2.0), 16, 2)
        l1, hs, hr = spk.density_compliance(spk.SamplingPattern(rng.uniform(-1, 1, (2, 500, 2))),
                                            rho2, bins=8)
        assert hs.sum() == pytest.approx(1.0) and hr.sum() == pytest.approx(1.0)
        assert 0.0 <= l1 <= 2.0
        with pytest.raises(ValueError, match="bins"):
            spk.density_compliance(spk.SamplingPattern(rng.uniform(-1, 1, (1, 10, 2))), rho2,
                                   bins=2)
