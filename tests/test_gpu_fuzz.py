"""Randomised parity (hypothesis, derandomised).  Projection: shot length, dims, pin
position (incl. the ends), bounds, monotone mode, n_pit and the sweep cap drawn at
random; the GPU K3 must equal the CPU oracle bit for bit, outputs and sweep counts.
The ring's edge cases -- N_s below one warp, a pin at sample 0 / N_s - 1, caps that stop
inside a ring round -- are all in the drawn space."""

import numpy as np
import pytest
from hypothesis import HealthCheck, assume, given, settings
from hypothesis import strategies as st

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@st.composite
def cases(draw):
    dims = draw(st.sampled_from([2, 3]))
    ns = draw(st.sampled_from([3, 4, 5, 7, 16, 31, 33, 64, 100, 129, 257, 300, 700, 1030]))
    n_c = draw(st.integers(1, 6))
    pin = draw(st.sampled_from([-1, 0, ns // 2, ns - 1]))
    a = draw(st.sampled_from([0.02, 0.05, 0.2, 0.5]))
    b = draw(st.sampled_from([0.005, 0.01, 0.05, 0.3]))
    mono = draw(st.booleans())
    n_pit = draw(st.sampled_from([1, 5, 40]))
    cap = draw(st.sampled_from([1, 7, 33, 300, 50000]))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    scale = draw(st.sampled_from([0.3, 1.0, 1.4]))
    return dims, ns, n_c, pin, a, b, mono, n_pit, cap, seed, scale


@settings(max_examples=150, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(cases())
def test_projection_bitwise_random(case):
    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.projection import project_device
    import torch

    dims, ns, n_c, pin, a, b, mono, n_pit, cap, seed, scale = case
    rng = np.random.default_rng(seed)
    shots = rng.uniform(-scale, scale, (n_c, ns, dims))
    pv = rng.uniform(-0.3, 0.3, dims) if pin >= 0 else None
    pc = None if pin < 0 else spk.LinearConstraint(pin, pv)
    cfg = spk.ProjectionConfig(alpha=a, beta=b, raster_dt=1.0, n_pit=n_pit, pin=pc,
                               monotone=mono)
    tau = 1.0 / spk.projection.stacked_operator_norm(ns, pin)
    dev = _device.h2d(shots)
    sw = torch.zeros(n_c, dtype=torch.int32, device=dev.device)
    out = _device.d2h(project_device(dev, cfg, tau=tau, sweeps=sw, max_sweeps=cap))
    ref, rsw = orc.project_all(shots, a, b, pin, pv, n_pit, tau, 0.1 * cfg.feas_tol,
                               monotone=mono, max_sweeps=cap)
    assert np.array_equal(_device.d2h(sw), rsw), case
    assert np.array_equal(out, ref), (case, np.abs(out - ref).max())


@st.composite
def clouds(draw):
    dims = draw(st.sampled_from([2, 3]))
    p = draw(st.sampled_from([1, 2, 31, 513, 4099, 20000]))
    kind = draw(st.sampled_from(["uniform", "radial", "clustered", "duplicates"]))
    eps = draw(st.sampled_from([0.0, 1e-3, 0.05]))
    return dims, p, kind, eps, draw(st.integers(0, 2 ** 31 - 1))


def _cloud(dims, p, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(-1, 1, (p, dims))
    if kind == "radial":
        v = rng.normal(size=(p, dims))
        return (rng.uniform(0, 1, p) ** 2)[:, None] * v / np.linalg.norm(v, axis=1, keepdims=True)
    if kind == "clustered":
        c = rng.uniform(-0.8, 0.8, (4, dims))
        return c[rng.integers(0, 4, p)] + 1e-3 * rng.normal(size=(p, dims))
    base = rng.uniform(-1, 1, (max(1, p // 3), dims))
    return base[rng.integers(0, base.shape[0], p)]  # exact duplicates


@settings(max_examples=40, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(clouds())
def test_direct_sums_random_clouds(case):
    """K1 vs the fp64 oracle on random clouds (incl. exact duplicates with eps = 0, where
    coincident pairs contribute nothing): value rel l2 <= 1e-5, gradient <= 1e-4."""
    import paper_2108_02991_b200  # noqa: F401
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.repulsion import direct_sums_device

    dims, p, kind, eps, seed = case
    pts = _cloud(dims, p, kind, seed)
    p4 = _device.pack_positions(_device.h2d(pts))
    val, grad = direct_sums_device(p4, p4, dims, eps * eps)
    vref, gref = orc.direct_sums(pts, eps * eps)
    val, grad = _device.d2h(val), _device.d2h(grad)
    if np.linalg.norm(vref) > 0:
        assert np.linalg.norm(val - vref) / np.linalg.norm(vref) <= 1e-5, case
    else:
        assert np.all(val == 0.0), case
    gn = np.linalg.norm(gref)
    if gn > 1e-12 * max(1.0, np.linalg.norm(vref)):
        assert np.linalg.norm(grad - gref) / gn <= 1e-4, case
    assert np.all(np.isfinite(grad)), case


@settings(max_examples=24, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from(["uniform", "radial", "clustered", "duplicates"]),
       st.sampled_from([1e-2, 1e-3, 1e-4, 1e-5, 1e-6]), st.integers(0, 2 ** 31 - 1))
def test_treecode_precision_contract_random_clouds(dims, kind, prec, seed):
    """eval_repulsion_tree meets tree_precision on cost and gradient l2 on random clouds
    large enough (150k) to run the treecode, incl. clustered and duplicated points."""
    import paper_2108_02991_b200 as spk

    # Against the exact fp32-pair kernel: its own distance to fp64 is ~4e-8 on spread
    # clouds but ~3e-6 on clouds clustered at the eps scale (fp32 cancellation in
    # t - s; scripts/fp32_floor.py), within the north star's 1e-4 (checked against the
    # oracle by test_direct_sums_random_clouds) -- so the 1e-6 row is a contract on the
    # approximation, not on fp64 agreement, for such clouds.
    # On eps-scale clusters the fp32 arithmetic of the proxies and of the exact kernel
    # differ by ~1e-6 themselves, so the 1e-6 row is only asserted on the other clouds.
    assume(not (kind == "clustered" and prec < 1e-5))
    pts = _cloud(dims, 150_000, kind, seed)
    cfg = spk.RepulsionConfig(backend="tree", tree_precision=prec)
    c_t, g_t = spk.eval_repulsion_tree(pts, cfg)
    c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
    assert abs(c_t - c_d) / abs(c_d) <= prec, (dims, kind, prec)
    assert np.linalg.norm(g_t - g_d) / np.linalg.norm(g_d) <= prec, (dims, kind, prec)


@settings(max_examples=16, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from(["uniform", "radial", "clustered"]),
       st.sampled_from([1e-2, 1e-3, 1e-4, 1e-5]), st.sampled_from([0.1, 0.25, 0.5]),
       st.sampled_from([0.0, 1.0, 2.0, 4.0]), st.integers(0, 2 ** 31 - 1))
def test_attraction_treecode_precision_random(dims, kind, prec, cutoff, decay, seed):
    """The lattice treecode (attraction_tree_precision) meets its precision on the cost
    and the gradient l2 against exact K2, for random densities and target clouds."""
    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.attraction import grid_sums_device, tree_grid_sums_device

    n = 96 if dims == 2 else 24
    fld = spk.precompute_field(spk.discretize(spk.DensityParams(cutoff, decay), n, dims))
    pts = np.clip(_cloud(dims, 100_000, kind, seed), -1.0, 1.0)
    p4 = _device.pack_positions(_device.h2d(pts))
    eps2 = fld.kernel_eps ** 2
    v0, g0 = (_device.d2h(x) for x in grid_sums_device(p4, fld, eps2))
    v1, g1 = (_device.d2h(x) for x in tree_grid_sums_device(p4, fld, eps2, prec))
    case = (dims, kind, prec, cutoff, decay)
    assert abs(v1.sum() - v0.sum()) / abs(v0.sum()) <= prec, case
    assert np.linalg.norm(g1 - g0) / np.linalg.norm(g0) <= prec, case


@settings(max_examples=30, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.integers(1, 3000), st.integers(1, 70), st.integers(1, 70),
       st.integers(1, 40), st.sampled_from(["fp64", "mixed"]), st.integers(0, 2 ** 31 - 1))
def test_nudft_random_shapes(dims, p, n0, n1, n2, precision, seed):
    """Adjoint and forward NUDFT on random sample counts and grid shapes (odd, even,
    1-wide axes) vs the numpy dense-phase oracle: 1e-12 (fp64) / 2e-5 (mixed) of max."""
    from oracle import nudft_oracle as no
    from paper_2108_02991_b200.analysis import nudft_adjoint, nudft_forward

    grid = (n0, n1) if dims == 2 else (n0, n1, n2)
    if p * int(np.prod(grid)) > 4_000_000:  # keep the numpy oracle small
        p = max(1, 4_000_000 // int(np.prod(grid)))
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-1, 1, (p, dims))
    w = rng.normal(size=p) + 1j * rng.normal(size=p)
    img = rng.normal(size=grid) + 1j * rng.normal(size=grid)
    tol = 1e-12 if precision == "fp64" else 2e-5
    ref = no.nudft_adjoint(pts, w, grid)
    got = nudft_adjoint(pts, w, grid, precision=precision)
    assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), (grid, p, precision)
    ref = no.nudft_forward(pts, img)
    got = nudft_forward(pts, img, precision=precision)
    assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), (grid, p, precision)


@settings(max_examples=12, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from(["uniform", "radial", "clustered"]),
       st.integers(2, 6), st.sampled_from([1e-3, 1e-4, 1e-5]), st.integers(0, 2 ** 31 - 1))
def test_explicit_order_probe_meets_precision(dims, kind, order, prec, seed):
    """An explicit interp_order goes through the reference's 64-target probe: it escalates
    the order (or falls back to exact sums) until the probe meets tree_precision; the
    result then meets it on the full gradient too (repulsion.py:165-200)."""
    import warnings

    import paper_2108_02991_b200 as spk

    pts = _cloud(dims, 150_000, kind, seed)
    cfg = spk.RepulsionConfig(backend="tree", tree_precision=prec, interp_order=order)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        c_t, g_t = spk.eval_repulsion_tree(pts, cfg)
    c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
    # the probe checks 64 targets, so allow 3x on the full-cloud l2 (the reference's probe
    # has the same sampling limitation)
    assert abs(c_t - c_d) / abs(c_d) <= 3 * prec, (dims, kind, order, prec)
    assert np.linalg.norm(g_t - g_d) / np.linalg.norm(g_d) <= 3 * prec, (dims, kind, order, prec)


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from([4, 9, 16]), st.sampled_from([32, 64, 128]),
       st.sampled_from([0, 1]), st.sampled_from([0.0, 0.25, 0.75]), st.integers(0, 10_000))
def test_optimize_gpu_vs_oracle_engine(dims, n_c, n_s, n_decim, pert, seed):
    """The whole GPU-resident optimize loop (exact mode) against the same engine driven by
    the CPU oracle ops (fp64 sums of the fp32-rounded positions): the only difference is
    the fp32 pair arithmetic, so costs agree to 1e-6 and coordinates to ~1e-6 after a few
    fixed-step iterations."""
    from cpu_ops import OracleOps

    import paper_2108_02991_b200 as spk

    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=1e-5, fov=0.192, matrix=32, dims=dims)
    cfg = spk.OptimizerConfig(n_c=n_c, n_s=n_s, dims=dims, n_decim=n_decim, n_git=3, n_pit=40,
                              grad_mode="exact", grid_n=8, seed=seed, perturbation=pert)
    gpu = spk.optimize(cfg, hw)
    cpu = spk.optimize(cfg, hw, ops=OracleOps())
    cg, cc = gpu.trace.costs(), cpu.trace.costs()
    assert np.abs(cg - cc).max() <= 1e-6 * np.abs(cc).max(), (cg, cc)
    # coordinates: the ~1e-6 relative gradient difference times the fixed step (eta0 =
    # 1024 eps p) moves samples by ~1e-6 before the projection; measured worst 1.3e-6
    assert np.abs(gpu.pattern.coords - cpu.pattern.coords).max() <= 1e-5


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from(["uniform", "radial", "clustered"]),
       st.sampled_from([2, 3, 8]), st.integers(0, 7), st.sampled_from([1e-3, 1e-4]),
       st.integers(0, 2 ** 31 - 1))
def test_sharded_targets_treecode(dims, kind, world, rank, prec, seed):
    """A rank's contiguous target shard against all sources (the multi-GPU form of the
    treecode repulsion) meets the precision on that shard."""
    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.repulsion import direct_sums_device, tree_sums_checked

    rank = rank % world
    pts = _cloud(dims, 200_000, kind, seed)
    lo, hi = pts.shape[0] * rank // world, pts.shape[0] * (rank + 1) // world
    src4 = _device.pack_positions(_device.h2d(pts))
    tgt4 = src4[lo:hi].contiguous()
    cfg = spk.RepulsionConfig(backend="tree", tree_precision=prec)
    v1, g1 = (_device.d2h(x) for x in tree_sums_checked(tgt4, src4, dims, cfg))
    v0, g0 = (_device.d2h(x) for x in direct_sums_device(tgt4, src4, dims, cfg.kernel_eps ** 2))
    assert abs(v1.sum() - v0.sum()) / abs(v0.sum()) <= prec, (dims, kind, world, rank, prec)
    assert np.linalg.norm(g1 - g0) / np.linalg.norm(g0) <= prec, (dims, kind, world, rank, prec)


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from(["uniform", "radial", "clustered", "duplicates"]),
       st.sampled_from([128, 512, 1024]), st.sampled_from([(4, 0.7, 1e-3), (5, 0.7, 1e-4)]),
       st.integers(0, 2 ** 31 - 1))
def test_far_level_random_clouds(dims, kind, cap, row, seed):
    """The far level (P2L at parents' Chebyshev points + L2P; the repulsion uses it from
    4M targets) on random clouds and parent capacities: every source counted once, the
    row's precision met (same bar as the plain walk)."""
    from paper_2108_02991_b200 import _device, tree
    from paper_2108_02991_b200.repulsion import direct_sums_device

    order, theta, prec = row
    pts = _cloud(dims, 200_000, kind, seed)
    pos4 = _device.pack_positions(_device.h2d(pts))
    src = tree.SourceTree(pos4, dims)
    tg = tree.TargetGroups(pos4, dims, same_as=src, parent_cap=cap)
    vt, gt = (_device.d2h(x) for x in tree.tree_eval(tg, src, order, theta, 1e-6, static=True))
    vd, gd = (_device.d2h(x) for x in direct_sums_device(pos4, pos4, dims, 1e-6))
    case = (dims, kind, cap, row)
    assert abs(vt.sum() - vd.sum()) / abs(vd.sum()) <= prec, case
    assert np.linalg.norm(gt - gd) / np.linalg.norm(gd) <= prec, case


def _residuals_numpy(coords, speed_bound, accel_bound, pin):
    """feasibility_residuals restated in numpy (projection.py:435-452)."""
    amp = float(np.max(np.abs(coords)) - 1.0)
    d1 = np.linalg.norm(np.diff(coords, axis=1), axis=2)
    d2 = np.linalg.norm(np.diff(coords, 2, axis=1), axis=2)
    res = {"amplitude": max(amp, 0.0),
           "speed": max(float(d1.max() - speed_bound) if d1.size else -np.inf, 0.0),
           "acceleration": max(float(d2.max() - accel_bound) if d2.size else -np.inf, 0.0)}
    if pin is not None:
        res["pin"] = float(np.abs(coords[:, pin.pinned_index, :] - pin.pinned_value).max())
    res["max"] = max(res.values())
    return res


@settings(max_examples=60, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.integers(1, 5), st.sampled_from([2, 3, 5, 64, 257]),
       st.booleans(), st.sampled_from([0.3, 1.0, 1.3]), st.integers(0, 2 ** 31 - 1),
       st.sampled_from([0.0, 1e-3, 0.3]))
def test_step_projection_and_residuals(dims, n_c, ns, pinned, scale, seed, eta):
    """The optimizer's fused step + projection (in = coords - eta * grad, per-shot eta
    too) bit-identical to the oracle on the stepped input, and feasibility_residuals
    bit-identical to the reference's numpy formula."""
    import torch

    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.projection import project_device

    rng = np.random.default_rng(seed)
    coords = rng.uniform(-scale, scale, (n_c, ns, dims))
    grad = rng.normal(size=coords.shape)
    pin = spk.LinearConstraint(ns // 2, rng.uniform(-0.2, 0.2, dims)) if pinned else None
    cfg = spk.ProjectionConfig(alpha=0.08, beta=0.02, raster_dt=1.0, n_pit=15, pin=pin)
    pin_idx = -1 if pin is None else pin.pinned_index
    tau = 1.0 / spk.projection.stacked_operator_norm(ns, pin_idx)
    etas = rng.uniform(0, 2 * eta, n_c) if eta > 0 else np.zeros(n_c)
    for per_shot in (False, True):
        stepped = coords - (etas[:, None, None] if per_shot else eta) * grad
        d_eta = _device.h2d(etas) if per_shot else None
        out = _device.d2h(project_device(_device.h2d(coords), cfg, grad=_device.h2d(grad),
                                         eta=eta, tau=tau, eta_per_shot=d_eta))
        ref, _ = orc.project_all(stepped, cfg.speed_bound, cfg.accel_bound, pin_idx,
                                 None if pin is None else pin.pinned_value, 15, tau,
                                 0.1 * cfg.feas_tol)
        assert np.array_equal(out, ref), (dims, n_c, ns, pinned, per_shot)
    for pat in (coords, ref):
        got = spk.feasibility_residuals(spk.SamplingPattern(pat), cfg)
        want = _residuals_numpy(pat, cfg.speed_bound, cfg.accel_bound, pin)
        assert got == want, (got, want)


@settings(max_examples=20, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.integers(2, 40), st.integers(2, 40), st.integers(2, 20),
       st.sampled_from([0.1, 0.25, 0.5]), st.sampled_from([0.0, 2.0, 4.0]),
       st.integers(1, 3000), st.integers(0, 2 ** 31 - 1))
def test_exact_attraction_anisotropic_random(dims, n0, n1, n2, cutoff, decay, p, seed):
    """K2 over random anisotropic (2 N_a + 1 per axis) lattices and random targets
    (incl. outside [-1, 1]) vs the fp64 oracle: cost 1e-5, gradient rel l2 1e-4."""
    import paper_2108_02991_b200 as spk

    ns = (n0, n1) if dims == 2 else (n0, n1, n2)
    rho = spk.discretize_anisotropic(spk.DensityParams(cutoff, decay), ns, dims)
    fld = spk.precompute_field(rho)
    pts = np.random.default_rng(seed).uniform(-1.1, 1.1, (p, dims))
    res = spk.eval_attraction(spk.SamplingPattern(pts[None]), fld, "exact")
    cref, gref = orc.attraction_exact(pts, rho.grid, fld.kernel_eps)
    assert abs(res.cost - cref) <= 1e-5 * abs(cref), ns
    assert np.linalg.norm(res.grad - gref) <= 1e-4 * max(np.linalg.norm(gref), 1e-300), ns


@settings(max_examples=8, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from([4, 9]), st.sampled_from([32, 64]),
       st.sampled_from([0, 1]), st.sampled_from(["exact", "consistent", "smooth"]),
       st.integers(1, 5), st.integers(0, 1000))
def test_stack_vs_individual_random(dims, n_c, n_s, n_decim, mode, n_prob, seed):
    """optimize_stack (independent problems as one device batch) follows each
    single-problem optimize(): same init, costs to 1e-9, coordinates to 1e-6."""
    import paper_2108_02991_b200 as spk

    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=1e-5, fov=0.192, matrix=32, dims=dims)
    cfg = spk.OptimizerConfig(n_c=n_c, n_s=n_s, dims=dims, n_decim=n_decim, n_git=3,
                              perturbation=0.25, seed=seed, grad_mode=mode, grid_n=8)
    batch = spk.optimize_stack(cfg, hw, n_prob)
    for q, res in enumerate(batch):
        single = spk.optimize(spk.OptimizerConfig(**{**cfg.__dict__, "seed": seed + q}), hw)
        assert np.array_equal(res.initial.coords, single.initial.coords)
        c1, c2 = res.trace.costs(), single.trace.costs()
        assert np.abs(c1 - c2).max() <= 1e-9 * np.abs(c2).max(), (q, c1, c2)
        assert np.abs(res.pattern.coords - single.pattern.coords).max() <= 1e-6


@settings(max_examples=10, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.sampled_from([2, 3]), st.sampled_from([4, 9, 16, 25]), st.sampled_from([32, 64, 96]),
       st.sampled_from([0, 1]), st.sampled_from([0.25, 0.75]), st.integers(0, 10_000),
       st.sampled_from(["overlap", "spatial"]))
def test_schedules_match_plain_loop(dims, n_c, n_s, n_decim, pert, seed, schedule):
    """The multi-GPU schedules on random configurations, forced on one GPU: K2 under the
    polish (exact sums) and the Morton-order target layout (lattice treecode) each give
    the plain loop's trajectory to the accuracy of their sums."""
    import os

    import paper_2108_02991_b200 as spk

    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=1e-5, fov=0.192, matrix=32, dims=dims)
    extra = {} if schedule == "overlap" else {"attraction_tree_precision": 1e-4}
    cfg = spk.OptimizerConfig(n_c=n_c, n_s=n_s, dims=dims, n_decim=n_decim, n_git=3, n_pit=40,
                              grad_mode="exact", grid_n=8, seed=seed, perturbation=pert,
                              **extra)
    env = "SPK_OVERLAP" if schedule == "overlap" else "SPK_SPATIAL"
    old = os.environ.get(env)
    try:
        os.environ[env] = "0"
        plain = spk.optimize(cfg, hw)
        os.environ[env] = "1"
        other = spk.optimize(cfg, hw)
    finally:
        if old is None:
            os.environ.pop(env, None)
        else:
            os.environ[env] = old
    tol = 1e-6 if schedule == "overlap" else 1e-4
    cp, co = plain.trace.costs(), other.trace.costs()
    assert np.abs(co - cp).max() <= tol * np.abs(cp).max(), (schedule, co, cp)
    assert np.abs(other.pattern.coords - plain.pattern.coords).max() <= 1e-3
