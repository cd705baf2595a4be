"""Field-path attraction (bitwise with the reference's grids) and the GPU-resident
optimize loop (drop-in behaviour, determinism, guards, drift vs the reference)."""

import numpy as np
import pytest

from spk_golden import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


def desk_hw(spk, dims=2, matrix=64):
    return spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=1e-5, fov=0.192, matrix=matrix, dims=dims)


def test_field_eval_bitwise_with_reference_grids(spk):
    att = golden("attraction")
    for name in att["names"]:
        fld = spk.KernelField(potential=att[f"{name}_potential"], force=att[f"{name}_force"],
                              grid_n=int(att[f"{name}_n"]), kernel_eps=float(att[f"{name}_eps"]))
        pat = spk.SamplingPattern(att[f"{name}_pts"][None])
        for mode in ("consistent", "smooth"):
            res = spk.eval_attraction(pat, fld, mode)
            assert res.cost == float(att[f"{name}_{mode}_cost"]), (name, mode)
            assert np.array_equal(res.grad, att[f"{name}_{mode}_grad"]), (name, mode)
            assert res.n_clamped == int(att[f"{name}_{mode}_nclamp"])
        from paper_2108_02991_b200.attraction import interpolate

        vals = interpolate(att[f"{name}_potential"], att[f"{name}_pts"], int(att[f"{name}_n"]))
        assert np.array_equal(vals, att[f"{name}_interp"])


def test_n_git_zero_is_projected_init(spk):
    g = golden("optimize")
    cfg = spk.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=0, n_git=0, perturbation=0.2,
                              seed=5, repulsion=spk.RepulsionConfig(backend="direct"))
    res = spk.optimize(cfg, desk_hw(spk))
    assert np.array_equal(res.initial.coords, g["ngit0_initial"])
    assert np.array_equal(res.pattern.coords, g["ngit0_coords"])
    assert len(res.trace.records) == 0


def test_deterministic(spk):
    cfg = spk.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=1, n_git=5, perturbation=0.2,
                              seed=5, repulsion=spk.RepulsionConfig(backend="direct"))
    a = spk.optimize(cfg, desk_hw(spk))
    b = spk.optimize(cfg, desk_hw(spk))
    assert np.array_equal(a.pattern.coords, b.pattern.coords)


@pytest.mark.parametrize("mode", ["consistent", "smooth"])
def test_drift_vs_reference_optimize(spk, mode):
    """Same config / seed / attraction field as the reference run in
    tests/golden/optimize.npz (the reference's own FFT field is passed in, so attraction is
    bit-identical).  The only numeric difference left is the fp32 repulsion sums (rel
    ~1e-6), amplified by the BB steps and active-set changes of the projection; the drift
    is reported and bounded loosely (cost rel 1e-4, coords 1e-3)."""
    g = golden("optimize")
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=1e-5, fov=0.192, matrix=32, dims=2)
    cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=1, n_git=6, n_pit=100,
                              perturbation=0.25, seed=3, grad_mode=mode,
                              repulsion=spk.RepulsionConfig(backend="direct"))
    fld = spk.KernelField(potential=g["field_potential"], force=g["field_force"],
                          grid_n=64, kernel_eps=float(g["field_eps"]))
    res = spk.optimize(cfg, hw, fld=fld)
    costs = res.trace.costs()
    cdrift = np.abs(costs - g[f"{mode}_costs"]).max() / np.abs(g[f"{mode}_costs"]).max()
    drift = np.abs(res.pattern.coords - g[f"{mode}_coords"]).max()
    print(f"[drift] {mode}: cost rel {cdrift:.3e}, max |coords - reference| = {drift:.3e}")
    assert cdrift <= 1e-4
    # The reference itself drifts by 2.0e-2 (consistent: the interpolant gradient is
    # discontinuous across cells) and 7.1e-6 (smooth) under 1e-6 relative noise in the
    # repulsion gradient (scripts/drift_sensitivity.py); bound at ~2.5x / 140x that.
    assert drift <= (5e-2 if mode == "consistent" else 1e-3)


def test_final_pattern_feasible(spk):
    hw = desk_hw(spk)
    cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=2, n_git=8, perturbation=0.25,
                              seed=2, repulsion=spk.RepulsionConfig(backend="direct"))
    res = spk.optimize(cfg, hw)
    lim = spk.normalized_limits(hw)
    pc = spk.ProjectionConfig(alpha=lim.alpha, beta=lim.beta, raster_dt=hw.raster_dt)
    assert spk.feasibility_residuals(res.pattern, pc)["max"] <= pc.feas_tol
    assert res.pattern.samples_per_shot == 64


def test_exact_mode_runs_3d(spk):
    hw = desk_hw(spk, dims=3, matrix=16)
    cfg = spk.OptimizerConfig(n_c=16, n_s=64, dims=3, n_decim=1, n_git=4, grad_mode="exact",
                              seed=2)
    res = spk.optimize(cfg, hw)
    assert np.all(np.isfinite(res.trace.costs()))
    assert len(res.trace.records) == 8


def test_divergence_guard_with_patched_evaluator(spk, monkeypatch):
    import paper_2108_02991_b200.optimizer as om

    calls = {"n": 0}

    def exploding(k, cfg2):
        calls["n"] += 1
        return -(10.0 ** calls["n"]), np.zeros((k.n_samples, k.dims))

    monkeypatch.setattr(om, "eval_repulsion", exploding)
    cfg = spk.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=0, n_git=10, perturbation=0.2,
                              seed=1, repulsion=spk.RepulsionConfig(backend="direct"))
    with pytest.raises(spk.DivergenceError, match="divergence guard"):
        spk.optimize(cfg, desk_hw(spk))


def test_non_finite_aborts(spk, monkeypatch):
    import paper_2108_02991_b200.optimizer as om

    monkeypatch.setattr(om, "eval_repulsion",
                        lambda k, c: (np.nan, np.zeros((k.n_samples, k.dims))))
    cfg = spk.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=0, n_git=5, perturbation=0.2,
                              seed=1)
    with pytest.raises(spk.DivergenceError, match="non-finite"):
        spk.optimize(cfg, desk_hw(spk))


def test_fixed_phase_monotone(spk):
    cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=0, n_git=20, n_pit=400,
                              perturbation=0.25, seed=3,
                              repulsion=spk.RepulsionConfig(backend="direct"))
    res = spk.optimize(cfg, desk_hw(spk))
    # The reference asserts <= 1e-8 (test_optimizer.py:202-211) with fp64 pair sums.  Here
    # the repulsion cost (~0.34) is summed from fp32 pair terms, ~1e-7 relative => ~3e-8
    # absolute noise per evaluated cost; late steps change the cost by only 1e-7..1e-6,
    # so the bound is set at that noise floor (measured worst +6e-8).
    assert np.max(np.diff(res.trace.costs())) <= 1e-7


def test_multiresolution_3d_exact_full3d_limits(spk):
    """C5-shaped schedule at reduced size: 3D, full3d hardware limits, 4 levels
    (N_s = 32 -> 256), exact attraction; every level starts from the upsampled pattern
    and the final pattern is feasible at the unscaled limits."""
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                          dims=3)
    cfg = spk.OptimizerConfig(n_c=64, n_s=256, dims=3, n_decim=3, n_git=3, n_pit=100,
                              perturbation=0.75, seed=0, grad_mode="exact", grid_n=12)
    res = spk.optimize(cfg, hw)
    recs = res.trace.records
    assert [r.samples_per_shot for r in recs] == [32] * 3 + [64] * 3 + [128] * 3 + [256] * 3
    assert np.all(np.isfinite(res.trace.costs()))
    lim = spk.normalized_limits(hw)
    pin = spk.LinearConstraint(128, np.zeros(3))
    pc = spk.ProjectionConfig(alpha=lim.alpha, beta=lim.beta, raster_dt=hw.raster_dt, pin=pin)
    assert spk.feasibility_residuals(res.pattern, pc)["max"] <= pc.feas_tol
    assert res.pattern.coords.shape == (64, 256, 3)


def test_step_api_equals_optimize(spk):
    """start / step / finish (the `step` entry point) reproduces optimize() bitwise."""
    cfg = spk.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=1, n_git=3, perturbation=0.2,
                              seed=7, grad_mode="exact")
    hw = desk_hw(spk)
    ref = spk.optimize(cfg, hw)
    st = spk.start(cfg, hw)
    recs = []
    while (rec := spk.step(st)) is not None:
        recs.append(rec)
    res = spk.finish(st)
    assert len(recs) == 6 and [r.level for r in recs] == [0, 0, 0, 1, 1, 1]
    assert np.array_equal(res.pattern.coords, ref.pattern.coords)
    assert np.array_equal(res.trace.costs(), ref.trace.costs())


@pytest.mark.parametrize("dims,n_c", [(3, 16), (2, 40)])
def test_k2_under_polish_overlap_matches_plain_loop(spk, monkeypatch, dims, n_c):
    """The multi-GPU schedule that runs each polish group's lattice sums (K2) under the
    polish of the slower shots (ShardedRun.overlap, forced on with SPK_OVERLAP=1) gives
    the same iteration as the plain fused loop: projections bit-identical per shot, K2 from
    a different chunking (fp32 partial sums, ~1e-7), so costs agree to 1e-6 relative and
    trajectories by far less than the reference's own noise drift."""
    hw = desk_hw(spk, dims=dims, matrix=16)
    cfg = spk.OptimizerConfig(n_c=n_c, n_s=64, dims=dims, n_decim=1, n_git=6,
                              grad_mode="exact", seed=4, grid_n=12)
    monkeypatch.setenv("SPK_OVERLAP", "0")
    plain = spk.optimize(cfg, hw)
    monkeypatch.setenv("SPK_OVERLAP", "1")
    from paper_2108_02991_b200 import optimizer as om

    st = om.start(cfg, hw)
    assert st.run.overlap
    ovl = om.finish(st)
    rel = np.abs(ovl.trace.costs() - plain.trace.costs()) / np.abs(plain.trace.costs())
    assert rel.max() <= 1e-6, rel.max()
    assert np.abs(ovl.pattern.coords - plain.pattern.coords).max() <= 1e-5


@pytest.mark.parametrize("dims,n_c", [(3, 16), (2, 40)])
def test_k1_pipeline_matches_plain_loop(spk, monkeypatch, dims, n_c):
    """K1 block by block under the polish (engine.k1_pipelined, opt-in with SPK_K1_PIPE=1,
    here on one GPU): per-group gathers on a side stream,
    (target group, source group) K1 blocks on another, shot-order scatter -- the same
    iteration as the plain fused loop to fp32 partial-sum order."""
    hw = desk_hw(spk, dims=dims, matrix=16)
    cfg = spk.OptimizerConfig(n_c=n_c, n_s=64, dims=dims, n_decim=1, n_git=6,
                              grad_mode="exact", seed=4, grid_n=12)
    monkeypatch.setenv("SPK_OVERLAP", "0")
    plain = spk.optimize(cfg, hw)
    monkeypatch.setenv("SPK_OVERLAP", "1")
    monkeypatch.setenv("SPK_K1_PIPE", "1")
    from paper_2108_02991_b200 import engine
    from paper_2108_02991_b200 import optimizer as om

    calls = []
    orig = engine.k1_pipelined

    def counted(*a, **k):
        out = orig(*a, **k)
        calls.append(out is not None)
        return out

    monkeypatch.setattr(engine, "k1_pipelined", counted)
    st = om.start(cfg, hw)
    assert st.run.overlap
    pipe = om.finish(st)
    assert calls and all(calls)
    rel = np.abs(pipe.trace.costs() - plain.trace.costs()) / np.abs(plain.trace.costs())
    assert rel.max() <= 1e-6, rel.max()
    assert np.abs(pipe.pattern.coords - plain.pattern.coords).max() <= 1e-5


def test_spatial_target_partition_on_device(spk, monkeypatch):
    """The treecodes' spatial layout (ShardedRun.spatial: N-body targets in Morton-order
    blocks, results returned to the shot owners; forced on a single GPU with
    SPK_SPATIAL=1) gives the same iteration as the shot layout to the treecode's
    precision: the lattice treecode groups a differently ordered target set."""
    hw = desk_hw(spk, dims=3, matrix=16)
    cfg = spk.OptimizerConfig(n_c=16, n_s=64, dims=3, n_decim=1, n_git=4, grad_mode="exact",
                              seed=4, grid_n=12, attraction_tree_precision=1e-4)
    monkeypatch.setenv("SPK_SPATIAL", "0")
    plain = spk.optimize(cfg, hw)
    monkeypatch.setenv("SPK_SPATIAL", "1")
    from paper_2108_02991_b200 import optimizer as om

    st = om.start(cfg, hw)
    assert st.run.spatial
    sp = om.finish(st)
    rel = np.abs(sp.trace.costs() - plain.trace.costs()) / np.abs(plain.trace.costs())
    assert rel.max() <= 1e-4, rel.max()
    assert np.abs(sp.pattern.coords - plain.pattern.coords).max() <= 1e-3
