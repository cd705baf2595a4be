"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the authoring container only (the reference does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``vdtraj`` from /root/reference/pkg/src (read-only, never copied) and writes
small ``.npz`` files of seeded inputs and the reference's outputs.  The tests compare
the CPU oracle (bitwise), the host-side mirror (bitwise) and the CUDA kernels (bitwise
for fp64 projection, tolerance for fp32 N-body) against these vectors.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from vdtraj import _treecode as tc  # noqa: E402
from vdtraj import attraction as at  # noqa: E402
from vdtraj import core, density, optimizer as om, projection as pr  # noqa: E402
from vdtraj.repulsion import eval_repulsion_direct  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def radial_cloud(rng, p, d):
    r = rng.uniform(0, 1, p) ** 2
    v = rng.normal(size=(p, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return np.ascontiguousarray(r[:, None] * v)


def repulsion_fixtures():
    rng = np.random.default_rng(20260101)
    cases = {}
    inputs = {
        "u2d": (rng.uniform(-1, 1, (257, 2)), 1e-6),
        "r3d": (radial_cloud(rng, 300, 3), 1e-6),
        "pair0": (np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]]), 0.0),
        "coinc": (np.zeros((3, 2)), 0.01),
        "spokes3d": (om.perturb(om.init_radial(16, 64, 3), 0.25, 0).points().copy(), 1e-6),
        "spokes2d": (om.perturb(om.init_radial(8, 128, 2), 0.25, 0).points().copy(), 1e-6),
        "dup3d": (np.repeat(rng.uniform(-0.5, 0.5, (40, 3)), 3, axis=0), 1e-6),
    }
    for name, (pts, eps2) in inputs.items():
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        val = np.empty(pts.shape[0])
        grad = np.empty_like(pts)
        tc.direct_sums(pts, eps2, val, grad)
        cases[f"{name}_pos"] = pts
        cases[f"{name}_eps2"] = np.float64(eps2)
        cases[f"{name}_val"] = val
        cases[f"{name}_grad"] = grad
        c, g = eval_repulsion_direct(pts, float(np.sqrt(eps2)))
        cases[f"{name}_cost"] = np.float64(c)
        cases[f"{name}_gnorm"] = g
    # subset rows
    pts = cases["spokes3d_pos"]
    tg = np.arange(0, pts.shape[0], 7, dtype=np.int64)
    val = np.empty(tg.shape[0])
    grad = np.empty((tg.shape[0], 3))
    tc.direct_sums_subset(pts, tg, 1e-6, val, grad)
    cases["subset_targets"] = tg
    cases["subset_val"] = val
    cases["subset_grad"] = grad
    cases["names"] = np.array(list(inputs.keys()))
    np.savez_compressed(os.path.join(OUT, "repulsion.npz"), **cases)


def attraction_fixtures():
    rng = np.random.default_rng(20260202)
    out = {}
    # (name, grid, grid_n, eps)
    specs = [
        ("d2", density.discretize(density.DensityParams(0.25, 2.0), 8, 2).grid, 8, 0.05),
        ("d3", density.discretize(density.DensityParams(0.25, 2.0), 4, 3).grid, 4, None),
        ("r2", density.TargetDensity(rng.uniform(0, 1, (13, 13)), 6).grid, 6, 0.1),
        ("delta2", None, 8, 0.05),
    ]
    for name, grid, n, eps in specs:
        if grid is None:
            grid = np.zeros((2 * n + 1,) * 2)
            grid[n, n] = 1.0
        rho = density.TargetDensity(grid=grid, grid_n=n)
        fld = at.precompute_field(rho, kernel_eps=eps)
        out[f"{name}_rho"] = rho.grid
        out[f"{name}_n"] = np.int64(n)
        out[f"{name}_eps"] = np.float64(fld.kernel_eps)
        out[f"{name}_potential"] = fld.potential
        out[f"{name}_force"] = fld.force
        d = rho.dims
        pts = rng.uniform(-1.05, 1.05, (37, d))
        pts[0] = 0.0
        pts[1] = np.array([1.0, -1.0, 0.5][:d])  # on the boundary / a node
        pat = core.SamplingPattern(pts[None])
        for mode in ("consistent", "smooth"):
            res = at.eval_attraction(pat, fld, mode)
            out[f"{name}_{mode}_cost"] = np.float64(res.cost)
            out[f"{name}_{mode}_grad"] = res.grad
            out[f"{name}_{mode}_nclamp"] = np.int64(res.n_clamped)
        out[f"{name}_pts"] = pts
        out[f"{name}_interp"] = at.interpolate(fld.potential, pts, n)
    out["names"] = np.array([s[0] for s in specs])
    np.savez_compressed(os.path.join(OUT, "attraction.npz"), **out)


def _project_case(shot, cfg, want_trace=False):
    if want_trace:
        o, tr = pr.project_shot(shot, cfg, return_trace=True)
        return o, tr
    return pr.project_shot(shot, cfg), None


def projection_fixtures():
    rng = np.random.default_rng(20260303)
    out = {}
    names = []

    def add(name, shots, cfg, trace=False):
        names.append(name)
        pin_idx, pin_val = pr._pin_arrays(cfg, shots.shape[2])
        out[f"{name}_in"] = shots
        out[f"{name}_a"] = np.float64(cfg.speed_bound)
        out[f"{name}_b"] = np.float64(cfg.accel_bound)
        out[f"{name}_pin"] = np.int64(pin_idx)
        out[f"{name}_pinval"] = pin_val
        out[f"{name}_npit"] = np.int64(cfg.n_pit)
        out[f"{name}_mono"] = np.int64(cfg.monotone)
        out[f"{name}_tol"] = np.float64(0.1 * cfg.feas_tol)
        out[f"{name}_lam"] = np.float64(pr._stacked_operator_norm(shots.shape[1], pin_idx))
        if trace:
            o, tr = pr.project_shot(shots[0], cfg, return_trace=True)
            out[f"{name}_out"] = o[None]
            out[f"{name}_trace"] = tr
        else:
            out[f"{name}_out"] = pr.project_pattern(core.SamplingPattern(shots), cfg).coords
        # FISTA-only output (n_pit iterations, no polish) via the numba kernel
        fo = np.empty_like(shots)
        for c in range(shots.shape[0]):
            pr._project_shot(shots[c], cfg.speed_bound, cfg.accel_bound, pin_idx, pin_val,
                             cfg.n_pit, 1.0 / out[f"{name}_lam"], cfg.monotone, fo[c],
                             np.empty(0))
        out[f"{name}_fista"] = fo

    desk = dict(alpha=10216.0, beta=4.6e7, raster_dt=1e-5)
    add("desk2d", rng.uniform(-1.1, 1.1, (6, 24, 2)), pr.ProjectionConfig(n_pit=60, **desk))
    add("qp2d", rng.uniform(-1.5, 1.5, (3, 8, 2)),
        pr.ProjectionConfig(alpha=0.3, beta=0.15, raster_dt=1.0, n_pit=1000))
    pin = core.LinearConstraint(pinned_index=3, pinned_value=np.array([0.1, -0.2]))
    add("pin2d", rng.uniform(-1.2, 1.2, (2, 9, 2)),
        pr.ProjectionConfig(alpha=0.4, beta=0.2, raster_dt=1.0, n_pit=200, pin=pin))
    add("mono2d", rng.uniform(-1.4, 1.4, (1, 32, 2)),
        pr.ProjectionConfig(alpha=0.3, beta=0.15, raster_dt=1.0, n_pit=150, monotone=True),
        trace=True)
    add("trace3d", rng.uniform(-1.2, 1.2, (1, 20, 3)),
        pr.ProjectionConfig(alpha=0.5, beta=0.3, raster_dt=1.0, n_pit=80), trace=True)
    add("clamp2d", np.full((1, 12, 2), 1.5),
        pr.ProjectionConfig(alpha=1e9, beta=1e12, raster_dt=1.0, n_pit=200))
    add("tiny", rng.uniform(-1.5, 1.5, (3, 2, 3)),
        pr.ProjectionConfig(alpha=0.3, beta=0.1, raster_dt=1.0, n_pit=30))
    # In-loop 3D shots at full3d hardware limits (scale 4): projected init + a step.
    hw = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                           dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                           dims=3)
    lim = core.normalized_limits(hw).scaled(4.0)
    ns = 512
    pin3 = core.LinearConstraint(pinned_index=ns // 2, pinned_value=np.zeros(3))
    cfg3 = pr.ProjectionConfig(alpha=lim.alpha, beta=lim.beta, raster_dt=1e-5, n_pit=100,
                               pin=pin3)
    base = om.perturb(om.init_radial(9, ns, 3), 0.75, 0)
    feas = pr.project_pattern(base, cfg3)
    stepped = feas.coords[:4] + rng.uniform(-2e-3, 2e-3, (4, ns, 3))
    add("inloop3d", stepped, cfg3)
    add("fresh3d", base.coords[:2].copy(), cfg3)
    # 2D in-loop shots at desk limits, N_s=256 (config-1-like)
    hw2 = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=2e-6, fov=0.192, matrix=64, dims=2)
    lim2 = core.normalized_limits(hw2)
    pin2 = core.LinearConstraint(pinned_index=128, pinned_value=np.zeros(2))
    cfg2 = pr.ProjectionConfig(alpha=lim2.alpha, beta=lim2.beta, raster_dt=1e-5, n_pit=100,
                               pin=pin2)
    base2 = om.perturb(om.init_radial(8, 256, 2), 0.25, 1)
    feas2 = pr.project_pattern(base2, cfg2)
    add("inloop2d", feas2.coords[:3] + rng.uniform(-5e-3, 5e-3, (3, 256, 2)), cfg2)

    # Polish-only cases with sweep counts (reference kernel called directly).
    pol_in = out["inloop3d_fista"][:2].copy()
    pol_out = pol_in.copy()
    for c in range(2):
        pr._feasibility_polish(pol_out[c], cfg3.speed_bound, cfg3.accel_bound, ns // 2,
                               np.zeros(3), 1e-7, 50000)
    out["polish_in"] = pol_in
    out["polish_out"] = pol_out
    out["polish_a"] = np.float64(cfg3.speed_bound)
    out["polish_b"] = np.float64(cfg3.accel_bound)
    out["polish_pin"] = np.int64(ns // 2)
    # max_sweeps-capped polish
    capped = pol_in.copy()
    for c in range(2):
        pr._feasibility_polish(capped[c], cfg3.speed_bound, cfg3.accel_bound, ns // 2,
                               np.zeros(3), 1e-7, 37)
    out["polish_capped37"] = capped

    # operator norms
    lam_keys = [(32, 16), (1024, 512), (2048, 1024), (256, -1), (9, 3), (2, -1), (3, 1)]
    out["lam_keys"] = np.array(lam_keys, dtype=np.int64)
    out["lam_vals"] = np.array([pr._stacked_operator_norm(n, p) for n, p in lam_keys])
    # feasibility residuals
    fr = pr.feasibility_residuals(core.SamplingPattern(out["inloop3d_in"]), cfg3)
    out["feas_inloop3d_in"] = np.array([fr["amplitude"], fr["speed"], fr["acceleration"],
                                        fr["pin"], fr["max"]])
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "projection.npz"), **out)


def nonfinite_fixtures():
    """The reference's _project_all on shots holding NaN / +-inf samples (numba kernel
    called directly: SamplingPattern rejects non-finite coordinates at the API)."""
    rng = np.random.default_rng(20261019)
    out = {}
    names = []
    for d in (2, 3):
        for ns, pin in ((64, -1), (300, 150)):
            name = f"nf{d}_{ns}"
            shots = rng.uniform(-1.3, 1.3, (4, ns, d))
            shots[0, 10, 0] = np.nan
            shots[1, 20, d - 1] = np.inf
            shots[2, 5, 1] = -np.inf
            shots[2, 7, 0] = np.nan
            a, b, pv = 0.05, 0.01, np.full(d, 0.05)
            lam = pr._stacked_operator_norm(ns, pin)
            res = np.empty_like(shots)
            pr._project_all(shots, a, b, pin, pv, 50, 1.0 / lam, False, 1e-7, res)
            out.update({f"{name}_in": shots, f"{name}_out": res, f"{name}_a": np.float64(a),
                        f"{name}_b": np.float64(b), f"{name}_pin": np.int64(pin),
                        f"{name}_pinval": pv, f"{name}_lam": np.float64(lam)})
            names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "projection_nonfinite.npz"), **out)


def host_fixtures():
    out = {}
    for n_c, n_s, d in ((8, 33, 2), (16, 32, 3), (4096, 4, 3), (1, 9, 2)):
        out[f"init_{n_c}_{n_s}_{d}"] = om.init_radial(n_c, n_s, d).coords
    base = om.init_radial(16, 64, 3)
    out["perturb_3d_s7"] = om.perturb(base, 0.5, 7).coords
    out["perturb_2d_s0"] = om.perturb(om.init_radial(64, 512, 2), 0.25, 0).coords
    rng = np.random.default_rng(5)
    c = rng.uniform(-0.9, 0.9, (3, 16, 3))
    out["ups_in"] = c
    out["ups_out"] = om.upsample_shots(core.SamplingPattern(c)).coords
    hw = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                           dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                           dims=3)
    lim = core.normalized_limits(hw)
    out["lim_full3d"] = np.array([lim.alpha, lim.beta])
    out["dens_2d_16"] = density.discretize(density.DensityParams(0.25, 2.0), 16, 2).grid
    out["dens_3d_6"] = density.discretize(density.DensityParams(0.3, 1.0), 6, 3).grid
    dk = rng.normal(size=40)
    dg = rng.normal(size=40)
    out["bb_dk"] = dk
    out["bb_dg"] = dg
    out["bb_eta"] = np.float64(om.step_size(25, 0.5, dk, dg, 0.01, 20))
    # SPKT bytes written by the reference (format kept byte-identical)
    import tempfile
    from vdtraj import io as vio
    pat = core.SamplingPattern(rng.uniform(-1, 1, (3, 7, 3)))
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.spkt")
        vio.write_spkt(path, pat, (834.78, 834.78, 833.33), 1e-5)
        out["spkt_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        vio.write_spkd(os.path.join(tmp, "d.spkd"), out["dens_2d_16"])
        out["spkd_bytes"] = np.frombuffer(open(os.path.join(tmp, "d.spkd"), "rb").read(),
                                          dtype=np.uint8)
    out["spkt_coords"] = pat.coords
    np.savez_compressed(os.path.join(OUT, "host.npz"), **out)


def optimize_fixture():
    """A tiny stock ``optimize`` run (2D, direct backend) for end-to-end drift checks."""
    hw = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                           dwell_dt=1e-5, fov=0.192, matrix=32, dims=2)
    out = {}
    for mode in ("consistent", "smooth"):
        cfg = om.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=1, n_git=6, n_pit=100,
                                 perturbation=0.25, seed=3, grad_mode=mode,
                                 repulsion=om.RepulsionConfig(backend="direct"))
        res = om.optimize(cfg, hw)
        out[f"{mode}_coords"] = res.pattern.coords
        out[f"{mode}_costs"] = res.trace.costs()
        out[f"{mode}_steps"] = np.array([r.step for r in res.trace.records])
        out[f"{mode}_att"] = np.array([r.attraction for r in res.trace.records])
        out[f"{mode}_rep"] = np.array([r.repulsion for r in res.trace.records])
        out[f"{mode}_feas"] = np.array([r.feas_residual for r in res.trace.records])
        out["field_potential"] = res.field.potential
        out["field_force"] = res.field.force
        out["field_eps"] = np.float64(res.field.kernel_eps)
    cfg = om.OptimizerConfig(n_c=4, n_s=32, dims=2, n_decim=0, n_git=0, perturbation=0.2,
                             seed=5, repulsion=om.RepulsionConfig(backend="direct"))
    res = om.optimize(cfg, core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6,
                                             raster_dt=1e-5, dwell_dt=1e-5, fov=0.192,
                                             matrix=64, dims=2))
    out["ngit0_coords"] = res.pattern.coords
    out["ngit0_initial"] = res.initial.coords
    np.savez_compressed(os.path.join(OUT, "optimize.npz"), **out)


# ---------------------------------------------------------------------------- trajectories
# End-to-end trajectories of the reference's own ``optimize`` (optimizer.py:239-349) at
# BASELINE configs[0] (C1: 2D, 64 shots x 512 samples, 257^2 density grid) and on a reduced
# 3D multi-resolution schedule, for tests/test_gpu_trajectory.py.  Each case also records
# the reference's OWN sensitivity: the same run with 1e-6 relative noise injected into its
# repulsion gradient (the size of the fp32 pair-sum error of the GPU kernels), three noise
# seeds; the test bounds the GPU drift against that.

sys.path.insert(0, os.path.dirname(OUT))
import trajectory_cases as _tc  # noqa: E402  (the case table, shared with the GPU tests)

TRAJ_CASES = _tc.CASES
TRAJ_NOISE = _tc.NOISE
TRAJ_NOISE_SEEDS = _tc.NOISE_SEEDS


def _run_reference(cfg_kw, hw_kw, patched_exact, noise_seed=None):
    """One reference optimize; returns (per-level final coords, trace arrays)."""
    from vdtraj import repulsion as rp

    repo = os.path.dirname(os.path.dirname(OUT))
    sys.path.insert(0, repo)
    from oracle import oracle as orc

    hw = core.HardwareSpec(**_tc.hardware_kwargs(hw_kw))
    cfg = om.OptimizerConfig(repulsion=om.RepulsionConfig(backend="direct"), **cfg_kw)
    levels = []
    saved = (om.eval_attraction, om.eval_repulsion, om.upsample_shots)

    def capture_upsample(k):
        levels.append(k.coords.copy())
        return saved[2](k)

    om.upsample_shots = capture_upsample
    if patched_exact:
        def exact_attraction(k, fld, grad_mode="consistent"):
            cost, grad = orc.attraction_exact(k.points(), fld_holder["rho"].grid,
                                              fld.kernel_eps)
            n_out = int(np.count_nonzero((np.abs(k.points()) > 1.0).any(axis=1)))
            return at.AttractionResult(cost=cost, grad=grad, n_clamped=n_out)
        om.eval_attraction = exact_attraction
    if noise_seed is not None:
        rng = np.random.default_rng(noise_seed)

        def noisy(k, c):
            cost, g = rp.eval_repulsion(k, c)
            return (cost * (1 + 0.1 * TRAJ_NOISE * rng.standard_normal()),
                    g * (1 + TRAJ_NOISE * rng.standard_normal(g.shape)))
        om.eval_repulsion = noisy
    fld_holder = {}
    try:
        rho = density.discretize(cfg.density, cfg.grid_n, cfg.dims)
        fld_holder["rho"] = rho
        res = om.optimize(cfg, hw, rho=rho)
    finally:
        om.eval_attraction, om.eval_repulsion, om.upsample_shots = saved
    levels.append(res.pattern.coords.copy())
    recs = res.trace.records
    trace = {k: np.array([getattr(r, k) for r in recs])
             for k in ("level", "cost", "attraction", "repulsion", "step", "feas_residual")}
    return levels, trace


def trajectory_fixtures():
    out = {}
    for name, (cfg_kw, hw_kw, patched) in TRAJ_CASES.items():
        t0 = time.perf_counter()
        levels, trace = _run_reference(cfg_kw, hw_kw, patched)
        for li, c in enumerate(levels):
            out[f"{name}_level{li}"] = c
        for k, v in trace.items():
            out[f"{name}_{k}"] = v
        # the reference's own drift under 1e-6 relative repulsion-gradient noise
        nd = np.zeros((len(TRAJ_NOISE_SEEDS), len(levels)))
        nl2 = np.zeros_like(nd)
        ncost = np.zeros(len(TRAJ_NOISE_SEEDS))
        for si, s in enumerate(TRAJ_NOISE_SEEDS):
            nlev, ntr = _run_reference(cfg_kw, hw_kw, patched, noise_seed=s)
            for li, (a, b) in enumerate(zip(nlev, levels)):
                nd[si, li] = np.abs(a - b).max()
                nl2[si, li] = np.linalg.norm(a - b) / np.linalg.norm(b)
            ncost[si] = np.abs(ntr["cost"] - trace["cost"]).max() / np.abs(trace["cost"]).max()
        out[f"{name}_noise_max"] = nd.max(axis=0)
        out[f"{name}_noise_rel_l2"] = nl2.max(axis=0)
        out[f"{name}_noise_cost_rel"] = np.float64(ncost.max())
        print(f"{name}: {time.perf_counter() - t0:.1f} s; noise drift per level "
              f"{nd.max(axis=0)}, cost {ncost.max():.2e}", flush=True)
    out["names"] = np.array(list(TRAJ_CASES))
    out["noise"] = np.float64(TRAJ_NOISE)
    np.savez_compressed(os.path.join(OUT, "trajectory.npz"), **out)


def analysis_fixtures():
    """NUDFT adjoint / forward, density compensation, PSF + metrics, dwell resampling and
    density compliance (analysis.py, core.py:286-311)."""
    from vdtraj import analysis as an

    rng = np.random.default_rng(424242)
    out = {}
    # raw NUDFT
    for name, (p, grid) in {"a2": (200, (16, 13)), "a3": (150, (8, 7, 10))}.items():
        pts = rng.uniform(-1, 1, (p, len(grid)))
        w = rng.normal(size=p) + 1j * rng.normal(size=p)
        img = rng.normal(size=grid) + 1j * rng.normal(size=grid)
        out[f"{name}_pts"] = pts
        out[f"{name}_grid"] = np.array(grid)
        out[f"{name}_w"] = w
        out[f"{name}_adj"] = an.nudft_adjoint(pts, w, grid)
        out[f"{name}_img"] = img
        out[f"{name}_fwd"] = an.nudft_forward(pts, img)
    # density compensation and PSF on SPARKLING-like patterns
    hw2 = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=2e-6, fov=0.192, matrix=32, dims=2)
    k2 = om.perturb(om.init_radial(8, 32, 2), 0.25, 0)
    k3 = om.perturb(om.init_radial(4, 16, 3), 0.25, 0)
    out["dcf2_coords"] = k2.coords
    out["dcf2"] = an.density_compensation(k2, (16, 16), iters=3)
    out["dcf3_coords"] = k3.coords
    out["dcf3"] = an.density_compensation(k3, (8, 8, 8), iters=2)
    psf2 = an.compute_psf(k2, (32, 32), weights=out["dcf2"])
    out["psf2"] = psf2.values
    out["psf2_peak"] = np.array(psf2.peak_index)
    psf2h = an.compute_psf(k2, (24, 24), hw=hw2)
    out["psf2h"] = psf2h.values
    psf3 = an.compute_psf(k3, (12, 12, 12))
    out["psf3"] = psf3.values
    for name, psf in (("psf2", psf2), ("psf2h", psf2h), ("psf3", psf3)):
        m = an.psf_metrics(psf)
        out[f"{name}_metrics"] = np.array(list(m.fwhm) + [m.psl_db, m.pnl_db,
                                                          float(m.fwhm_bounded)])
    # the acceptance-test PSF leg (test_acceptance.py:310-317): radial 64 x 128 3D init,
    # 10 density-compensation iterations on 32^3 -- an ill-conditioned fixed point that
    # pins the NUDFT's fp64 accuracy end to end
    kr = om.init_radial(64, 128, 3)
    out["dcfr3"] = an.density_compensation(kr, (32, 32, 32), iters=10)
    mr = an.psf_metrics(an.compute_psf(kr, (32, 32, 32), out["dcfr3"]))
    out["dcfr3_metrics"] = np.array(list(mr.fwhm) + [mr.psl_db, mr.pnl_db,
                                                     float(mr.fwhm_bounded)])
    # a smooth synthetic PSF (Gaussian) for the FWHM interpolation
    ax = np.arange(33) - 16
    g = np.exp(-0.5 * (ax[:, None] ** 2 + ax[None, :] ** 2) / 2.0 ** 2)
    gv = an.PsfVolume(values=g, peak_index=(16, 16), peak_value=1.0)
    mg = an.psf_metrics(gv)
    out["gauss"] = g
    out["gauss_metrics"] = np.array(list(mg.fwhm) + [mg.psl_db, mg.pnl_db,
                                                      float(mg.fwhm_bounded)])
    # dwell resampling (ratio 5) and density compliance
    out["dwell_in"] = k2.coords
    out["dwell_out"] = core.resample_to_dwell(k2, hw2).coords
    rho = density.discretize(density.DensityParams(0.25, 2.0), 16, 2)
    l1, hs, hr = an.density_compliance(k2, rho, bins=8)
    out["compl_l1"] = np.float64(l1)
    out["compl_hs"] = hs
    out["compl_hr"] = hr
    # waveform export of a projected (feasible) and of a raw pattern
    hw3 = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                            dims=3)
    for name, kk in (("wf3", k3), ("wf2", k2)):
        hw = hw3 if kk.dims == 3 else hw2
        g, sl, rep = core.kspace_to_waveforms(kk, hw)
        out[f"{name}_in"] = kk.coords
        out[f"{name}_g"] = g
        out[f"{name}_s"] = sl
        out[f"{name}_rep"] = np.array([rep.max_grad, rep.max_slew, rep.grad_saturation_fraction,
                                       rep.slew_saturation_fraction, float(rep.feasible)])
        out[f"{name}_back"] = core.integrate_waveforms(kk.coords[:, 0, :], g, hw)
    np.savez_compressed(os.path.join(OUT, "analysis.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["repulsion", "attraction", "projection", "host", "optimize",
                             "analysis", "trajectory", "nonfinite"]
    if "repulsion" in which:
        repulsion_fixtures()
    if "attraction" in which:
        attraction_fixtures()
    if "projection" in which:
        projection_fixtures()
    if "host" in which:
        host_fixtures()
    if "optimize" in which:
        optimize_fixture()
    if "analysis" in which:
        analysis_fixtures()
    if "trajectory" in which:
        trajectory_fixtures()
    if "nonfinite" in which:
        nonfinite_fixtures()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
