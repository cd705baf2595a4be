"""End-to-end trajectory cases shared by tests/golden/make_golden.py (which runs the
REFERENCE's optimize on them, /root/reference/pkg/src/vdtraj/optimizer.py:239-349) and
tests/test_gpu_trajectory.py / scripts/trajectory_drift.py (which run this package's
optimize on the B200 and compare).

C1 is BASELINE configs[0] (2D, 64 shots x 512 samples, 257^2 density grid); ml3d is a
reduced full3d multi-resolution schedule (64 shots, N_s 32 -> 256 over 4 levels, full3d
hardware limits).  ``patched``: the reference runs with om.eval_attraction monkeypatched to
the fp64 exact density-weighted sum (SURVEY 8c drift attribution); this package runs
grad_mode="exact".
"""

import numpy as np

C1_HW = dict(fov=0.192, matrix=64, dwell_dt=2e-6, dims=2)
FULL3D_HW = dict(fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dwell_dt=2e-6, dims=3)
C1 = dict(n_c=64, n_s=512, dims=2, n_decim=0, n_git=30, grid_n=128, seed=0,
          perturbation=0.25)
ML3D = dict(n_c=64, n_s=256, dims=3, n_decim=3, n_git=12, grid_n=24, seed=0,
            perturbation=0.75)

# name: (OptimizerConfig kwargs, HardwareSpec kwargs, patched exact attraction?)
CASES = {
    "c1_consistent": (dict(C1, grad_mode="consistent"), C1_HW, False),
    "c1_smooth": (dict(C1, grad_mode="smooth"), C1_HW, False),
    "c1_exact": (dict(C1, grad_mode="smooth"), C1_HW, True),
    "ml3d_smooth": (dict(ML3D, grad_mode="smooth"), FULL3D_HW, False),
    "ml3d_consistent": (dict(ML3D, grad_mode="consistent"), FULL3D_HW, False),
    "ml3d_exact": (dict(ML3D, grad_mode="smooth"), FULL3D_HW, True),
}
NOISE = 1e-6               # relative noise injected into the reference's repulsion gradient
NOISE_SEEDS = (11, 12, 13)


def hardware_kwargs(hw_kw):
    return dict(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, **hw_kw)


def run_ours(spk, name, ops=None):
    """This package's optimize on case ``name``: per-level final coords (the pattern
    before each upsample, then the final one) and the trace arrays.  ``ops``: the device
    operations (default: the sm_100a kernels; tests/cpu_ops.OracleOps on the CPU)."""
    from paper_2108_02991_b200 import optimizer as om

    cfg_kw, hw_kw, patched = CASES[name]
    if patched:
        cfg_kw = dict(cfg_kw, grad_mode="exact")
    cfg = spk.OptimizerConfig(repulsion=spk.RepulsionConfig(backend="direct"), **cfg_kw)
    hw = spk.HardwareSpec(**hardware_kwargs(hw_kw))
    state = om.start(cfg, hw, ops=ops)
    levels = []
    while True:
        rec = om.step(state)
        if rec is None:
            break
        if state.it == cfg.n_git:
            levels.append(state.run.gather_coords())
    recs = state.trace.records
    trace = {k: np.array([getattr(r, k) for r in recs])
             for k in ("level", "cost", "attraction", "repulsion", "step", "feas_residual")}
    return levels, trace


def drift_report(g, name, levels, trace):
    """Per-level coordinate drift (max, relative l2) and trace drift vs the reference
    fixture, next to the reference's own drift under NOISE (same fields)."""
    rows = []
    for li, c in enumerate(levels):
        ref = g[f"{name}_level{li}"]
        rows.append({"level": li, "n_s": int(ref.shape[1]),
                     "max": float(np.abs(c - ref).max()),
                     "rel_l2": float(np.linalg.norm(c - ref) / np.linalg.norm(ref)),
                     "ref_noise_max": float(g[f"{name}_noise_max"][li]),
                     "ref_noise_rel_l2": float(g[f"{name}_noise_rel_l2"][li])})
    rc = g[f"{name}_cost"]
    return {"case": name, "levels": rows,
            "cost_rel": float(np.abs(trace["cost"] - rc).max() / np.abs(rc).max()),
            "ref_noise_cost_rel": float(g[f"{name}_noise_cost_rel"]),
            "step_rel": float(np.abs(trace["step"] - g[f"{name}_step"]).max()
                              / np.abs(g[f"{name}_step"]).max()),
            "final_feas": float(trace["feas_residual"][-1]),
            "ref_final_feas": float(g[f"{name}_feas_residual"][-1])}
