"""K3 projection kernels vs the reference's golden vectors: BIT-IDENTICAL.

tau is taken from the fixture (the reference's lambda) so that the comparison does not
depend on the host BLAS used for the power iteration on the GPU box."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from spk_golden import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


@pytest.fixture(scope="module")
def proj():
    return golden("projection")


def cfg_of(spk, proj, name):
    a, b = float(proj[f"{name}_a"]), float(proj[f"{name}_b"])
    pin = int(proj[f"{name}_pin"])
    pc = None if pin < 0 else spk.LinearConstraint(pin, proj[f"{name}_pinval"])
    # raster_dt = 1 so that speed_bound == a and accel_bound == b exactly
    cfg = spk.ProjectionConfig(alpha=a, beta=b, raster_dt=1.0, n_pit=int(proj[f"{name}_npit"]),
                               pin=pc, monotone=bool(proj[f"{name}_mono"]))
    return cfg, 1.0 / float(proj[f"{name}_lam"])


def run(spk, shots, cfg, tau, trace=False, max_sweeps=50000):
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.projection import project_device

    dev = _device.h2d(shots)
    tr = None
    if trace:
        tr = torch.empty(shots.shape[0] * cfg.n_pit, dtype=torch.float64, device=dev.device)
    sweeps = torch.empty(shots.shape[0], dtype=torch.int32, device=dev.device)
    out = project_device(dev, cfg, tau=tau, trace=tr, sweeps=sweeps, max_sweeps=max_sweeps)
    return (_device.d2h(out), None if tr is None else _device.d2h(tr), _device.d2h(sweeps))


def test_bounds_roundtrip(spk, proj):
    # speed_bound/accel_bound with raster_dt=1 reproduce the fixture's a, b exactly
    for name in proj["names"]:
        cfg, _ = cfg_of(spk, proj, name)
        assert cfg.speed_bound == float(proj[f"{name}_a"])
        assert cfg.accel_bound == float(proj[f"{name}_b"])


def test_project_all_bitwise(spk, proj):
    for name in proj["names"]:
        cfg, tau = cfg_of(spk, proj, name)
        out, _, _ = run(spk, proj[f"{name}_in"], cfg, tau)
        ref = proj[f"{name}_out"]
        assert np.array_equal(out, ref), (name, np.abs(out - ref).max())


def test_trace_bitwise(spk, proj):
    for name in ("mono2d", "trace3d"):
        cfg, tau = cfg_of(spk, proj, name)
        out, tr, _ = run(spk, proj[f"{name}_in"], cfg, tau, trace=True)
        assert np.array_equal(tr, proj[f"{name}_trace"]), name
        assert np.array_equal(out, proj[f"{name}_out"]), name


def test_polish_sweeps_and_cap(spk, proj):
    """Wavefront polish reproduces the sequential stopping sweep and the max_sweeps cap."""
    name = "inloop3d"
    cfg, tau = cfg_of(spk, proj, name)
    shots = proj[f"{name}_in"]
    _, ref_sweeps = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound,
                                    cfg.pin.pinned_index, np.zeros(3), cfg.n_pit, tau,
                                    0.1 * cfg.feas_tol)
    out, _, sweeps = run(spk, shots, cfg, tau)
    assert np.array_equal(sweeps, ref_sweeps)
    assert np.array_equal(out, proj[f"{name}_out"])
    for cap in (1, 31, 32, 33, 37):
        ref_c, _ = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound,
                                   cfg.pin.pinned_index, np.zeros(3), cfg.n_pit, tau,
                                   0.1 * cfg.feas_tol, max_sweeps=cap)
        out_c, _, sw = run(spk, shots, cfg, tau, max_sweeps=cap)
        assert np.all(sw == cap)
        assert np.array_equal(out_c, ref_c), cap


def test_random_cases_vs_oracle(spk):
    rng = np.random.default_rng(99)
    for d in (2, 3):
        for ns, pin in ((5, 2), (64, -1), (300, 150), (1024, 512)):
            shots = rng.uniform(-1.3, 1.3, (3, ns, d))
            pc = None if pin < 0 else spk.LinearConstraint(pin, np.full(d, 0.05))
            cfg = spk.ProjectionConfig(alpha=0.05, beta=0.01, raster_dt=1.0, n_pit=50, pin=pc)
            tau = 1.0 / spk.projection.stacked_operator_norm(ns, pin)
            out, _, sw = run(spk, shots, cfg, tau)
            ref, rsw = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, pin,
                                       np.full(d, 0.05), 50, tau, 0.1 * cfg.feas_tol)
            assert np.array_equal(sw, rsw), (d, ns)
            assert np.array_equal(out, ref), (d, ns, np.abs(out - ref).max())


def test_nonfinite_samples_match_reference(spk):
    """Shots holding NaN / +-inf samples through the K3 kernels: outputs equal the
    reference's _project_all (NaN positions included) and the sweep counts the oracle's."""
    nf = golden("projection_nonfinite")
    for name in nf["names"]:
        shots = nf[f"{name}_in"]
        d, pin = shots.shape[2], int(nf[f"{name}_pin"])
        pc = None if pin < 0 else spk.LinearConstraint(pin, nf[f"{name}_pinval"])
        cfg = spk.ProjectionConfig(alpha=float(nf[f"{name}_a"]), beta=float(nf[f"{name}_b"]),
                                   raster_dt=1.0, n_pit=50, pin=pc)
        tau = 1.0 / float(nf[f"{name}_lam"])
        out, _, sw = run(spk, shots, cfg, tau)
        assert np.array_equal(out, nf[f"{name}_out"], equal_nan=True), name
        _, rsw = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, pin,
                                 nf[f"{name}_pinval"] if pin >= 0 else np.zeros(d), 50, tau,
                                 0.1 * cfg.feas_tol)
        assert np.array_equal(sw, rsw), name


def test_public_api(spk, proj):
    rng = np.random.default_rng(4)
    cfg = spk.ProjectionConfig(alpha=10216.0, beta=4.6e7, raster_dt=1e-5, n_pit=80)
    shot = rng.uniform(-1.1, 1.1, (32, 2))
    single = spk.project_shot(shot, cfg)
    pat = spk.project_pattern(spk.SamplingPattern(shot[None]), cfg)
    assert np.array_equal(pat.coords[0], single)
    coords = rng.uniform(-1.1, 1.1, (6, 24, 2))
    out = spk.project_pattern(spk.SamplingPattern(coords), cfg)
    perm = rng.permutation(6)
    out_p = spk.project_pattern(spk.SamplingPattern(coords[perm]), cfg)
    assert np.array_equal(out_p.coords, out.coords[perm])
    pin = spk.LinearConstraint(pinned_index=4, pinned_value=np.array([0.1, -0.2]))
    c2 = spk.ProjectionConfig(alpha=0.4, beta=0.2, raster_dt=1.0, n_pit=200, pin=pin)
    o = spk.project_shot(rng.uniform(-1, 1, (9, 2)), c2)
    assert np.array_equal(o[4], pin.pinned_value)
    with pytest.raises(ValueError):
        spk.project_shot(rng.uniform(-1, 1, (3, 2)), c2)  # pin out of range


def test_feasibility_residuals(spk, proj):
    name = "inloop3d"
    cfg, _ = cfg_of(spk, proj, name)
    res = spk.feasibility_residuals(spk.SamplingPattern(proj[f"{name}_in"]), cfg)
    ref = proj["feas_inloop3d_in"]
    got = np.array([res["amplitude"], res["speed"], res["acceleration"], res["pin"],
                    res["max"]])
    assert np.array_equal(got, ref)


def test_upsample_device_bitwise(spk):
    from paper_2108_02991_b200 import _device
    from paper_2108_02991_b200.engine import CudaOps

    h = golden("host")
    out = CudaOps().upsample(_device.h2d(h["ups_in"]))
    assert np.array_equal(_device.d2h(out), h["ups_out"])


def test_very_long_shot_global_fallbacks(spk):
    """N_s = 12000 (3D): FISTA state and the polish wrap buffer exceed shared memory and
    fall back to the workspace; ring capped at 32 warps.  Still bit-identical."""
    rng = np.random.default_rng(21)
    ns = 12000
    shots = np.cumsum(rng.normal(0, 3e-3, (2, ns, 3)), axis=1)
    shots -= shots[:, ns // 2:ns // 2 + 1, :]
    pin = spk.LinearConstraint(ns // 2, np.zeros(3))
    cfg = spk.ProjectionConfig(alpha=2.0e-3, beta=3.0e-4, raster_dt=1.0, n_pit=30, pin=pin)
    tau = 1.0 / spk.projection.stacked_operator_norm(ns, ns // 2)
    for cap in (3, 200):
        out, _, sw = run(spk, shots, cfg, tau, max_sweeps=cap)
        ref, rsw = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, ns // 2,
                                   np.zeros(3), 30, tau, 0.1 * cfg.feas_tol, max_sweeps=cap)
        assert np.array_equal(sw, rsw)
        assert np.array_equal(out, ref), np.abs(out - ref).max()


@pytest.mark.parametrize("d,ns,pin,mono,cap", [
    (3, 1500, 700, False, 3000),   # 12-warp ring (<1024,1> instantiation)
    (2, 2100, -1, False, 2000),    # 17 warps, unpinned 2D
    (3, 5000, 2500, False, 300),   # single shared wrap buffer + global snapshots
    (2, 700, 350, True, 5000),     # monotone FISTA + 6-warp ring
    (3, 3, 1, False, 50),          # smallest pinned shot
])
def test_ring_configurations_vs_oracle(spk, d, ns, pin, mono, cap):
    """Bit-identity across the ring's instantiations and wrap-buffer modes (sweep caps
    bound the oracle's run time; the cap path and the stop/replay path are both hit)."""
    rng = np.random.default_rng(ns + d)
    shots = np.cumsum(rng.normal(0, 6e-3, (2, ns, d)), axis=1)
    shots = np.clip(shots - shots.mean(axis=1, keepdims=True), -1.05, 1.05)
    pv = np.zeros(d)
    pc = None if pin < 0 else spk.LinearConstraint(pin, pv)
    cfg = spk.ProjectionConfig(alpha=4e-3, beta=8e-4, raster_dt=1.0, n_pit=40, pin=pc,
                               monotone=mono)
    tau = 1.0 / spk.projection.stacked_operator_norm(ns, pin)
    out, _, sw = run(spk, shots, cfg, tau, max_sweeps=cap)
    ref, rsw = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, pin, pv, 40, tau,
                               0.1 * cfg.feas_tol, monotone=mono, max_sweeps=cap)
    assert np.array_equal(sw, rsw), (sw, rsw)
    assert np.array_equal(out, ref), np.abs(out - ref).max()



@pytest.mark.parametrize("d,ns", [(3, 256), (2, 100), (3, 1030)])
def test_fista_then_polish_subsets_equal_project_all(spk, d, ns):
    """spk_project_fista + spk_polish_shots on shuffled disjoint shot lists, launched on
    two streams, equal spk_project_all bit for bit (outputs, positions, sweep counts) --
    the building blocks of the multi-GPU overlap schedule."""
    from paper_2108_02991_b200 import _device, _native
    from paper_2108_02991_b200.projection import _pin_arrays, project_device, stacked_operator_norm

    rng = np.random.default_rng(ns + d)
    n = 11
    shots = rng.uniform(-1.1, 1.1, (n, ns, d)) * np.linspace(0.2, 1.0, ns)[None, :, None]
    cfg = spk.ProjectionConfig(alpha=0.05, beta=0.004, raster_dt=1.0, n_pit=80,
                               pin=spk.LinearConstraint(ns // 2, np.zeros(d)))
    dev = _device.h2d(shots)
    ref = torch.empty_like(dev)
    ref4 = torch.empty((n * ns, 4), dtype=torch.float32, device=dev.device)
    ref_sw = torch.empty(n, dtype=torch.int32, device=dev.device)
    project_device(dev, cfg, out=ref, pos4=ref4, sweeps=ref_sw)
    pin_idx, pin_val = _pin_arrays(cfg, d)
    pv = _native.f64_array(list(pin_val) + [0.0] * (3 - d))
    tau = 1.0 / stacked_operator_norm(ns, pin_idx)
    ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, ns, d, 0), "t_split")
    out = torch.empty_like(dev)
    pos4 = torch.empty_like(ref4)
    sw = torch.empty_like(ref_sw)
    _native.call("spk_project_fista", dev.data_ptr(), None, 0.0, None, out.data_ptr(), n, ns, d,
                 cfg.speed_bound, cfg.accel_bound, pin_idx, pv, cfg.n_pit, tau, 0, None, None,
                 ws.data_ptr(), ws.numel(), _device.stream())
    perm = torch.tensor(rng.permutation(n), dtype=torch.int32, device=dev.device)
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(main)
    for ids, st in ((perm[:5], main), (perm[5:], side)):
        _native.call("spk_polish_shots", out.data_ptr(), ids.data_ptr(), ids.numel(), n, ns, d,
                     cfg.speed_bound, cfg.accel_bound, pin_idx, pv, 0.1 * cfg.feas_tol,
                     50000, pos4.data_ptr(), sw.data_ptr(), None, None, 0, 0, ws.data_ptr(),
                     ws.numel(), st.cuda_stream)
    main.wait_stream(side)
    assert torch.equal(out, ref) and torch.equal(pos4, ref4) and torch.equal(sw, ref_sw)
    # argument errors are reported, not executed
    with pytest.raises(ValueError):
        _native.call("spk_polish_shots", out.data_ptr(), perm.data_ptr(), n + 1, n, ns, d,
                     cfg.speed_bound, cfg.accel_bound, pin_idx, pv, 1e-7, 50000, None, None,
                     None, None, 0, 0, ws.data_ptr(), ws.numel(), _device.stream())


def test_grid_sums_on_shot_subset(spk):
    """spk_grid_sums_shots fills exactly the rows of the listed shots with the lattice
    sums (fp32 pair math: <= 1e-4 relative l2 of the gradient vs the fp64 oracle, like
    spk_grid_sums) and leaves the other rows untouched."""
    from paper_2108_02991_b200 import _device, _native

    rng = np.random.default_rng(5)
    n, ns, d = 9, 300, 3
    pts = rng.uniform(-1, 1, (n * ns, d))
    rho = spk.discretize(spk.DensityParams(0.25, 2.0), 10, d)
    fld = spk.precompute_field(rho)
    pos4 = _device.pack_positions(_device.h2d(pts))
    ids = torch.tensor([7, 2, 4], dtype=torch.int32, device=pos4.device)
    val = torch.full((n * ns,), -7.0, dtype=torch.float64, device=pos4.device)
    grad = torch.full((n * ns, d), -7.0, dtype=torch.float64, device=pos4.device)
    w = fld.device_sources()
    nb = _native.query("spk_grid_sums_shots_workspace_bytes", 3, ns, int(np.prod(fld.sides)))
    ws = _device.workspace(nb, "t_gs")
    _native.call("spk_grid_sums_shots", pos4.data_ptr(), ids.data_ptr(), 3, ns, w.data_ptr(),
                 _native.i64_array(fld.sides), d, float(fld.kernel_eps ** 2), val.data_ptr(),
                 grad.data_ptr(), None, ws.data_ptr(), ws.numel(), _device.stream())
    v, g = _device.d2h(val), _device.d2h(grad)
    rows = np.concatenate([np.arange(s * ns, (s + 1) * ns) for s in (7, 2, 4)])
    other = np.setdiff1d(np.arange(n * ns), rows)
    assert np.all(v[other] == -7.0) and np.all(g[other] == -7.0)
    vo, go = orc.grid_sums(pts[rows], rho.grid, fld.kernel_eps ** 2)
    assert np.linalg.norm(g[rows] - go) <= 1e-4 * np.linalg.norm(go)
    assert np.abs(v[rows] - vo).max() <= 1e-5 * np.abs(vo).max()
