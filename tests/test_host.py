"""Host-side mirror of the reference API (no GPU): types, validation, schedules, the
operator-norm power iteration and file formats, bit-identical to the reference's own
outputs (tests/golden/host.npz, projection.npz, optimize.npz)."""

import numpy as np
import pytest

import paper_2108_02991_b200 as spk
from paper_2108_02991_b200 import io as spk_io
from paper_2108_02991_b200.optimizer import _bb_step
from paper_2108_02991_b200.projection import stacked_operator_norm
from spk_golden import golden


@pytest.fixture(scope="module")
def host():
    return golden("host")


def test_init_radial_bitwise(host):
    for key in host.files:
        if key.startswith("init_"):
            _, n_c, n_s, d = key.split("_")
            pat = spk.init_radial(int(n_c), int(n_s), int(d))
            assert np.array_equal(pat.coords, host[key]), key


def test_perturb_bitwise(host):
    assert np.array_equal(spk.perturb(spk.init_radial(16, 64, 3), 0.5, 7).coords,
                          host["perturb_3d_s7"])
    assert np.array_equal(spk.perturb(spk.init_radial(64, 512, 2), 0.25, 0).coords,
                          host["perturb_2d_s0"])


def test_upsample_bitwise(host):
    out = spk.upsample_shots(spk.SamplingPattern(host["ups_in"]))
    assert np.array_equal(out.coords, host["ups_out"])


def test_limits_and_density_bitwise(host):
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                          dims=3)
    lim = spk.normalized_limits(hw)
    assert np.array_equal(np.array([lim.alpha, lim.beta]), host["lim_full3d"])
    g2 = spk.discretize(spk.DensityParams(0.25, 2.0), 16, 2).grid
    assert np.array_equal(g2, host["dens_2d_16"])
    g3 = spk.discretize(spk.DensityParams(0.3, 1.0), 6, 3).grid
    assert np.array_equal(g3, host["dens_3d_6"])


def test_step_size(host):
    eta = spk.step_size(25, 0.5, host["bb_dk"], host["bb_dg"], 0.01, 20)
    assert eta == float(host["bb_eta"])
    # reference tests/test_optimizer.py:99-129
    assert spk.step_size(1, 0.5, None, None, eta0=2.0, fixed_step_iters=20) == 2.0
    assert spk.step_size(20, 0.5, np.ones(4), np.ones(4), eta0=2.0, fixed_step_iters=20) == 2.0
    assert spk.step_size(25, 1.0, np.array([1.0]), np.array([1e-9]), 1.0, 20) == 1e3
    assert spk.step_size(25, 0.37, np.array([1.0]), np.array([0.0]), 1.0, 20) == 0.37
    rng = np.random.default_rng(0)
    x0 = rng.normal(size=8)
    g0 = 7.0 * x0
    x1 = x0 - 0.01 * g0
    assert spk.step_size(21, 0.01, x1 - x0, 7.0 * x1 - g0, 0.1, 20) == pytest.approx(1 / 7.0,
                                                                                      rel=1e-12)
    assert _bb_step(25, 0.37, 5.0, 0.0, True, 1.0, 20) == 0.37
    assert _bb_step(3, 0.37, 5.0, 1.0, True, 1.0, 20) == 1.0


def test_operator_norm_bitwise():
    proj = golden("projection")
    for (n, p), lam in zip(proj["lam_keys"], proj["lam_vals"]):
        assert stacked_operator_norm(int(n), int(p)) == float(lam), (n, p)


def test_validation_messages():
    with pytest.raises(ValueError, match="divisible"):
        spk.OptimizerConfig(n_c=4, n_s=30, dims=2, n_decim=2)
    with pytest.raises(ValueError, match="square"):
        spk.OptimizerConfig(n_c=10, n_s=32, dims=3)
    with pytest.raises(ValueError):
        spk.OptimizerConfig(n_c=4, n_s=32, dims=2, perturbation=1.5)
    with pytest.raises(ValueError):
        spk.OptimizerConfig(n_c=4, n_s=32, dims=2, grad_mode="bogus")
    with pytest.raises(ValueError):
        spk.RepulsionConfig(backend="gpu")  # reference tests/test_repulsion.py:154
    with pytest.raises(ValueError):
        spk.RepulsionConfig(leaf_size=4)
    with pytest.raises(ValueError):
        spk.ProjectionConfig(alpha=1.0, beta=1.0, raster_dt=1.0, n_pit=0)
    with pytest.raises(ValueError, match="Omega"):
        spk.LinearConstraint(pinned_index=0, pinned_value=np.array([1.5, 0.0]))
    with pytest.raises(ValueError):
        spk.SamplingPattern(np.full((1, 2, 2), np.nan))
    with pytest.raises(ValueError):
        spk.HardwareSpec(g_max=0.04, s_max=180, gamma=42e6, raster_dt=1e-5, dwell_dt=3e-6,
                         fov=0.2, matrix=64, dims=2)
    with pytest.raises(MemoryError, match="grid"):
        spk.precompute_field(spk.TargetDensity(np.ones((9, 9, 9)), 4), kernel_eps=0.1,
                             mem_cap_bytes=1024)
    cfg = spk.OptimizerConfig(n_c=4096, n_s=2048, dims=3, n_decim=6, n_git=100, n_pit=100,
                              perturbation=0.75)
    assert cfg.resolved_pin() == 1024
    assert spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2), 10, 2)).kernel_eps \
        == pytest.approx(1 / 20)


def test_spkt_spkd_roundtrip(tmp_path):
    rng = np.random.default_rng(2)
    pat = spk.SamplingPattern(rng.uniform(-1, 1, (3, 5, 3)))
    path = tmp_path / "t.spkt"
    spk_io.write_spkt(path, pat, (100.0, 100.0, 80.0), 1e-5)
    raw = path.read_bytes()
    assert raw[:4] == b"SPKT" and len(raw) == 17 + 3 * 8 + 8 + 3 * 5 * 3 * 4
    back, hdr = spk_io.read_spkt(path)
    assert np.array_equal(back.coords, pat.coords.astype(np.float32).astype(np.float64))
    assert hdr.k_max == (100.0, 100.0, 80.0) and hdr.raster_dt == 1e-5
    path.write_bytes(raw[:-1])
    with pytest.raises(spk_io.FileFormatError, match="offset"):
        spk_io.read_spkt(path)
    grid = rng.uniform(0, 1, (5, 5))
    spk_io.write_spkd(tmp_path / "d.spkd", grid)
    assert np.array_equal(spk_io.read_spkd(tmp_path / "d.spkd"), grid)


def test_trace_csv(tmp_path):
    tr = spk.RunTrace()
    tr.append(spk.TraceRecord(0, 1, 32, 1.0, 2.0, 1.0, 0.5, 0.0, 0.1))
    tr.write_csv(tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0].startswith("level,iteration") and len(lines) == 2


def test_spkt_spkd_bytes_identical_to_reference(host, tmp_path):
    pat = spk.SamplingPattern(host["spkt_coords"])
    spk_io.write_spkt(tmp_path / "t.spkt", pat, (834.78, 834.78, 833.33), 1e-5)
    assert (tmp_path / "t.spkt").read_bytes() == host["spkt_bytes"].tobytes()
    spk_io.write_spkd(tmp_path / "d.spkd", host["dens_2d_16"])
    assert (tmp_path / "d.spkd").read_bytes() == host["spkd_bytes"].tobytes()


def test_trajectory_csv_roundtrip_and_dispatch(tmp_path):
    """io.py:96-126,162-169: CSV header, 9-digit round trip, SPKT/CSV dispatch, errors."""
    rng = np.random.default_rng(5)
    for dims in (2, 3):
        coords = rng.uniform(-1, 1, (3, 16, dims))
        pat = spk.SamplingPattern(coords)
        csv = tmp_path / f"t{dims}.csv"
        spk_io.write_trajectory_csv(csv, pat)
        assert csv.read_text().splitlines()[0] == "shot,sample," + ",".join("kx ky kz".split()[:dims])
        assert np.allclose(spk_io.read_trajectory_csv(csv).coords, coords, rtol=1e-8, atol=1e-9)
        spkt = tmp_path / f"t{dims}.spkt"
        spk_io.write_spkt(spkt, pat, (100.0,) * dims, 1e-5)
        assert np.allclose(spk_io.load_trajectory(spkt).coords, coords, atol=1e-7)
        assert np.allclose(spk_io.load_trajectory(csv).coords, coords, atol=1e-8)
    # rows in any order
    lines = (tmp_path / "t2.csv").read_text().splitlines()
    (tmp_path / "r.csv").write_text("\n".join([lines[0]] + lines[1:][::-1]) + "\n")
    assert np.array_equal(spk_io.read_trajectory_csv(tmp_path / "r.csv").coords,
                          spk_io.read_trajectory_csv(tmp_path / "t2.csv").coords)
    (tmp_path / "e.csv").write_text("shot,sample,kx,ky\n")
    with pytest.raises(spk_io.FileFormatError, match="empty"):
        spk_io.read_trajectory_csv(tmp_path / "e.csv")
    (tmp_path / "m.csv").write_text("\n".join(lines[:-1]) + "\n")
    with pytest.raises(spk_io.FileFormatError, match="rows"):
        spk_io.read_trajectory_csv(tmp_path / "m.csv")
    (tmp_path / "c.csv").write_text("shot,sample,kx\n0,0,0.5\n")
    with pytest.raises(spk_io.FileFormatError, match="columns"):
        spk_io.read_trajectory_csv(tmp_path / "c.csv")


def test_default_density_grid_guard():
    """full3d.cfg's cubic default (grid_n = 2 * 384 -> 1537^3 cells, 29 GB) raises a
    MemoryError with guidance before allocating (the reference would run out of host
    memory); no GPU is touched before the check."""
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                          dims=3)
    cfg = spk.OptimizerConfig(n_c=4096, n_s=2048, dims=3, n_decim=6, grad_mode="exact")
    with pytest.raises(MemoryError, match="discretize_anisotropic"):
        spk.optimize(cfg, hw)
