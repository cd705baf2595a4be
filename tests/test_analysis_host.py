"""Analysis path, CPU side: the numpy NUDFT oracle pinned against the reference's own
outputs (tests/golden/analysis.npz), and the host-side metrics / resampling / binning of
paper_2108_02991_b200.analysis against the same fixtures."""

import numpy as np

import paper_2108_02991_b200 as spk
from oracle import nudft_oracle as no
from paper_2108_02991_b200 import analysis as an
from spk_golden import golden


def test_oracle_nudft_pinned():
    g = golden("analysis")
    for name in ("a2", "a3"):
        grid = tuple(int(x) for x in g[f"{name}_grid"])
        adj = no.nudft_adjoint(g[f"{name}_pts"], g[f"{name}_w"], grid)
        ref = g[f"{name}_adj"]
        assert np.abs(adj - ref).max() <= 1e-12 * np.abs(ref).max()
        fwd = no.nudft_forward(g[f"{name}_pts"], g[f"{name}_img"])
        ref = g[f"{name}_fwd"]
        assert np.abs(fwd - ref).max() <= 1e-12 * np.abs(ref).max()


def test_oracle_dcf_and_psf_pinned():
    g = golden("analysis")
    k2 = g["dcf2_coords"].reshape(-1, 2)
    assert np.allclose(no.density_compensation(k2, (16, 16), 3), g["dcf2"], rtol=1e-10)
    k3 = g["dcf3_coords"].reshape(-1, 3)
    assert np.allclose(no.density_compensation(k3, (8, 8, 8), 2), g["dcf3"], rtol=1e-10)
    assert np.allclose(no.psf_values(k2, (32, 32), g["dcf2"]), g["psf2"], rtol=1e-10,
                       atol=1e-14)
    assert np.allclose(no.psf_values(k3, (12, 12, 12)), g["psf3"], rtol=1e-10, atol=1e-14)


def _metrics_vec(m):
    return np.array(list(m.fwhm) + [m.psl_db, m.pnl_db, float(m.fwhm_bounded)])


def test_psf_metrics_match_reference():
    g = golden("analysis")
    for name in ("psf2", "psf2h", "psf3", "gauss"):
        vals = g[name]
        peak = tuple(int(i) for i in np.unravel_index(int(np.argmax(vals)), vals.shape))
        psf = an.PsfVolume(values=vals, peak_index=peak, peak_value=float(vals[peak]))
        got = _metrics_vec(an.psf_metrics(psf))
        assert np.array_equal(got, g[f"{name}_metrics"]), (name, got, g[f"{name}_metrics"])


def test_resample_to_dwell_bitwise():
    g = golden("analysis")
    hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                          dwell_dt=2e-6, fov=0.192, matrix=32, dims=2)
    out = spk.resample_to_dwell(spk.SamplingPattern(g["dwell_in"]), hw)
    assert np.array_equal(out.coords, g["dwell_out"])


def test_density_compliance_bitwise():
    g = golden("analysis")
    rho = spk.discretize(spk.DensityParams(0.25, 2.0), 16, 2)
    l1, hs, hr = spk.density_compliance(spk.SamplingPattern(g["dcf2_coords"]), rho, bins=8)
    assert l1 == float(g["compl_l1"])
    assert np.array_equal(hs, g["compl_hs"]) and np.array_equal(hr, g["compl_hr"])


def test_budget_guard_and_validation():
    import pytest

    k = spk.SamplingPattern(np.zeros((1, 4, 2)))
    with pytest.raises(ValueError, match="budget"):
        an.nudft_adjoint(np.zeros((1 << 20, 2)), np.ones(1 << 20), (2048, 2048))
    with pytest.raises(ValueError, match="iters"):
        spk.density_compensation(k, (8, 8), iters=0)
    with pytest.raises(ValueError, match="bins"):
        spk.density_compliance(k, spk.discretize(spk.DensityParams(0.25, 2.0), 4, 2), bins=3)
    psf = an.PsfVolume(values=np.zeros((4, 4)), peak_index=(0, 0), peak_value=0.0)
    with pytest.raises(ValueError, match="peak"):
        spk.psf_metrics(psf)


def test_waveform_export_bitwise():
    g = golden("analysis")
    hw3 = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                           dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208),
                           dims=3)
    hw2 = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                           dwell_dt=2e-6, fov=0.192, matrix=32, dims=2)
    for name, hw in (("wf3", hw3), ("wf2", hw2)):
        k = spk.SamplingPattern(g[f"{name}_in"])
        gr, sl, rep = spk.kspace_to_waveforms(k, hw)
        assert np.array_equal(gr, g[f"{name}_g"]) and np.array_equal(sl, g[f"{name}_s"])
        got = np.array([rep.max_grad, rep.max_slew, rep.grad_saturation_fraction,
                        rep.slew_saturation_fraction, float(rep.feasible)])
        assert np.array_equal(got, g[f"{name}_rep"])
        back = spk.integrate_waveforms(k.coords[:, 0, :], gr, hw)
        assert np.array_equal(back, g[f"{name}_back"])
