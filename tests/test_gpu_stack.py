"""Stack-of-SPARKLING (BASELINE configs[2]): independent problems as one device batch."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


def hw2(spk, matrix=32):
    return spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=1e-5, fov=0.192, matrix=matrix, dims=2)


@pytest.mark.parametrize("mode", ["exact", "smooth"])
def test_stack_matches_individual_runs(spk, mode, monkeypatch):
    """Each problem of the batch follows the single-problem optimize() (the batched N-body
    only changes the fp64 summation order of partial slots, ~1e-16).  Both sides on the
    fused N-body schedule (SPK_OVERLAP=0; the overlap schedule is compared below)."""
    monkeypatch.setenv("SPK_OVERLAP", "0")
    cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=1, n_git=4, perturbation=0.25,
                              seed=11, grad_mode=mode)
    hw = hw2(spk)
    batch = spk.optimize_stack(cfg, hw, 3)
    for q, res in enumerate(batch):
        single = spk.optimize(spk.OptimizerConfig(**{**cfg.__dict__, "seed": 11 + q}), hw)
        assert np.array_equal(res.initial.coords, single.initial.coords)
        c1, c2 = res.trace.costs(), single.trace.costs()
        assert np.abs(c1 - c2).max() <= 1e-9 * np.abs(c2).max(), (q, c1, c2)
        assert np.abs(res.pattern.coords - single.pattern.coords).max() <= 1e-6


def test_stack_c3_shape(spk):
    """C3: 64 independent 2D problems of 64 shots x 512 samples on a 257^2 grid."""
    cfg = spk.OptimizerConfig(n_c=64, n_s=512, dims=2, n_decim=0, n_git=2, grad_mode="exact",
                              grid_n=128, perturbation=0.25, seed=0)
    res = spk.optimize_stack(cfg, hw2(spk, 64), 64)
    assert len(res) == 64
    for r in res:
        assert r.pattern.coords.shape == (64, 512, 2)
        assert np.all(np.isfinite(r.trace.costs())) and len(r.trace.records) == 2
        assert r.trace.records[-1].feas_residual <= 1e-6
    # distinct seeds -> distinct patterns
    assert not np.array_equal(res[0].pattern.coords, res[1].pattern.coords)


def test_stack_k2_under_polish_matches_fused(spk, monkeypatch):
    """The stack with each polish group's lattice sums under the slower shots' polish and
    the batched K1 alone (forced with SPK_OVERLAP=1) follows the fused-launch stack: the
    projection is bit-identical per shot, K2's fp32 partial sums are chunked differently
    (~1e-7), so costs agree to 1e-6 and patterns to far less than the reference's own noise
    drift."""
    cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=1, n_git=5, perturbation=0.25,
                              seed=11, grad_mode="exact")
    hw = hw2(spk)
    monkeypatch.setenv("SPK_OVERLAP", "0")
    fused = spk.optimize_stack(cfg, hw, 4)
    monkeypatch.setenv("SPK_OVERLAP", "1")
    ovl = spk.optimize_stack(cfg, hw, 4)
    for a, b in zip(ovl, fused):
        ca, cb = a.trace.costs(), b.trace.costs()
        assert np.abs(ca - cb).max() <= 1e-6 * np.abs(cb).max()
        assert np.abs(a.pattern.coords - b.pattern.coords).max() <= 1e-5
