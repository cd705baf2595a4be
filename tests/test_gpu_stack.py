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
def test_stack_matches_individual_runs(spk, mode):
    """Each problem of the batch follows the single-problem optimize() (the batched N-body
    only changes the fp64 summation order of partial slots, ~1e-16)."""
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
