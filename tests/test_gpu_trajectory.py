"""End-to-end trajectories vs the REFERENCE's own optimize (tests/golden/trajectory.npz,
made by tests/golden/make_golden.py from /root/reference/pkg/src/vdtraj/optimizer.py:
239-349) at BASELINE configs[0] (C1: 2D 64 x 512, 257^2 grid, 30 iterations incl. 10
Barzilai-Borwein steps) in consistent / smooth / exact mode, and on a reduced full3d
multi-resolution schedule (3D, 64 shots, N_s 32 -> 256 over 4 levels).

The GPU sums pairs in fp32 (relative gradient error ~1e-6); the projection, field
interpolation, step and upsampling are bit-identical.  The trajectories therefore drift
by the reference's own sensitivity to a 1e-6 relative perturbation of the gradient: the
fixture holds the reference's drift under exactly that noise (3 seeds, per level), and the
test bounds this package's per-level drift by a fixed multiple of it.  The "exact" case
runs the reference with om.eval_attraction monkeypatched to the fp64 exact sum (SURVEY 8c
drift attribution): both sides then evaluate the same smooth objective.
"""

import json
import os

import numpy as np
import pytest

from spk_golden import golden
import trajectory_cases as tc

pytestmark = pytest.mark.gpu

# drift <= K x the reference's own drift under 1e-6 noise (max over 3 seeds), per level.
# The GPU's perturbation is of the same size (fp32 pair sums, ~1e-6 relative) but not the
# same distribution (it is correlated across iterations, where the injected noise is
# not), so a small multiple is allowed.
K_COORDS = 3.0
K_COST = 3.0


@pytest.fixture(scope="module")
def spk():
    import paper_2108_02991_b200 as m

    return m


@pytest.mark.parametrize("name", list(tc.CASES))
def test_trajectory_vs_reference(spk, name):
    g = golden("trajectory")
    levels, trace = tc.run_ours(spk, name)
    assert len(levels) == len(g[f"{name}_noise_max"])
    rep = tc.drift_report(g, name, levels, trace)
    print("[trajectory]", json.dumps(rep))
    out = os.environ.get("SPK_DRIFT_REPORT")
    if out:
        with open(out, "a") as fh:
            fh.write(json.dumps(rep) + "\n")
    # same schedule, same iteration count, feasible like the reference
    assert np.array_equal(trace["level"], g[f"{name}_level"])
    assert rep["final_feas"] <= 1e-6
    for row in rep["levels"]:
        assert row["max"] <= K_COORDS * max(row["ref_noise_max"], 1e-9), row
    assert rep["cost_rel"] <= K_COST * max(rep["ref_noise_cost_rel"], 1e-9), rep
