"""The optimizer loop (schedule, guards, Barzilai-Borwein step, sharded engine) on the
CPU oracle ops against the REFERENCE's own optimize at BASELINE configs[0] (C1, 2D 64 x
512, 30 iterations incl. 10 BB steps) with its attraction monkeypatched to the fp64
exact sum (tests/golden/trajectory.npz, case c1_exact).  The oracle ops sum fp32-rounded
positions like the kernels, so the trajectory drifts by the reference's own sensitivity
to a ~1e-7..1e-6 relative gradient perturbation; it is bounded by the same multiple of
the fixture's recorded noise drift as the GPU test."""
import numpy as np

from spk_golden import golden
import trajectory_cases as tc
from test_gpu_trajectory import K_COORDS, K_COST


def test_c1_exact_loop_on_oracle_ops_vs_reference():
    import paper_2108_02991_b200 as spk
    from cpu_ops import OracleOps

    g = golden("trajectory")
    levels, trace = tc.run_ours(spk, "c1_exact", ops=OracleOps())
    rep = tc.drift_report(g, "c1_exact", levels, trace)
    print("[trajectory host]", rep)
    assert np.array_equal(trace["level"], g["c1_exact_level"])
    assert rep["final_feas"] <= 1e-6
    for row in rep["levels"]:
        assert row["max"] <= K_COORDS * row["ref_noise_max"], row
    assert rep["cost_rel"] <= K_COST * rep["ref_noise_cost_rel"], rep
