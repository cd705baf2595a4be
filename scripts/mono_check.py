"""Cost trace of the reference's fixed-phase monotonicity instance (test_optimizer.py:202)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402

hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=1e-5,
                      fov=0.192, matrix=64, dims=2)
cfg = spk.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=0, n_git=20, n_pit=400,
                          perturbation=0.25, seed=3,
                          repulsion=spk.RepulsionConfig(backend="direct"))
res = spk.optimize(cfg, hw)
c = res.trace.costs()
np.set_printoptions(precision=3)
print("costs", c)
print("diffs", np.diff(c))
print("steps", [r.step for r in res.trace.records])
