"""fp32 pair-arithmetic floor of the exact K1 kernel vs the fp64 oracle on the fuzz
clouds (clustered points at 1e-3 scale ~ eps cancel in dx = t - s)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

for dims in (2, 3):
    for kind in ("uniform", "radial", "clustered", "duplicates"):
        pts = _cloud(dims, 60_000, kind, 0)
        c0, g0 = orc.repulsion(pts, 1e-3)
        cd, gd = spk.eval_repulsion_direct(pts, 1e-3)
        ct, gt = spk.eval_repulsion_tree(pts, spk.RepulsionConfig(backend="tree", tree_precision=1e-6))
        print(f"dims={dims} {kind:10s} direct-vs-fp64 grad {np.linalg.norm(gd-g0)/np.linalg.norm(g0):.2e} "
              f"cost {abs(cd-c0)/c0:.2e}; tree1e-6-vs-fp64 grad {np.linalg.norm(gt-g0)/np.linalg.norm(g0):.2e}", flush=True)
