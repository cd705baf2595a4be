"""Tree precision on the 2D radial fuzz cloud (tests/test_gpu_fuzz.py): tree and GPU
direct both against the fp64 oracle, per precision row."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

for dims in (2, 3):
    pts = _cloud(dims, 150_000, "radial", 0)
    c0, g0 = orc.repulsion(pts, 1e-3)
    cd, gd = spk.eval_repulsion_direct(pts, 1e-3)
    print(f"dims={dims} direct(fp32) vs oracle: cost {abs(cd-c0)/c0:.2e} grad {np.linalg.norm(gd-g0)/np.linalg.norm(g0):.2e}", flush=True)
    for prec in (1e-3, 1e-4, 1e-5, 1e-6):
        ct, gt = spk.eval_repulsion_tree(pts, spk.RepulsionConfig(backend="tree", tree_precision=prec))
        print(f"  prec {prec:g}: tree vs oracle cost {abs(ct-c0)/c0:.2e} grad {np.linalg.norm(gt-g0)/np.linalg.norm(g0):.2e}; vs direct grad {np.linalg.norm(gt-gd)/np.linalg.norm(gd):.2e}", flush=True)
