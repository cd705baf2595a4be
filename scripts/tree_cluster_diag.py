"""Diagnose the clustered-cloud treecode miss (profiles/r01_tree_fuzz_sweep.txt): error vs
(order, theta) on the failing case, against the exact kernel."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.repulsion import direct_sums_device  # noqa: E402
from paper_2108_02991_b200.tree import tree_sums_device  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

pts = _cloud(3, 140_000, "clustered", 679326770)
print("cloud extent", pts.min(0), pts.max(0))
p4 = _device.pack_positions(_device.h2d(pts))
v0, g0 = (_device.d2h(x) for x in direct_sums_device(p4, p4, 3, 1e-6))
for order, theta in ((4, 0.7), (4, 0.5), (4, 0.3), (6, 0.7), (8, 0.7), (8, 0.3), (4, 0.0)):
    v, g = (_device.d2h(x) for x in tree_sums_device(p4, p4, 3, 1e-6, order, theta))
    err = np.linalg.norm(g - g0, axis=1)
    worst = np.argsort(err)[-3:]
    print(f"q={order} theta={theta}: grad rel {np.linalg.norm(g-g0)/np.linalg.norm(g0):.2e} "
          f"cost {abs(v.sum()-v0.sum())/abs(v0.sum()):.2e}; worst points {worst} err "
          f"{err[worst]} |g0| {np.linalg.norm(g0[worst], axis=1)}", flush=True)
