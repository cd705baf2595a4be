"""2D treecode calibration for the tight precision rows: gradient / cost error of
(order, theta) on dense-centre radial clouds, uniform clouds and a 2D spoke pattern,
against the exact K1 sums (fp32 pairs, ~3e-8 from fp64 here)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.repulsion import direct_sums_device  # noqa: E402
from paper_2108_02991_b200.tree import tree_sums_device  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

clouds = {
    "radial150k": _cloud(2, 150_000, "radial", 0),
    "radial1M": _cloud(2, 1 << 20, "radial", 1),
    "uniform1M": _cloud(2, 1 << 20, "uniform", 2),
    "clustered300k": _cloud(2, 300_000, "clustered", 3),
    "spokes512x512": spk.perturb(spk.init_radial(512, 512, 2), 0.25, 0).points().copy(),
}
for name, pts in clouds.items():
    p4 = _device.pack_positions(_device.h2d(pts))
    v0, g0 = direct_sums_device(p4, p4, 2, 1e-6)
    v0, g0 = _device.d2h(v0), _device.d2h(g0)
    for order, theta in ((5, 0.7), (6, 0.7), (6, 0.6), (7, 0.7), (7, 0.6), (8, 0.7), (8, 0.6), (6, 0.5)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v, g = tree_sums_device(p4, p4, 2, 1e-6, order, theta)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        v, g = _device.d2h(v), _device.d2h(g)
        print(json.dumps({"cloud": name, "order": order, "theta": theta,
                          "err_cost": abs(v.sum() - v0.sum()) / abs(v0.sum()),
                          "err_grad": float(np.linalg.norm(g - g0) / np.linalg.norm(g0)),
                          "t_s": dt}), flush=True)
