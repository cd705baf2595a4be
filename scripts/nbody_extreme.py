"""K1 / K2 on extreme parameters vs the fp64 oracle: eps from 0 to 10, coordinates up to
1e3, tiny and duplicated clouds (gradient rel l2 <= 1e-4, value <= 1e-5)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.repulsion import direct_sums_device  # noqa: E402
from oracle import oracle as orc  # noqa: E402

rng = np.random.default_rng(9)
bad = 0
n = 0
for dims in (2, 3):
    for eps in (0.0, 1e-20, 1e-6, 1e-3, 1.0, 10.0):
        for scale in (1e-6, 1.0, 1e3):
            for p in (1, 2, 777):
                pts = rng.uniform(-scale, scale, (p, dims))
                p4 = _device.pack_positions(_device.h2d(pts))
                v, g = (_device.d2h(x) for x in direct_sums_device(p4, p4, dims, eps * eps))
                vr, gr = orc.direct_sums(pts.astype(np.float32).astype(np.float64), eps * eps)
                ev = np.linalg.norm(v - vr) / max(np.linalg.norm(vr), 1e-300)
                gn = np.linalg.norm(gr)
                eg = np.linalg.norm(g - gr) / gn if gn > 0 else np.abs(g).max()
                n += 1
                # eps < 1.1e-19 has no fp32 square: coincident pairs then add 0 instead of eps
                ok = np.all(np.isfinite(v)) and np.all(np.isfinite(g)) and (
                    ev <= 1e-5 or np.abs(v - vr).max() <= 1e-18) and (
                    eg <= 1e-4 or (gn == 0 and eg == 0))
                if not ok:
                    bad += 1
                    print("MISS", dims, eps, scale, p, ev, eg, flush=True)
print(f"extreme K1 cases: {n - bad}/{n} within tolerance")
