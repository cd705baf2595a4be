"""Random sweep of the lattice treecode (attraction) vs exact K2: dims, lattice size,
density, target cloud kind, precision row."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.attraction import grid_sums_device, tree_grid_sums_device  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

rng = np.random.default_rng(777)
worst, fails = {}, []
for trial in range(120):
    dims = int(rng.choice([2, 3]))
    n = int(rng.choice([64, 128, 256])) if dims == 2 else int(rng.choice([16, 32, 48]))
    kind = str(rng.choice(["uniform", "radial", "clustered", "duplicates"]))
    prec = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-5]))
    cutoff, decay = float(rng.choice([0.1, 0.25, 0.5])), float(rng.choice([0.0, 2.0, 4.0]))
    p = int(rng.choice([50_000, 200_000]))
    fld = spk.precompute_field(spk.discretize(spk.DensityParams(cutoff, decay), n, dims))
    pts = np.clip(_cloud(dims, p, kind, int(rng.integers(0, 2**31 - 1))), -1, 1)
    p4 = _device.pack_positions(_device.h2d(pts))
    eps2 = fld.kernel_eps ** 2
    v0, g0 = (_device.d2h(x) for x in grid_sums_device(p4, fld, eps2))
    v1, g1 = (_device.d2h(x) for x in tree_grid_sums_device(p4, fld, eps2, prec))
    eg = np.linalg.norm(g1 - g0) / np.linalg.norm(g0)
    ec = abs(v1.sum() - v0.sum()) / abs(v0.sum())
    key = (dims, kind, prec)
    worst[key] = max(worst.get(key, 0.0), max(eg, ec) / prec)
    if eg > prec or ec > prec:
        fails.append((dims, n, kind, prec, cutoff, decay, p, eg, ec))
print("fails", len(fails))
for f in fails[:10]:
    print(f)
for k, v in sorted(worst.items()):
    print(k, f"worst err/prec {v:.2f}")
