"""tree_sums_checked (the optimizer's repulsion call) at C4, far level on/off via env."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.repulsion import tree_sums_checked  # noqa: E402

n_s = int(os.environ.get("NS", "2048"))
pts = spk.perturb(spk.init_radial(4096, n_s, 3), 0.75, 0).points()
pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(pts)))
cfg = spk.RepulsionConfig(backend="tree", tree_precision=float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3)
best = 1e30
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree_sums_checked(pos4, pos4, 3, cfg)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"p={pts.shape[0]} far_min={os.environ.get('SPK_FAR_LEVEL_MIN', 'default')} precision={cfg.tree_precision}: {best*1e3:.1f} ms", flush=True)
