"""One treecode repulsion evaluation at the C2 size (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402

pts = spk.perturb(spk.init_radial(1024, 1024, 3), 0.25, 0).points()
pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(pts)))
for _ in range(2):
    v, g = tree.tree_sums_device(pos4, pos4, 3, 1e-6, 4, 0.7)
torch.cuda.synchronize()
print("ok", float(v.sum()))
