"""One adjoint + one forward NUDFT launch at the C2 pattern / 64^3 grid (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, analysis as an  # noqa: E402

k = spk.perturb(spk.init_radial(1024, 1024, 3), 0.25, 0)
pts = _device.h2d(np.ascontiguousarray(k.points()))
w = torch.zeros((pts.shape[0], 2), dtype=torch.float64, device=pts.device)
w[:, 0] = 1.0
img = an.nudft_adjoint_device(pts, w, (64, 64, 64))
an.nudft_forward_device(pts, img, (64, 64, 64))
torch.cuda.synchronize()
print("ok")
