"""Treecode attraction at the full3d coarse levels vs the target octree's minimum split
level (TargetGroups(min_level=...)): device time of one evaluation, CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402

rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
fld = spk.precompute_field(rho)
src = fld.source_tree()
src.static_proxies(5)
for n_s in (32, 64, 128, 256):
    k = spk.perturb(spk.init_radial(4096, n_s, 3), 0.75, 0)
    pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(k.points())))
    for ml in (4, 5, 6, 7):
        best = 1e30
        for rep in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tg = tree.TargetGroups(pos4, 3, min_level=ml)
            tree.tree_eval(tg, src, 5, 0.7, fld.kernel_eps ** 2, static=True, far=False)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        print(f"n_s={n_s} p={pos4.shape[0]} min_level={ml} groups={tg.n_groups} {best:.1f} ms",
              flush=True)
