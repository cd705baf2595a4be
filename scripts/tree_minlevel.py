"""Treecode attraction at the full3d coarse levels vs the target octree's minimum split
level (TargetGroups(min_level=...)), for a rank's share of the targets (the first
`shots` shots): device time of one evaluation (groups + lists + eval), CUDA events."""
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
for n_s in (32, 128, 512):
    k = spk.perturb(spk.init_radial(4096, n_s, 3), 0.75, 0)
    full = _device.pack_positions(_device.h2d(np.ascontiguousarray(k.points())))
    for shots in (4096, 1024, 512):
        pos4 = full[:shots * n_s]
        for ml in (2, 3, 4, 5, 6):
            best = 1e30
            for rep in range(3):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                tg = tree.TargetGroups(pos4, 3, min_level=ml)
                tree.tree_eval(tg, src, 5, 0.7, fld.kernel_eps ** 2, static=True, far=False)
                e.record()
                torch.cuda.synchronize()
                best = min(best, s.elapsed_time(e))
            print(f"n_s={n_s} targets={pos4.shape[0]} min_level={ml} groups={tg.n_groups} "
                  f"{best:.1f} ms", flush=True)
