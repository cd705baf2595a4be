"""Where the time goes for the treecode attraction at small target counts (level 0 of
the full3d schedule: 131k targets against the 385x385x209 lattice)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402
from paper_2108_02991_b200.attraction import tree_grid_sums_device  # noqa: E402

rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
fld = spk.precompute_field(rho)
src = fld.source_tree()
src.static_proxies(5)
for n_s in (32, 128, 512, 2048):
    k = spk.perturb(spk.init_radial(4096, n_s, 3), 0.75, 0)
    pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(k.points())))
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tg = tree.TargetGroups(pos4, 3)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st = {"timing": True}
        tree.tree_eval(tg, src, 5, 0.8, fld.kernel_eps ** 2, static=True, stats=st)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    print(f"n_s={n_s} p={pos4.shape[0]} groups={tg.n_groups} targets_sort+groups={1e3*(t1-t0):.1f} ms "
          f"plan+eval={1e3*(t2-t1):.1f} ms pairs/target={st['pairs']/pos4.shape[0]:.0f} segs={st['segments']} "
          + " ".join(f"{k}={v:.1f}" for k, v in st["eval_phases_ms"].items()),
          flush=True)
