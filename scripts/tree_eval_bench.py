"""Device time of the treecode evaluation kernels at C2 / C4 (repulsion 1e-3 lists and
attraction 1e-4 lists), CUDA events around tree_eval only (lists prebuilt per call)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402


def timed(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


for name, n_c, n_s, grid, pert in (("C2", 1024, 1024, (64, 64, 64), 0.25),
                                   ("C4", 4096, 2048, (192, 192, 104), 0.75)):
    pts = spk.perturb(spk.init_radial(n_c, n_s, 3), pert, 0).points()
    pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(pts)))
    src = tree.SourceTree(pos4, 3)
    tg = tree.TargetGroups(pos4, 3, same_as=src)
    t_rep = timed(lambda: tree.tree_eval(tg, src, 4, 0.7, 1e-6))
    params = spk.DensityParams(0.25, 2.0)
    rho = (spk.discretize(params, grid[0], 3) if len(set(grid)) == 1 else
           spk.discretize_anisotropic(params, grid, 3))
    fld = spk.precompute_field(rho)
    lat = fld.source_tree()
    lat.static_proxies(5)
    tga = tree.TargetGroups(pos4, 3)
    t_att = timed(lambda: tree.tree_eval(tga, lat, 5, 0.7, fld.kernel_eps ** 2, static=True))
    print(f"{name}: repulsion tree_eval (q4, 0.7) {t_rep:.1f} ms, attraction tree_eval "
          f"(q5, 0.7, static) {t_att:.1f} ms", flush=True)
