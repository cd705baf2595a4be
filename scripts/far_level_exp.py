"""Far level (P2L/L2P on parents) vs the plain treecode: accuracy vs exact sums and time,
repulsion (C2, C4 positions) and lattice attraction (C2, C4)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402
from paper_2108_02991_b200.attraction import grid_sums_device  # noqa: E402
from paper_2108_02991_b200.repulsion import direct_sums_device  # noqa: E402


def timed(fn, reps=3):
    out = fn()
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return out, best


def err(a, b):
    va, ga = (_device.d2h(x) for x in a)
    vb, gb = b
    return abs(va.sum() - vb.sum()) / abs(vb.sum()), np.linalg.norm(ga - gb) / np.linalg.norm(gb)


cases = [("C2", 1024, 1024, (64, 64, 64), 0.25)]
if len(sys.argv) > 1 and sys.argv[1] == "c4":
    cases.append(("C4", 4096, 2048, (192, 192, 104), 0.75))
for name, n_c, n_s, grid, pert in cases:
    pts = spk.perturb(spk.init_radial(n_c, n_s, 3), pert, 0).points()
    pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(pts)))
    ref = [_device.d2h(x) for x in direct_sums_device(pos4, pos4, 3, 1e-6)]
    params = spk.DensityParams(0.25, 2.0)
    rho = (spk.discretize(params, grid[0], 3) if len(set(grid)) == 1 else
           spk.discretize_anisotropic(params, grid, 3))
    fld = spk.precompute_field(rho)
    eps2a = fld.kernel_eps ** 2
    refa = [_device.d2h(x) for x in grid_sums_device(pos4, fld, eps2a)]
    lat = fld.source_tree()
    for order, theta in ((4, 0.7), (5, 0.7)):
        src = tree.SourceTree(pos4, 3)
        lat.static_proxies(order)
        src.static_proxies(order)
        tg0 = tree.TargetGroups(pos4, 3, same_as=src)
        r0, t0 = timed(lambda: tree.tree_eval(tg0, src, order, theta, 1e-6, static=True))
        tga = tree.TargetGroups(pos4, 3)
        a0, ta0 = timed(lambda: tree.tree_eval(tga, lat, order, theta, eps2a, static=True))
        print(f"{name} q{order} th{theta} plain: rep {t0*1e3:.1f} ms err {err(r0, ref)} | "
              f"att {ta0*1e3:.1f} ms err {err(a0, refa)}", flush=True)
        for cap in (512, 1024, 2048):
            for fo in (order, order + 1):
                tgf = tree.TargetGroups(pos4, 3, same_as=src, parent_cap=cap)
                r1, t1 = timed(lambda: tree.tree_eval(tgf, src, order, theta, 1e-6, static=True,
                                                      far_order=fo))
                tgfa = tree.TargetGroups(pos4, 3, parent_cap=cap)
                a1, ta1 = timed(lambda: tree.tree_eval(tgfa, lat, order, theta, eps2a,
                                                       static=True, far_order=fo))
                print(f"   far cap {cap} qt {fo}: rep {t1*1e3:.1f} ms err {err(r1, ref)} | "
                      f"att {ta1*1e3:.1f} ms err {err(a1, refa)}", flush=True)
