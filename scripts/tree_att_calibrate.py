"""Treecode attraction calibration: the density lattice as a static weighted source tree
vs the exact lattice kernel K2 (grid_sums_device), relative error of the cost and of the
gradient l2 norm per precision row, and times (tree build once + per-call)."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402
from paper_2108_02991_b200.attraction import grid_sums_device  # noqa: E402

CASES = {
    "c1": (64, 512, 2, (128, 128), 0.25),
    "c2": (1024, 1024, 3, (64, 64, 64), 0.25),
    "c4": (4096, 2048, 3, (192, 192, 104), 0.75),
}


def sync_time(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2")
    ap.add_argument("--pairs", default="3:0.8,4:0.8,5:0.8,6:0.7,6:0.5")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lines = []
    for name in a.cases.split(","):
        n_c, n_s, d, grid, pert = CASES[name]
        pts = spk.perturb(spk.init_radial(n_c, n_s, d), pert, 0).points()
        params = spk.DensityParams(0.25, 2.0)
        rho = (spk.discretize(params, grid[0], d) if len(set(grid)) == 1 else
               spk.discretize_anisotropic(params, grid, d))
        fld = spk.precompute_field(rho)
        eps2 = fld.kernel_eps ** 2
        pos4 = _device.pack_positions(_device.h2d(pts))
        (vd, gd), t_exact = sync_time(lambda: grid_sums_device(pos4, fld, eps2))
        vd, gd = _device.d2h(vd), _device.d2h(gd)
        _, t_build = sync_time(lambda: fld.source_tree())
        for pr in a.pairs.split(","):
            order, theta = int(pr.split(":")[0]), float(pr.split(":")[1])
            src = fld.source_tree()
            _, t_prox = sync_time(lambda: src.static_proxies(order))
            best = 1e30
            for _ in range(3):
                (vt, gt), t = sync_time(lambda: tree.tree_eval(
                    tree.TargetGroups(pos4, d), src, order, theta, eps2, static=True))
                best = min(best, t)
            st = {}
            tree.tree_eval(tree.TargetGroups(pos4, d), src, order, theta, eps2, static=True,
                           stats=st)
            vt, gt = _device.d2h(vt), _device.d2h(gt)
            rec = dict(case=name, p=pts.shape[0], cells=int(np.prod(fld.sides)), order=order,
                       theta=theta,
                       err_cost=abs(vt.sum() - vd.sum()) / abs(vd.sum()),
                       err_grad=np.linalg.norm(gt - gd) / np.linalg.norm(gd),
                       t_tree_s=best, t_exact_s=t_exact, speedup=t_exact / best,
                       t_lattice_tree_build_s=t_build, t_static_proxies_s=t_prox,
                       pairs_per_target=st["pairs"] / pts.shape[0],
                       near_fraction=st["near_pairs"] / max(st["pairs"], 1),
                       **{k: v for k, v in st.items() if k not in ("interp_order", "opening_theta")})
            print(json.dumps(rec), flush=True)
            lines.append(rec)
    if a.out:
        with open(a.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
