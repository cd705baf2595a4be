"""Treecode calibration: relative error of the cost and of the gradient l2 norm (the
reference's tree_precision contract, repulsion.py:165-171) vs the exact K1 kernel, and
time, over (order, theta) on SPARKLING-shaped clouds.  One JSON line per case."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402
from paper_2108_02991_b200.repulsion import direct_sums_device  # noqa: E402


def clouds(which):
    if which == "c2":
        return spk.perturb(spk.init_radial(1024, 1024, 3), 0.25, 0).points()
    if which == "c1":
        return spk.perturb(spk.init_radial(64, 512, 2), 0.25, 0).points()
    if which == "c4":
        return spk.perturb(spk.init_radial(4096, 2048, 3), 0.75, 0).points()
    if which == "u3":
        return np.random.default_rng(0).uniform(-1, 1, (1 << 20, 3))
    if which == "u2":
        return np.random.default_rng(0).uniform(-1, 1, (1 << 17, 2))
    if which == "s3":  # small radial 3D
        return spk.perturb(spk.init_radial(64, 1024, 3), 0.25, 0).points()
    raise KeyError(which)


def timed(fn, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    out = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record()
        out = fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return out, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clouds", default="c1,s3,c2,u3")
    ap.add_argument("--orders", default="3,4,5,6,7")
    ap.add_argument("--thetas", default="0.3,0.4,0.5,0.6")
    ap.add_argument("--out", default=None)
    ap.add_argument("--leaf", type=int, default=tree.LEAF_CAP)
    ap.add_argument("--pairs", default=None, help="explicit order:theta list, e.g. 4:0.8,5:0.8")
    a = ap.parse_args()
    lines = []
    for cname in a.clouds.split(","):
        pts = clouds(cname)
        p, d = pts.shape
        pos4 = _device.pack_positions(_device.h2d(pts))
        eps2 = 1e-6
        (vd, gd), t_direct = timed(lambda: direct_sums_device(pos4, pos4, d, eps2), reps=2)
        vd = vd.double().cpu().numpy()
        gd = gd.cpu().numpy()
        if a.pairs:
            combos = [(int(x.split(":")[0]), float(x.split(":")[1])) for x in a.pairs.split(",")]
        else:
            combos = [(int(o), float(t)) for o in a.orders.split(",") for t in a.thetas.split(",")]
        for order, theta in combos:
            if True:
                (vt, gt), t_tree = timed(
                    lambda: tree.tree_sums_device(pos4, pos4, d, eps2, order, theta,
                                                  leaf_cap=a.leaf))
                st = {"timing": True}  # sizes and synchronised phase times, separate call
                tree.tree_sums_device(pos4, pos4, d, eps2, order, theta, stats=st,
                                      leaf_cap=a.leaf)
                vt = vt.cpu().numpy()
                gt = gt.cpu().numpy()
                e_cost = abs(vt.sum() - vd.sum()) / abs(vd.sum())
                e_grad = np.linalg.norm(gt - gd) / np.linalg.norm(gd)
                rec = dict(cloud=cname, p=p, dims=d,
                           err_cost=e_cost, err_grad=e_grad, t_tree_s=t_tree,
                           t_direct_s=t_direct, speedup=t_direct / t_tree,
                           leaf=a.leaf, pairs_per_target=st["pairs"] / p,
                           near_fraction=st["near_pairs"] / max(st["pairs"], 1), **st)
                print(json.dumps(rec), flush=True)
                lines.append(rec)
    if a.out:
        with open(a.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
