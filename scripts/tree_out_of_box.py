"""Treecode on clouds outside [-1, 1]^d (Morton keys clamp; tight boxes keep the MAC
honest): precision and time vs the exact kernel."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402

rng = np.random.default_rng(0)
for dims in (2, 3):
    for lo, hi in ((-3.0, 3.0), (0.5, 5.0), (-1e-3, 1e-3)):
        pts = rng.uniform(lo, hi, (200_000, dims))
        cfg = spk.RepulsionConfig(backend="tree", tree_precision=1e-4)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ct, gt = spk.eval_repulsion_tree(pts, cfg)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        cd, gd = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
        print(f"dims={dims} range=[{lo},{hi}] cost err {abs(ct-cd)/abs(cd):.2e} grad err "
              f"{np.linalg.norm(gt-gd)/np.linalg.norm(gd):.2e} tree {1e3*(t1-t0):.0f} ms", flush=True)
