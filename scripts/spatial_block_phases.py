"""Lattice treecode (attraction 1e-4, full3d lattice) for one rank's Morton-order target
block vs the number of ranks, at the full3d coarse levels (perturbed radial patterns):
where the per-rank time of the spatial layout goes."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())

import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, engine, tree  # noqa: E402

rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
fld = spk.precompute_field(rho)
order, theta = tree.auto_params(1e-4, 3)
src = fld.source_tree()
src.static_proxies(order)
eps2 = fld.kernel_eps ** 2
ops = engine.CudaOps()
NS = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,128").split(",")]
RANKS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")]
for ns in NS:
    full = spk.perturb(spk.init_radial(4096, ns, 3), 0.75, 0).points()
    pos4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(full)))
    perm = ops.spatial_order(pos4, 3)
    p = pos4.shape[0]
    for n, mode in [(r, m) for r in RANKS for m in ("0", "1")]:
        os.environ["SPK_TREE_SUBWALK"] = mode
        blk = pos4[perm[:p // n]].contiguous()
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tg = tree.TargetGroups(blk, 3)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st = {"timing": True}
            tree.tree_eval(tg, src, order, theta, eps2, static=True, far=False, stats=st)
            torch.cuda.synchronize()
        print(json.dumps({"n_s": ns, "ranks": n, "subwalk": mode == "1", "targets": blk.shape[0], "groups": tg.n_groups,
                          "groups_ms": 1e3 * (t1 - t0), "phases_ms": st["eval_phases_ms"],
                          "segments": st["segments"]}), flush=True)
