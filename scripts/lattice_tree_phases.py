"""Where a lattice-treecode attraction call spends its time vs the number of targets (the
multi-GPU per-rank share question): full3d lattice (385x385x209, attraction treecode
1e-4), targets = the first k shots of a perturbed radial pattern at N_s = 32 and 512.

    python scripts/lattice_tree_phases.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())

import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, tree  # noqa: E402

rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
fld = spk.precompute_field(rho)
order, theta = tree.auto_params(1e-4, 3)
src = fld.source_tree()
src.static_proxies(order)
eps2 = fld.kernel_eps ** 2
torch.cuda.synchronize()
for ns in (32, 512):
    full = spk.perturb(spk.init_radial(4096, ns, 3), 0.75, 0).points()
    for shots in (4096, 2048, 1024, 512):
        pts = np.ascontiguousarray(full[:shots * ns])
        tgt4 = _device.pack_positions(_device.h2d(pts))
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tg = tree.TargetGroups(tgt4, 3)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st = {"timing": True}
            tree.tree_eval(tg, src, order, theta, eps2, static=True, far=False, stats=st)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
        print(json.dumps({"n_s": ns, "shots": shots, "targets": shots * ns,
                          "groups_ms": 1e3 * (t1 - t0), "eval_total_ms": 1e3 * (t2 - t1),
                          "phases_ms": st.get("eval_phases_ms"), "groups": st.get("groups"),
                          "segments": st.get("segments"), "pairs": st.get("pairs")}),
              flush=True)

# repulsion treecode (1e-3): a rank's targets against all sources
order_r, theta_r = tree.auto_params(1e-3, 3)
for ns in (128, 512):
    full = spk.perturb(spk.init_radial(4096, ns, 3), 0.75, 0).points()
    src4 = _device.pack_positions(_device.h2d(np.ascontiguousarray(full)))
    for shots in (4096, 1024, 512):
        tgt4 = src4[:shots * ns]
        for rep in range(2):
            st = {"timing": True}
            tree.tree_sums_device(tgt4, src4, 3, 1e-6, order_r, theta_r, stats=st)
        print(json.dumps({"repulsion": True, "n_s": ns, "shots": shots,
                          "phases_ms": st.get("phases_ms"),
                          "eval_phases_ms": st.get("eval_phases_ms")}), flush=True)
