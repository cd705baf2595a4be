"""eval_repulsion_tree through the public numpy API on the C2 pattern (perturbed radial
1024 x 1024, 3D), wall time per call after a warm-up call (H2D/D2H included)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402

k = spk.perturb(spk.init_radial(1024, 1024, 3), 0.25, 0)
pts = k.points()
for prec in (1e-3, 1e-4):
    cfg = spk.RepulsionConfig(backend="tree", tree_precision=prec)
    spk.eval_repulsion_tree(pts, cfg)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        spk.eval_repulsion_tree(pts, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"tree_precision": prec, "p": len(pts), "wall_s_min": min(ts),
                      "wall_s_median": sorted(ts)[2]}), flush=True)
