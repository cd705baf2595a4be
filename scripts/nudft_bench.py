"""NUDFT kernel throughput (voxel-sample products / s) for the analysis path, device time
with CUDA events after warm-up; plus compute_psf / density_compensation wall times."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, analysis as an  # noqa: E402

CASES = [
    ("C1 pattern 64x512, 256^2 grid", (64, 512, 2), (256, 256)),
    ("C2 pattern 1024x1024, 64^3 grid", (1024, 1024, 3), (64, 64, 64)),
    ("C2 pattern 1024x1024, 128^3 grid", (1024, 1024, 3), (128, 128, 128)),
]


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


for name, (n_c, n_s, d), grid in CASES:
    k = spk.perturb(spk.init_radial(n_c, n_s, d), 0.25, 0)
    pts = _device.h2d(np.ascontiguousarray(k.points()))
    p = pts.shape[0]
    vox = int(np.prod(grid))
    w = torch.zeros((p, 2), dtype=torch.float64, device=pts.device)
    w[:, 0] = 1.0
    rec = dict(case=name, p=p, voxels=vox, products=p * vox)
    for prec in ("fp64", "mixed"):
        img = an.nudft_adjoint_device(pts, w, grid, prec)
        t_adj = dev_time(lambda: an.nudft_adjoint_device(pts, w, grid, prec))
        t_fwd = dev_time(lambda: an.nudft_forward_device(pts, img, grid, prec))
        rec[prec] = dict(adjoint_s=t_adj, adjoint_products_per_s=p * vox / t_adj,
                         forward_s=t_fwd, forward_products_per_s=p * vox / t_fwd)
    t0 = time.perf_counter()
    psf = spk.compute_psf(k, grid, allow_slow=True)
    rec.update(compute_psf_wall_s=time.perf_counter() - t0, psf_peak=psf.peak_value)
    print(json.dumps(rec), flush=True)
