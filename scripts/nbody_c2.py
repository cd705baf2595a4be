"""Fused N-body launch time at C2 (exact repulsion + lattice attraction), CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, engine  # noqa: E402

for key in ("c2", "c1", "c4"):
    bench.select_workload(key)
    cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, grad_mode="exact",
                              grid_n=bench.GRID_N, seed=0, perturbation=bench.W["pert"])
    fld = spk.precompute_field(bench.density())
    coords = _device.h2d(np.ascontiguousarray(bench.start_pattern().coords))
    pos4 = _device.pack_positions(coords)
    ops = engine.CudaOps()
    reps = 1 if key == "c4" else 3
    ops.sums(pos4, pos4, coords, fld, cfg)
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = ops.sums(pos4, pos4, coords, fld, cfg)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{key}: fused N-body {best:.1f} ms", flush=True)
