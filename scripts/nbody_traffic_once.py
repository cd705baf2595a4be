"""One fused N-body launch of a bench workload (ncu target for the per-workload DRAM
traffic in profiles/nbody_traffic.json): c1 / c2 / c4 through engine.CudaOps.sums on the
start positions, c3 through stack.StackedRun.evaluate (the batched launch).

    python scripts/nbody_traffic_once.py c1|c2|c3|c4
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())

import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, engine, stack  # noqa: E402

key = sys.argv[1]
bench.select_workload(key)
cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, grad_mode="exact",
                          grid_n=bench.GRID_N, seed=0, perturbation=bench.W["pert"])
fld = spk.precompute_field(bench.density())
if key == "c3":
    base = spk.init_radial(bench.N_C, bench.N_S, bench.DIMS)
    starts = np.stack([spk.perturb(base, bench.W["pert"], q).coords
                       for q in range(bench.W["stack"])])
    run = stack.StackedRun(starts, cfg, fld)
    run.evaluate()
else:
    coords = _device.h2d(np.ascontiguousarray(bench.start_pattern().coords))
    pos4 = _device.pack_positions(coords)
    engine.CudaOps().sums(pos4, pos4, coords, fld, cfg)
torch.cuda.synchronize()
print("ok", key)
