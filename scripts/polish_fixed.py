"""Polish timing at fixed sweep counts (tol < 0): C2 shape, in-loop shots
(bench_data/inloop_c2.npz after FISTA) tiled to n shots.  For A/B of polish variants
whose results may differ (experiments): the work is independent of convergence.

    python scripts/polish_fixed.py [n=16] [sweeps=3200]
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.getcwd())

import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3200
bench.select_workload("c2")
cfg = bench.proj_config()
shots = np.load(os.path.join(REPO, "bench_data", "inloop_c2.npz"))["shots"]
tiled = np.ascontiguousarray(np.concatenate([shots] * ((n + len(shots) - 1) // len(shots)))[:n])
dev = _device.h2d(tiled)
out = torch.empty_like(dev)
ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
pv = _native.f64_array([0, 0, 0])
from paper_2108_02991_b200.projection import stacked_operator_norm  # noqa: E402
tau = 1.0 / stacked_operator_norm(1024, 512)
best = 1e30
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _native.call("spk_project_all", dev.data_ptr(), None, 0.0, None, out.data_ptr(), n, 1024,
                 3, cfg.speed_bound, cfg.accel_bound, 512, pv, 100, tau, 0, -1.0, sweeps, None,
                 None, None, None, ws.data_ptr(), ws.numel(), _device.stream())
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
steps = (sweeps + 255) // 256 * 1056
print(f"n={n} FISTA 100 + {sweeps} sweeps: {best:.2f} ms  (~{best * 1e-3 * 1.965e9 / steps:.0f} "
      f"cycles per ring step incl. FISTA)", flush=True)
