"""Polish timing at the C4 shape (4096 shots x 2048 samples): 400 fixed sweeps (tol < 0)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

bench.select_workload("c4")
cfg = bench.proj_config()
base = bench.start_pattern().coords
n = base.shape[0]
shots = _device.h2d(np.ascontiguousarray(base))
out = torch.empty_like(shots)
ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 2048, 3, 0), "p")
pv = _native.f64_array([0, 0, 0])
for sweeps in (1, 400):
    best = 1e30
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), n,
                     2048, 3, cfg.speed_bound, cfg.accel_bound, 1024, pv, 100, 0.048, 0, -1.0,
                     sweeps, None, None, None, None, ws.data_ptr(), ws.numel(), _device.stream())
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"C4 shape, FISTA 100 + {sweeps} sweeps: {best:.1f} ms", flush=True)
