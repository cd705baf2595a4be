"""In-loop-like polish timing at the C2 shape: fixed 800 sweeps (tol < 0) for 1024 shots,
and the bench's real projection (step + projection) averaged over 3 optimizer steps."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

cfg = bench.proj_config()
base = bench.start_pattern().coords
for n in (1, 1024):
    shots = _device.h2d(np.ascontiguousarray(base[:n]))
    out = torch.empty_like(shots)
    ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
    pv = _native.f64_array([0, 0, 0])
    best = 1e30
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), n,
                     1024, 3, cfg.speed_bound, cfg.accel_bound, 512, pv, 1, 0.048, 0, -1.0,
                     1600, None, None, None, None, ws.data_ptr(), ws.numel(), _device.stream())
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"shots={n} 1600 sweeps: {best:.1f} ms", flush=True)
