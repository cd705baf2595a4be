"""Polish ring latency vs. concurrency: fixed sweep count (tol < 0 never converges)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

torch.cuda.set_device(0)
cfg = bench.proj_config()
base = bench.start_pattern().coords
sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
NS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 148, 296, 592, 1024]
for n in NS:
    shots = _device.h2d(np.ascontiguousarray(base[:n]))
    out = torch.empty_like(shots)
    ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
    pv = _native.f64_array([0, 0, 0])
    times = []
    for r in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), n, 1024, 3,
                     cfg.speed_bound, cfg.accel_bound, 512, pv, 1, 0.048, 0, -1.0, sweeps,
                     None, None, None, None, ws.data_ptr(), ws.numel(), _device.stream())
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    ms = min(times)
    steps = sweeps * 4.03
    print(f"shots={n:5d} sweeps={sweeps} {ms:8.2f} ms  {ms * 1e6 / steps:8.1f} ns/step  "
          f"~{ms * 1e-3 * 1.965e9 / steps:7.0f} cycles/step")
