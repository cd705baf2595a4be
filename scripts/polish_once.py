"""One polish run at the C2 shape with 400 fixed sweeps (for ncu instruction counts)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

cfg = bench.proj_config()
base = bench.start_pattern().coords
n = 296
shots = _device.h2d(np.ascontiguousarray(base[:n]))
out = torch.empty_like(shots)
ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
pv = _native.f64_array([0, 0, 0])
_native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), n, 1024, 3,
             cfg.speed_bound, cfg.accel_bound, 512, pv, 1, 0.048, 0, -1.0, 400, None, None,
             None, None, ws.data_ptr(), ws.numel(), _device.stream())
torch.cuda.synchronize()
print("ok")
