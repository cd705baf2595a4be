"""Per-phase cycle breakdown of one polish ring lane (diagnostic build with
-DSPK_POLISH_PROF): speed, accel, hand-over, box, barrier, per ring step."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

torch.cuda.set_device(0)
cfg = bench.proj_config()
base = bench.start_pattern().coords
lib = _native.load()
lib.spk_polish_prof_read.argtypes = [ctypes.c_void_p]
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,1024").split(",")]:
    shots = _device.h2d(np.ascontiguousarray(base[:n]))
    out = torch.empty_like(shots)
    ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
    pv = _native.f64_array([0, 0, 0])
    for _ in range(2):
        _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), n,
                     1024, 3, cfg.speed_bound, cfg.accel_bound, 512, pv, 1, 0.048, 0, -1.0, 800,
                     None, None, None, None, ws.data_ptr(), ws.numel(), _device.stream())
        torch.cuda.synchronize()
    prof = np.zeros((3, 7), dtype=np.uint64)
    lib.spk_polish_prof_read(prof.ctypes.data)
    names = ["speed", "accel", "handover", "box", "bookkeeping", "barrier"]
    for who, row in zip(("warp0 lane5", "warp1 lane8", "last warp"), prof):
        steps = float(row[6])
        per = {k: float(row[i]) / steps for i, k in enumerate(names)}
        print(f"shots={n} {who} steps={int(steps)} cycles/step={sum(per.values()):.0f} " +
              " ".join(f"{k}={v:.0f}" for k, v in per.items()), flush=True)
