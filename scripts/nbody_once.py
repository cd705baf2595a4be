"""Launch the fused K1+K2 N-body at the bench workload (C2) a few times; used as the
ncu target (the kernel of interest is launch index >= 1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
torch.cuda.set_device(0)
pts = bench.start_pattern().points().copy()
fld = spk.precompute_field(spk.discretize(spk.DensityParams(0.25, 2.0), bench.GRID_N, 3))
w = fld.device_sources()
ncell = int(np.prod(fld.sides))
p4 = _device.pack_positions(_device.h2d(pts))
p = p4.shape[0]
bufs = [torch.empty(p, dtype=torch.float64, device="cuda"),
        torch.empty((p, 3), dtype=torch.float64, device="cuda"),
        torch.empty(p, dtype=torch.float64, device="cuda"),
        torch.empty((p, 3), dtype=torch.float64, device="cuda")]
nb = _native.query("spk_nbody_workspace_bytes", p, ncell, p)
ws = _device.workspace(nb, "nbody")
times = []
for i in range(n):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _native.call("spk_fused_sums", p4.data_ptr(), p, 3, w.data_ptr(),
                 _native.i64_array(fld.sides), float(fld.kernel_eps ** 2), p4.data_ptr(), p, 1e-6,
                 *[b.data_ptr() for b in bufs], ws.data_ptr(), ws.numel(), _device.stream())
    e.record()
    times.append((s, e))
torch.cuda.synchronize()
ms = [s.elapsed_time(e) for s, e in times]
pairs = p * p + p * ncell
print("fused sums ms:", ["%.2f" % m for m in ms], "pairs/s: %.4g" % (pairs / (min(ms) / 1e3)))
