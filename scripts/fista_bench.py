"""FISTA-only projection time (max_sweeps = 1) at the C2 and C4 shapes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402

for key in ("c2", "c4"):
    bench.select_workload(key)
    pcfg = bench.proj_config()
    coords = _device.h2d(np.ascontiguousarray(bench.start_pattern().coords))
    out = torch.empty_like(coords)
    ms = []
    for r in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        project_device(coords, pcfg, out=out, max_sweeps=1)
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    print(key, coords.shape, "fista+1 sweep ms", [round(x, 1) for x in ms], flush=True)
