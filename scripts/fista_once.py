"""One FISTA-only projection at the C4 shape (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402

bench.select_workload(sys.argv[1] if len(sys.argv) > 1 else "c4")
pcfg = bench.proj_config()
coords = _device.h2d(np.ascontiguousarray(bench.start_pattern().coords))
out = torch.empty_like(coords)
project_device(coords, pcfg, out=out, max_sweeps=1)
torch.cuda.synchronize()
print("ok")
