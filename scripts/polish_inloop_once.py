"""One in-loop projection of recorded shots (bench_data/inloop_<config>.npz: the stepped,
pre-projection shots of optimizer iteration 6), tiled to N shots, FISTA 100 + polish to
the real tolerance -- the polish as it runs inside optimize (for ncu / timing).

    python scripts/polish_inloop_once.py [n_shots=128] [reps=1] [config=c2]
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.getcwd())

import bench  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
key = sys.argv[3] if len(sys.argv) > 3 else "c2"
bench.select_workload(key)
cfg = bench.proj_config()
shots = np.load(os.path.join(REPO, "bench_data", f"inloop_{key}.npz"))["shots"]
tiled = np.ascontiguousarray(np.concatenate([shots] * ((n + len(shots) - 1) // len(shots)))[:n])
dev = _device.h2d(tiled)
sw = torch.empty(n, dtype=torch.int32, device=dev.device)
for r in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = project_device(dev, cfg, sweeps=sw)
    e.record()
    torch.cuda.synchronize()
    swh = sw.cpu().numpy()
    print(f"n={n} projection {s.elapsed_time(e):.1f} ms; sweeps min {swh.min()} median "
          f"{int(np.median(swh))} max {swh.max()}", flush=True)
