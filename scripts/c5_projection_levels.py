"""C5 projection measurement: ms per project_pattern at every level of the
full3d multi-resolution schedule (N_s = 32 ... 2048, alpha/beta scaled 64 ... 1,
4096 shots), polish sweeps per shot, for a level-start input (decimated perturbed radial
init) and an in-loop input (projected pattern + a 2e-3 step), plus the CPU reference
(bit-exact C port, all host threads) on a shot sample scaled to 4096 shots."""
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2108_02991_b200 as spk  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.projection import project_device, stacked_operator_norm  # noqa: E402

N_C, N_S, N_D = 4096, 2048, 6
cpu_shots = int(sys.argv[1]) if len(sys.argv) > 1 else 8
torch.cuda.set_device(0)
hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=2e-6,
                      fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dims=3)
lim = spk.normalized_limits(hw)
full = spk.perturb(spk.init_radial(N_C, N_S, 3), 0.75, 0).coords
rng = np.random.default_rng(0)
rows = []
for level in range(N_D + 1):
    ns = N_S // 2 ** (N_D - level)
    scale = 2.0 ** (N_D - level)
    pin = spk.LinearConstraint(ns // 2, np.zeros(3))
    cfg = spk.ProjectionConfig(alpha=lim.alpha * scale, beta=lim.beta * scale, raster_dt=1e-5,
                               n_pit=100, pin=pin)
    tau = 1.0 / stacked_operator_norm(ns, ns // 2)
    start = np.ascontiguousarray(full[:, :: 2 ** (N_D - level), :])
    rec = {"level": level, "n_s": ns, "scale": scale}
    for kind in ("level_start", "in_loop"):
        x = start
        if kind == "in_loop":
            x = _device.d2h(project_device(_device.h2d(start), cfg, tau=tau))
            x = x + rng.uniform(-2e-3, 2e-3, x.shape)
        dev = _device.h2d(x)
        sweeps = torch.empty(N_C, dtype=torch.int32, device="cuda")
        project_device(dev, cfg, tau=tau, sweeps=sweeps)  # warm-up
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        project_device(dev, cfg, tau=tau, sweeps=sweeps)
        e.record()
        torch.cuda.synchronize()
        sw = sweeps.cpu().numpy()
        t0 = time.perf_counter()
        _, csw = orc.project_all(x[:cpu_shots], cfg.speed_bound, cfg.accel_bound, ns // 2,
                                 np.zeros(3), 100, tau, 0.1 * cfg.feas_tol)
        cpu_s = (time.perf_counter() - t0) * N_C / cpu_shots
        assert np.array_equal(csw, sw[:cpu_shots])  # same sweep counts (bit-exact polish)
        rec[kind] = {"gpu_ms": s.elapsed_time(e), "sweeps_median": float(np.median(sw)),
                     "sweeps_max": int(sw.max()), "sweeps_min": int(sw.min()),
                     "cpu_s_extrapolated": cpu_s, "cpu_threads": orc.max_threads()}
    rows.append(rec)
    print(json.dumps(rec), flush=True)
