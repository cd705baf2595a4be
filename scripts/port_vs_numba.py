"""The reference arm's CPU code (oracle/, a C port of the numba kernels) vs the
reference's own numba kernels on the same host threads: evidence that the port is a
conservative (not a slowed-down) stand-in.  Authoring container only (imports
/root/reference).  Writes profiles/r02_port_vs_numba.json.

    NUMBA_CACHE_DIR=/tmp/numba_cache python scripts/port_vs_numba.py
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import numba  # noqa: E402
from vdtraj import _treecode as tc  # noqa: E402
from vdtraj import optimizer as om, projection as pr, core  # noqa: E402
from oracle import oracle as orc  # noqa: E402

threads = os.cpu_count()
numba.set_num_threads(threads)
out = {"threads": threads, "cpu": open("/proc/cpuinfo").read().split("model name")[1]
       .split("\n")[0].strip(": \t")}

# direct_sums (K1), p = 2^16 full (4.3e9 pairs)
p = 1 << 16
pts = om.perturb(om.init_radial(64, 1024, 3), 0.25, 0).points().copy()
val = np.empty(p)
grad = np.empty_like(pts)
tc.direct_sums(pts[:256].copy(), 1e-6, val[:256], grad[:256])  # jit warm-up
best = {}
for name, fn in (("numba", lambda: tc.direct_sums(pts, 1e-6, val, grad)),
                 ("port", lambda: orc.direct_sums(pts, 1e-6, threads))):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    best[name] = min(ts)
out["direct_sums"] = {"p": p, "pairs": p * p,
                      "numba_pairs_per_s": p * p / best["numba"],
                      "port_pairs_per_s": p * p / best["port"]}

# projection: 16 in-loop C2 shots if recorded, else fresh-init shots
path = os.path.join(REPO, "bench_data", "inloop_c2.npz")
shots = np.load(path)["shots"] if os.path.exists(path) else \
    om.perturb(om.init_radial(1024, 1024, 3), 0.25, 0).coords[:16]
hw = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=2e-6,
                       fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dims=3)
lim = core.normalized_limits(hw)
ns = shots.shape[1]
cfg = pr.ProjectionConfig(alpha=lim.alpha, beta=lim.beta, raster_dt=1e-5, n_pit=100,
                          pin=core.LinearConstraint(pinned_index=ns // 2,
                                                    pinned_value=np.zeros(3)))
pr.project_pattern(core.SamplingPattern(shots[:1]), cfg)  # jit warm-up
t0 = time.perf_counter()
ref = pr.project_pattern(core.SamplingPattern(shots), cfg).coords
t_numba = time.perf_counter() - t0
tau = 1.0 / pr._stacked_operator_norm(ns, ns // 2)
t0 = time.perf_counter()
mine, _ = orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, ns // 2, np.zeros(3), 100,
                          tau, 0.1 * cfg.feas_tol, nthreads=threads)
t_port = time.perf_counter() - t0
out["project_pattern"] = {"shots": int(shots.shape[0]), "n_s": ns,
                          "input": os.path.basename(path) if os.path.exists(path) else "fresh",
                          "numba_s": t_numba, "port_s": t_port,
                          "bit_identical": bool(np.array_equal(ref, mine))}
print(json.dumps(out, indent=1))
with open(os.path.join(REPO, "profiles", "r02_port_vs_numba.json"), "w") as fh:
    json.dump(out, fh, indent=1)
