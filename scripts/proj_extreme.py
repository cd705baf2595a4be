import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk
from paper_2108_02991_b200 import _device
from paper_2108_02991_b200.projection import project_device
from oracle import oracle as orc
rng = np.random.default_rng(5)
bad = 0
for trial in range(80):
    dims = int(rng.choice([2, 3])); ns = int(rng.choice([2, 3, 9, 64, 513])); n_c = int(rng.integers(1, 4))
    a = float(rng.choice([1e-6, 1e-3, 0.5, 10.0])); b = float(rng.choice([1e-8, 1e-4, 0.2, 100.0]))
    scale = float(rng.choice([0.0, 1e-9, 5.0, 1e3]))
    pin = int(rng.choice([-1, 0, ns - 1]))
    pv = rng.uniform(-1, 1, dims) if pin >= 0 else None
    shots = rng.uniform(-scale, scale, (n_c, ns, dims))
    cfg = spk.ProjectionConfig(alpha=a, beta=b, raster_dt=1.0, n_pit=int(rng.choice([1, 20])),
                               pin=None if pin < 0 else spk.LinearConstraint(pin, pv),
                               monotone=bool(rng.integers(0, 2)))
    tau = 1.0 / spk.projection.stacked_operator_norm(ns, pin)
    cap = int(rng.choice([1, 50, 2000]))
    sw = torch.zeros(n_c, dtype=torch.int32, device="cuda")
    out = _device.d2h(project_device(_device.h2d(shots), cfg, tau=tau, sweeps=sw, max_sweeps=cap))
    ref, rsw = orc.project_all(shots, a, b, pin, pv, cfg.n_pit, tau, 0.1 * cfg.feas_tol, monotone=cfg.monotone, max_sweeps=cap)
    ok = np.array_equal(out, ref, equal_nan=True) and np.array_equal(_device.d2h(sw), rsw)
    if not ok:
        bad += 1
        print("MISMATCH", dims, ns, n_c, a, b, scale, pin, cfg.monotone, cap, np.nanmax(np.abs(out-ref)))
print("extreme projection cases:", 80 - bad, "bitwise /", 80)
