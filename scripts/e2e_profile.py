"""Per-call wall-time breakdown of bench.py's e2e loop body (C2, public numpy API)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200.optimizer import default_eta0, step_size  # noqa: E402

fld = spk.precompute_field(bench.density())
pcfg = bench.proj_config()
pattern = spk.project_pattern(bench.start_pattern(), pcfg)
rcfg = spk.RepulsionConfig(kernel_eps=bench.EPS_REP)
eta0 = default_eta0(pattern.n_samples, bench.EPS_REP)
prev_c = prev_g = None
eta = eta0
tim = {}


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    tim.setdefault(name, []).append(time.perf_counter() - t0)
    return out


for it in range(1, 5):
    att = t("eval_attraction", lambda: spk.eval_attraction(pattern, fld, "exact"))
    rep_cost, rep_grad = t("eval_repulsion", lambda: spk.eval_repulsion(pattern, rcfg))
    grad = t("host_grad", lambda: (att.grad - rep_grad).reshape(pattern.coords.shape))
    dk = None if prev_c is None else pattern.coords - prev_c
    dg = None if prev_g is None else grad - prev_g
    eta = t("step_size", lambda: step_size(it, eta, dk, dg, eta0, 20))
    prev_c, prev_g = pattern.coords.copy(), grad
    newc = t("host_update", lambda: spk.SamplingPattern(pattern.coords - eta * grad))
    pattern = t("project_pattern", lambda: spk.project_pattern(newc, pcfg))
    t("feasibility", lambda: spk.feasibility_residuals(pattern, pcfg))
print(json.dumps({k: [round(x * 1e3, 2) for x in v] for k, v in tim.items()}, indent=1))
