"""Per-phase timing of one optimize() iteration at the bench workload (C2), with CUDA
events on the launching stream, plus polish sweep statistics.  Used to pick the next
optimisation target; the numbers are copied into profiles/."""

import argparse
import json
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import engine  # noqa: E402
from paper_2108_02991_b200.optimizer import _bb_step, default_eta0  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402


class PhaseOps(engine.CudaOps):
    def __init__(self):
        super().__init__()
        self.times = {}
        self.sweeps = []

    def _t(self, name, fn, *a, **k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn(*a, **k)
        e.record()
        self.times.setdefault(name, []).append((s, e))
        return out

    def sums(self, *a, **k):
        return self._t("nbody", super().sums, *a, **k)

    def combine(self, *a, **k):
        return self._t("combine", super().combine, *a, **k)

    def project(self, coords, proj_cfg, grad, eta, out, pos4, nonfinite, sweeps=None):
        sw = sweeps if sweeps is not None else torch.empty(coords.shape[0], dtype=torch.int32,
                                                           device=coords.device)
        r = self._t("project", project_device, coords, proj_cfg, grad=grad, eta=eta, out=out,
                    pos4=pos4, nonfinite=nonfinite, sweeps=sw)
        self.sweeps.append(sw)
        # FISTA alone: same call with one polish sweep (polish cost ~ 1 batch)
        tmp = torch.empty_like(out)
        self._t("fista_only", project_device, coords, proj_cfg, grad=grad, eta=eta, out=tmp,
                max_sweeps=1)
        return r

    def residuals(self, *a, **k):
        return self._t("residuals", super().residuals, *a, **k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    bench.select_workload(args.config)
    W = bench.W
    torch.cuda.set_device(0)
    extra = {}
    if W.get("tree"):
        extra = dict(attraction_tree_precision=W["att_prec"],
                     repulsion=spk.RepulsionConfig(backend="tree", tree_precision=W["rep_prec"]))
    cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, grad_mode="exact",
                              grid_n=bench.GRID_N, seed=0, perturbation=W["pert"], **extra)
    fld = spk.precompute_field(bench.density())
    pcfg = bench.proj_config()
    ops = PhaseOps()
    run = engine.ShardedRun(np.ascontiguousarray(bench.start_pattern().coords), cfg, fld,
                            ops=ops)
    run.project(pcfg)
    eta0 = default_eta0(run.p, 1e-3)
    eta = eta0
    for it in range(1, args.iters + 1):
        att, rep, bad, dots = run.evaluate()
        eta = _bb_step(it, eta, dots[0], dots[1], it > 1, eta0, 20)
        run.step_project(pcfg, eta)
        run.residual_max(pcfg)
    torch.cuda.synchronize()
    out = {}
    for k, v in ops.times.items():
        ms = [s.elapsed_time(e) for s, e in v]
        out[k] = {"ms": ms, "mean_ms": float(np.mean(ms[1:] if len(ms) > 1 else ms))}
    sw = [x.cpu().numpy() for x in ops.sweeps]
    out["sweeps"] = [{"min": int(x.min()), "median": float(np.median(x)), "max": int(x.max())}
                     for x in sw]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
