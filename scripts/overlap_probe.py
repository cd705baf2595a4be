"""Can the lattice sums (K2) of finished shots hide under the polish tail?  At the C2 in-loop
state (bench's 5 warm-up iterations), rank 0's share at N ranks (N_C/N shots): time the
projection alone, K2 for those shots alone, and both launched concurrently on two streams
(projection on a high-priority stream).  Timing-only: K2 reads the pre-projection
positions.

    python scripts/overlap_probe.py [n_ranks=8] [k2|fused]

With "fused", the second kernel is the share's full fused K1 + K2 launch (its targets
against all sources): could the polish hide under the whole N-body?
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())

import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, engine  # noqa: E402
from paper_2108_02991_b200.attraction import grid_sums_device  # noqa: E402
from paper_2108_02991_b200.optimizer import _bb_step  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
what = sys.argv[2] if len(sys.argv) > 2 else "k2"
bench.select_workload("c2")
cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=3, grad_mode="exact",
                          grid_n=bench.GRID_N, seed=0, perturbation=bench.W["pert"])
fld = spk.precompute_field(bench.density())
pcfg = bench.proj_config()
run = engine.ShardedRun(np.ascontiguousarray(bench.start_pattern().coords), cfg, fld)
run.project(pcfg)
step, state = bench.optimizer_step(run, cfg)
for _ in range(5):
    step()
state["it"] += 1
att, rep, bad, dots = run.evaluate()
eta = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"], state["eta0"],
               cfg.fixed_step_iters)
ns = bench.N_S
cnt = bench.N_C // nr
coords = run.coords[:cnt]
grad = run.grad[:cnt]
tgt = run.pos4_all[:cnt * ns]
out = torch.empty_like(coords)
hi = torch.cuda.Stream(priority=-1)
lo = torch.cuda.Stream(priority=0)
eps2 = fld.kernel_eps ** 2


def proj():
    project_device(coords, pcfg, grad=grad, eta=eta, out=out)


def k2():
    if what == "fused":
        run.ops.sums(tgt, run.pos4_all, coords, fld, cfg)
    else:
        grid_sums_device(tgt, fld, eps2)


def timed(fn):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    hi.wait_event(ev)
    lo.wait_event(ev)
    with torch.cuda.stream(hi):
        proj()
    with torch.cuda.stream(lo):
        k2()
    cur.wait_stream(hi)
    cur.wait_stream(lo)


k2()
for rep in range(2):
    tp, tk, tb = timed(proj), timed(k2), timed(both)
    print(f"N={nr} ({cnt} shots): projection {tp:.1f} ms, {what} {tk:.1f} ms, sum {tp + tk:.1f}, "
          f"concurrent {tb:.1f} ms (hidden {tp + tk - tb:.1f} of {min(tp, tk):.1f})", flush=True)
