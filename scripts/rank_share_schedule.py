"""Projected multi-GPU scaling of the full3d multi-resolution schedule (4096
shots x 2048 samples, n_decim 6, N_s 32 ... 2048, constraints scaled 64 ... 1; repulsion
tree 1e-3, attraction treecode 1e-4), timed on ONE B200.

The schedule runs for real on one GPU.  At iteration --probe of every level (inside the
fixed-step phase, so every rank would use the same step eta0) each rank's share of that
iteration at N = 1, 2, 4, 8 is timed in isolation: its targets against all sources
(treecode repulsion and lattice attraction, incl. the per-rank tree builds; the
auto-mode probe, which a run does once per level, is warmed untimed), the
combine, the projection of its shots.  The N-rank iteration is the slowest rank plus the
position all-gather (estimated at 600 GB/s).  Two layouts of the N-body targets are timed:
by shot (each rank's own samples) and spatial (engine.ShardedRun.spatial: rank r takes the
r-th Morton-order block of all samples; plus the all-gather that returns the results to
the shots' owners, estimated likewise).  Per level the projected time is
n_git x that; the sum over levels is the projected schedule time.

    python scripts/rank_share_schedule.py [--n-git 100] [--probe 10] > profiles/r02_rank_share_full3d.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())

import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import optimizer as om  # noqa: E402
from paper_2108_02991_b200 import tree  # noqa: E402

# A run re-probes the treecode rows every tree.REPROBE_EVERY calls (amortised over the
# level); the timed shares here must not land on a probe, so the row cache is kept.
tree.REPROBE_EVERY = 10 ** 9

ap = argparse.ArgumentParser()
ap.add_argument("--n-git", type=int, default=100)
ap.add_argument("--probe", type=int, default=10)
ap.add_argument("--ranks", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
worlds = [int(x) for x in a.ranks.split(",")]
REPS = a.reps

hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=2e-6,
                      fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dims=3)
cfg = spk.OptimizerConfig(n_c=4096, n_s=2048, dims=3, n_decim=6, n_git=a.n_git, n_pit=100,
                          perturbation=0.75, seed=0, grad_mode="exact",
                          attraction_tree_precision=1e-4,
                          repulsion=spk.RepulsionConfig(backend="tree", kernel_eps=1e-3,
                                                        tree_precision=1e-3))
rho = spk.discretize_anisotropic(spk.DensityParams(0.25, 2.0), (192, 192, 104), 3)
state = om.start(cfg, hw, rho)
run, ops = state.run, state.run.ops


def ev():
    return torch.cuda.Event(enable_timing=True)


levels = []
t0 = time.perf_counter()
while True:
    if state.it == a.probe - 1 and not state.done and state.it < cfg.n_git:
        assert state.it + 1 <= cfg.fixed_step_iters
        ns, d = run.n_s, run.d
        rec = {"level": state.level, "n_s": ns, "iteration": state.it + 1, "ranks": {}}
        for n in worlds:
            base, extra = divmod(cfg.n_c, n)
            counts = [base + (1 if r < extra else 0) for r in range(n)]
            offs = [sum(counts[:r]) for r in range(n)]
            # the treecodes' auto-mode probe runs once per (sizes, precision) and level
            # in a real run (row cache): warm it for this share size, untimed
            g0 = torch.empty((counts[0], ns, d), dtype=torch.float64, device="cuda")
            ops.sums(run.pos4_all[:counts[0] * ns], run.pos4_all, run.coords[:counts[0]],
                     state.fld, cfg)
            del g0
            per = []
            perm = ops.spatial_order(run.pos4_all, d)
            sb = [run.p * r // n for r in range(n + 1)]
            # warm the probe for the spatial block size too
            ops.sums(run.pos4_all[perm[sb[0]:sb[1]]].contiguous(), run.pos4_all, None,
                     state.fld, cfg)
            for r in range(n):
                lo, cnt = offs[r], counts[r]
                coords = run.coords[lo:lo + cnt]
                tgt = run.pos4_all[lo * ns:(lo + cnt) * ns]
                grad = torch.empty((cnt, ns, d), dtype=torch.float64, device="cuda")
                out = torch.empty_like(grad)
                pos4 = torch.empty((cnt * ns, 4), dtype=torch.float32, device="cuda")
                reps = []
                for _ in range(REPS):
                    e = [ev() for _ in range(5)]
                    torch.cuda.synchronize()
                    e[0].record()
                    va, ga, vr, gr = ops.sums(tgt, run.pos4_all, coords, state.fld, cfg)
                    ops.combine(va, ga, vr, gr, run.p, coords, None, None, grad.view(-1, d))
                    e[1].record()
                    ops.project(coords, state.proj_cfg, grad, float(state.eta0), out, pos4,
                                None)
                    ops.residuals(out, state.proj_cfg)
                    e[2].record()
                    # spatial layout (engine.ShardedRun.spatial): this rank's Morton block
                    blk = run.pos4_all[perm[sb[r]:sb[r + 1]]].contiguous()
                    e[3].record()
                    ops.sums(blk, run.pos4_all, None, state.fld, cfg)
                    e[4].record()
                    torch.cuda.synchronize()
                    reps.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]),
                                 e[3].elapsed_time(e[4])))
                # median of REPS timings per component (single timings vary by up to 40 %)
                per.append(tuple(float(np.median([x[k] for x in reps])) for k in range(3)))
            gather = 16.0 * run.p * (n - 1) / n / 600e9 * 1e3 if n > 1 else 0.0
            exch = 8.0 * (2 + 2 * d) * run.p * (n - 1) / n / 600e9 * 1e3 if n > 1 else 0.0
            step = max(s + p for s, p, _ in per) + gather
            # spatial: sums of the Morton block + combine (same cost as in the shot
            # layout's sums column, dominated by the sums), projection of the shots
            step_sp = max(sp for _, _, sp in per) + max(p for _, p, _ in per) + gather + exch
            rec["ranks"][n] = {"step_ms": step, "max_sums_ms": max(s for s, _, _ in per),
                               "max_project_ms": max(p for _, p, _ in per),
                               "allgather_est_ms": gather,
                               "spatial_step_ms": step_sp,
                               "spatial_max_sums_ms": max(sp for _, _, sp in per),
                               "spatial_exchange_est_ms": exch}
        levels.append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    if om.step(state) is None:
        break
torch.cuda.synchronize()
wall = time.perf_counter() - t0
summary = {"schedule": "full3d.cfg: 4096 x 2048, n_decim 6, n_git %d, repulsion tree 1e-3, "
                       "attraction treecode 1e-4 over 385x385x209" % cfg.n_git,
           "one_gpu_wall_s_incl_probes": wall, "levels": levels, "projected": {}}
for n in worlds:
    tot = sum(cfg.n_git * lv["ranks"][n]["step_ms"] for lv in levels) / 1e3
    tsp = sum(cfg.n_git * lv["ranks"][n]["spatial_step_ms"] for lv in levels) / 1e3
    summary["projected"][n] = {"schedule_s": tot, "spatial_schedule_s": tsp}
t1 = summary["projected"][worlds[0]]["schedule_s"]
for n in worlds:
    summary["projected"][n]["efficiency"] = t1 / (n * summary["projected"][n]["schedule_s"])
    summary["projected"][n]["spatial_efficiency"] = (
        t1 / (n * summary["projected"][n]["spatial_schedule_s"]))
print(json.dumps(summary))
