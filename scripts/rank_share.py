"""Per-rank share of one optimizer iteration at N = 2, 4, 8 ranks, timed on ONE B200.

With shots sharded contiguously (engine.ShardedRun), rank r of N evaluates its own
targets against ALL sources (fused K1 + K2), combines, and projects its own shots; the
ranks then meet in the position all-gather.  So the N-rank iteration takes
max_r (sums_r + combine_r + project_r + residuals_r) + all-gather.  This script brings a
single-GPU run to the in-loop state (bench.py's 5 warm-up iterations), then times every
rank's share of the next iterations in isolation on the same device and reports the
projected strong-scaling efficiency t_1 / (N t_N).  The all-gather (16 B per sample over
NVLink 5, 16 MiB at C2) is added as an estimate at 600 GB/s.

Each share is timed twice: the plain schedule (fused K1 + K2, combine, projection) and the
overlap schedule the engine uses on tail-bound ranks (ShardedRun.overlap): projection with
every polish group's K2 on a side stream, then K1 alone; the polish order comes from the
previous iteration's sweep counts of the same shots, as in the engine.

    python scripts/rank_share.py [--config c2|c4] [--iters 3] > profiles/r02_rank_share_c2.jsonl
"""
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
from paper_2108_02991_b200.optimizer import _bb_step  # noqa: E402
from paper_2108_02991_b200.projection import project_device  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--groups", type=int, default=None,
                    help="polish groups of the overlap schedule (default: the engine's)")
    args = ap.parse_args()
    if args.groups:
        engine.CudaOps.OVERLAP_GROUPS = args.groups
    bench.select_workload(args.config)
    cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, n_pit=100,
                              grad_mode="exact", grid_n=bench.GRID_N, seed=0,
                              perturbation=bench.W["pert"])
    fld = spk.precompute_field(bench.density())
    pcfg = bench.proj_config()
    run = engine.ShardedRun(np.ascontiguousarray(bench.start_pattern().coords), cfg, fld)
    run.project(pcfg)
    step, state = bench.optimizer_step(run, cfg)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ops, ns, d = run.ops, run.n_s, run.d
    worlds = [int(x) for x in args.ranks.split(",")]
    rows = {n: [] for n in worlds}
    prev_sweeps = {}
    for it in range(args.iters):
        # this iteration's step size, from the full evaluation (as every rank would get)
        state["it"] += 1
        att, rep, bad, dots = run.evaluate()
        eta = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                       state["eta0"], cfg.fixed_step_iters)
        for n in worlds:
            base, extra = divmod(bench.N_C, n)
            counts = [base + (1 if r < extra else 0) for r in range(n)]
            offs = [sum(counts[:r]) for r in range(n)]
            per = []
            for r in range(n):
                lo, cnt = offs[r], counts[r]
                coords = run.coords[lo:lo + cnt]
                tgt = run.pos4_all[lo * ns:(lo + cnt) * ns]
                grad = torch.empty((cnt, ns, d), dtype=torch.float64, device="cuda")
                out = torch.empty_like(grad)
                pos4 = torch.empty((cnt * ns, 4), dtype=torch.float32, device="cuda")
                flag = torch.zeros(1, dtype=torch.int32, device="cuda")
                sw = torch.empty(cnt, dtype=torch.int32, device="cuda")
                e = [ev() for _ in range(4)]
                torch.cuda.synchronize()
                e[0].record()
                va, ga, vr, gr = ops.sums(tgt, run.pos4_all, coords, fld, cfg)
                ops.combine(va, ga, vr, gr, run.p, coords, None, None, grad.view(-1, d))
                e[1].record()
                project_device(coords, pcfg, grad=grad, eta=float(eta), out=out, pos4=pos4,
                               nonfinite=flag, sweeps=sw)
                e[2].record()
                ops.residuals(out, pcfg)
                e[3].record()
                torch.cuda.synchronize()
                rec = {"rank": r, "shots": cnt, "sums_ms": e[0].elapsed_time(e[1]),
                       "project_ms": e[1].elapsed_time(e[2]),
                       "residual_ms": e[2].elapsed_time(e[3])}
                # overlap schedule: order by the previous iteration's sweeps of these shots
                key = (n, r)
                order = prev_sweeps.get(key)
                if order is not None:
                    order = torch.argsort(order, descending=True, stable=True).to(torch.int32)
                av = torch.empty(cnt * ns, dtype=torch.float64, device="cuda")
                ag = torch.empty((cnt * ns, d), dtype=torch.float64, device="cuda")
                sw2 = torch.empty(cnt, dtype=torch.int32, device="cuda")
                f = [ev() for _ in range(4)]
                torch.cuda.synchronize()
                f[0].record()
                _, k2ev = ops.project_overlap(coords, pcfg, grad, float(eta), out, pos4, flag,
                                              fld, av, ag, sw2, order)
                f[1].record()
                vr2, gr2 = ops.repulsion_sums(tgt, run.pos4_all, cfg)
                f[3].record()
                for e_ in k2ev:
                    torch.cuda.current_stream().wait_event(e_)
                ops.combine(av, ag, vr2, gr2, run.p, coords, None, None, grad.view(-1, d))
                ops.residuals(out, pcfg)
                f[2].record()
                torch.cuda.synchronize()
                # projection (K2 may continue past f[1]), then K1 co-running with K2's tail
                rec["overlap_project_k2_ms"] = f[0].elapsed_time(f[1])
                rec["overlap_k1_combine_ms"] = f[1].elapsed_time(f[2])
                rec["overlap_k1_ms"] = f[1].elapsed_time(f[3])
                # the same with K2 only on SMs without polish CTAs (sm_busy, "polite")
                sw4 = torch.empty_like(sw2)
                h4 = [ev() for _ in range(2)]
                torch.cuda.synchronize()
                h4[0].record()
                _, k2ev4 = ops.project_overlap(coords, pcfg, grad, float(eta), out, pos4, flag,
                                               fld, av, ag, sw4, order, polite=True)
                vr4, gr4 = ops.repulsion_sums(tgt, run.pos4_all, cfg)
                for e_ in k2ev4:
                    torch.cuda.current_stream().wait_event(e_)
                ops.combine(av, ag, vr4, gr4, run.p, coords, None, None, grad.view(-1, d))
                ops.residuals(out, pcfg)
                h4[1].record()
                torch.cuda.synchronize()
                rec["polite_step_ms"] = h4[0].elapsed_time(h4[1])
                # pipelined K1 (engine.k1_pipelined, several ranks): every polish group's
                # block is gathered as it finishes and the K1 blocks run under the polish.
                # The other ranks' q-th groups are taken from the current positions and
                # assumed final when ours is (one GPU: their timing cannot be observed).
                if True:
                    orders = []
                    for r2 in range(n):
                        o2 = prev_sweeps.get((n, r2))
                        o2 = (torch.argsort(o2, descending=True, stable=True)
                              if o2 is not None else torch.arange(counts[r2], device="cuda"))
                        orders.append(o2.long() + offs[r2])

                    def gather(q, loc_q, src_q, orders=orders):
                        G = ngroups[0]
                        gl = G - 1 - q
                        rows = []
                        for r2 in range(n):
                            c2 = counts[r2]
                            sh = orders[r2][c2 * gl // G:c2 * (gl + 1) // G]
                            rows.append((sh[:, None] * ns + torch.arange(ns, device="cuda")
                                         ).reshape(-1))
                        src_q.copy_(run.pos4_all.index_select(0, torch.cat(rows)))

                    groups = []
                    av3 = torch.empty_like(av)
                    ag3 = torch.empty_like(ag)
                    sw3 = torch.empty_like(sw2)
                    h = [ev() for _ in range(2)]
                    torch.cuda.synchronize()
                    h[0].record()
                    _, k2ev3 = ops.project_overlap(coords, pcfg, grad, float(eta), out, pos4,
                                                   flag, fld, av3, ag3, sw3, order,
                                                   groups_out=groups)
                    ngroups = [len(groups)]
                    res = engine.k1_pipelined(ops, cfg, pos4.view(cnt, ns, 4), groups, n,
                                              gather)
                    if res is not None:
                        vr3, gr3, k1ev = res
                        for e_ in list(k2ev3) + list(k1ev):
                            torch.cuda.current_stream().wait_event(e_)
                        ops.combine(av3, ag3, vr3, gr3, run.p, coords, None, None,
                                    grad.view(-1, d))
                        ops.residuals(out, pcfg)
                        h[1].record()
                        torch.cuda.synchronize()
                        rec["pipelined_step_ms"] = h[0].elapsed_time(h[1])
                prev_sweeps[key] = sw.clone()
                per.append(rec)
            gather_ms = 16.0 * bench.N_C * ns * (n - 1) / n / 600e9 * 1e3 if n > 1 else 0.0
            tot = [p["sums_ms"] + p["project_ms"] + p["residual_ms"] for p in per]
            tot_o = [p["overlap_project_k2_ms"] + p["overlap_k1_combine_ms"] for p in per]
            tot_p = [p.get("pipelined_step_ms") for p in per]
            tot_q = [p["polite_step_ms"] for p in per]
            rows[n].append({"iteration": state["it"], "eta": eta, "max_rank_ms": max(tot),
                            "allgather_est_ms": gather_ms,
                            "step_ms": max(tot) + gather_ms,
                            "overlap_step_ms": max(tot_o) + gather_ms,
                            "pipelined_step_ms": (max(tot_p) + gather_ms
                                                  if None not in tot_p else None),
                            "polite_step_ms": max(tot_q) + gather_ms,
                            "max_sums_ms": max(p["sums_ms"] for p in per),
                            "max_project_ms": max(p["project_ms"] for p in per),
                            "ranks": per})
        # advance the real single-GPU run by this iteration
        state["eta"] = eta
        state["have"] = True
        run.step_project(pcfg, eta)
        run.residual_max(pcfg)
    # the first iteration has no previous sweep counts (shot-order polish groups); the
    # averages below skip it
    t1 = np.mean([x["step_ms"] for x in rows[1][1:]]) if 1 in rows else None
    for n in worlds:
        tn = float(np.mean([x["step_ms"] for x in rows[n][1:]]))
        to = float(np.mean([x["overlap_step_ms"] for x in rows[n][1:]]))
        tq = float(np.mean([x["polite_step_ms"] for x in rows[n][1:]]))
        tp = [x["pipelined_step_ms"] for x in rows[n][1:]]
        tp = float(np.mean(tp)) if None not in tp else None
        rec = {"config": args.config, "n_ranks": n, "groups": ops.OVERLAP_GROUPS,
               "step_ms": tn,
               "sums_ms": float(np.mean([x["max_sums_ms"] for x in rows[n][1:]])),
               "project_ms": float(np.mean([x["max_project_ms"] for x in rows[n][1:]])),
               "efficiency": (t1 / (n * tn)) if t1 else None,
               "overlap_step_ms": to,
               "overlap_efficiency": (t1 / (n * to)) if t1 else None,
               "polite_step_ms": tq,
               "polite_efficiency": (t1 / (n * tq)) if t1 else None,
               "pipelined_step_ms": tp,
               "pipelined_efficiency": (t1 / (n * tp)) if (t1 and tp) else None,
               "iterations": rows[n]}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
