"""A/B timings for the round-2 kernel changes (device time, CUDA events):
  polish  -- single shot / 1024 shots at 1600 fixed sweeps, and the real in-loop C2
             projection (5 warm-up optimizer iterations, then 3 timed step+projections)
  nbody   -- fused K1+K2 at C2 and on a C4 target subset (1/16 of the targets against all
             sources and the whole lattice)
    python scripts/ab_r02.py polish|nbody
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.getcwd())

import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device, _native, engine  # noqa: E402


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def polish():
    bench.select_workload("c2")
    cfg = bench.proj_config()
    base = bench.start_pattern().coords
    for n in (1, 1024):
        shots = _device.h2d(np.ascontiguousarray(base[:n]))
        out = torch.empty_like(shots)
        ws = _device.workspace(_native.query("spk_project_workspace_bytes", n, 1024, 3, 0), "p")
        pv = _native.f64_array([0, 0, 0])

        def go():
            _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(),
                         n, 1024, 3, cfg.speed_bound, cfg.accel_bound, 512, pv, 1, 0.048, 0,
                         -1.0, 1600, None, None, None, None, ws.data_ptr(), ws.numel(),
                         _device.stream())
        print(f"polish shots={n} 1600 sweeps: {timed(go):.2f} ms", flush=True)
    ocfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=3, grad_mode="exact",
                               grid_n=bench.GRID_N, seed=0, perturbation=bench.W["pert"])
    fld = spk.precompute_field(bench.density())
    run = engine.ShardedRun(np.ascontiguousarray(base), ocfg, fld)
    run.project(cfg)
    step, state = bench.optimizer_step(run, ocfg)
    for _ in range(5):
        step()
    from paper_2108_02991_b200.optimizer import _bb_step
    ms = []
    for _ in range(3):
        state["it"] += 1
        att, rep, bad, dots = run.evaluate()
        eta = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                       state["eta0"], ocfg.fixed_step_iters)
        state["eta"], state["have"] = eta, True
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run.step_project(cfg, eta)
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
        run.residual_max(cfg)
    print(f"in-loop C2 step+projection (iterations 6-8): {[round(x, 1) for x in ms]} "
          f"mean {np.mean(ms):.1f} ms", flush=True)


def nbody():
    for key, frac in (("c2", 1), ("c4", 16)):
        bench.select_workload(key)
        cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=3, grad_mode="exact",
                                  grid_n=bench.GRID_N, seed=0, perturbation=bench.W["pert"])
        fld = spk.precompute_field(bench.density())
        coords = _device.h2d(np.ascontiguousarray(bench.start_pattern().coords))
        pos4 = _device.pack_positions(coords)
        n_t = pos4.shape[0] // frac
        tgt = pos4[:n_t]
        ops = engine.CudaOps()
        ops.sums(tgt, pos4, coords[:n_t // bench.N_S], fld, cfg)
        for rep in range(2):
            t = timed(lambda: ops.sums(tgt, pos4, coords[:n_t // bench.N_S], fld, cfg), 2)
            print(f"{key} (targets {n_t}) fused N-body: {t:.1f} ms", flush=True)
        del fld, pos4, coords
        _device.release_workspaces()


if __name__ == "__main__":
    {"polish": polish, "nbody": nbody}[sys.argv[1]]()
