"""Record in-loop shots for bench.py's CPU projection sample (run on a B200).

For each bench workload (c2, c4) run the device optimizer loop exactly as bench.py does
(level-start projection, then optimizer iterations) and, at iteration 6 (after the
driver's 5 warm-up steps), save the stepped shots coords - eta * grad of a strided subset
of shots BEFORE projection: the input the reference's project_pattern receives at that
iteration.  Written to bench_data/inloop_<key>.npz.

    python scripts/make_inloop_shots.py [c2] [c4]
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import engine  # noqa: E402

ITERATION = 6
N_SHOTS = {"c2": 16, "c4": 8}


def record(key):
    bench.select_workload(key)
    cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, n_pit=100,
                              grad_mode="exact", grid_n=bench.GRID_N, seed=0,
                              perturbation=bench.W["pert"])
    if key == "c4":
        # the exact C4 iteration is ~85 s; the treecode backends (tree 1e-3 / 1e-4) give
        # the same in-loop regime in ~4 s per iteration
        cfg = spk.OptimizerConfig(n_c=bench.N_C, n_s=bench.N_S, dims=bench.DIMS, n_pit=100,
                                  grad_mode="exact", grid_n=bench.GRID_N, seed=0,
                                  perturbation=bench.W["pert"],
                                  attraction_tree_precision=1e-4,
                                  repulsion=spk.RepulsionConfig(backend="tree",
                                                                tree_precision=1e-3))
    fld = spk.precompute_field(bench.density())
    run = engine.ShardedRun(np.ascontiguousarray(bench.start_pattern().coords), cfg, fld)
    pcfg = bench.proj_config()
    run.project(pcfg)
    step, state = bench.optimizer_step(run, cfg)
    for _ in range(ITERATION - 1):
        step()
    # iteration ITERATION up to the step: evaluate + step size, then stepped shots
    from paper_2108_02991_b200.optimizer import _bb_step

    state["it"] += 1
    att, rep, bad, dots = run.evaluate()
    eta = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                   state["eta0"], cfg.fixed_step_iters)
    stepped = (run.coords - eta * run.grad).cpu().numpy()
    pick = np.linspace(0, bench.N_C - 1, N_SHOTS[key]).astype(int)
    out = os.path.join(REPO, "bench_data", f"inloop_{key}.npz")
    np.savez_compressed(out, shots=np.ascontiguousarray(stepped[pick]), shot_index=pick,
                        iteration=np.int64(ITERATION), eta=np.float64(eta))
    # sweep counts of these shots on the device, for the record
    res = spk.project_pattern(spk.SamplingPattern(stepped[pick]), pcfg)
    print(key, out, "eta", eta, "feasible", spk.feasibility_residuals(res, pcfg)["max"])
    del run, fld
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for k in sys.argv[1:] or ["c2", "c4"]:
        record(k)
