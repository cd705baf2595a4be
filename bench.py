"""Benchmark: pair-interactions/s and s/iteration of the SPARKLING hot path.

Workload (BASELINE.json configs[1], "C2"): 3D, 1024 shots x 1024 samples (p = 2^20),
129^3 density grid (N = 64, "128^3"), exact attraction (north star), eps_rep = 1e-3,
eps_att = 1/(2N), full3d hardware limits, pin at N_s/2, perturbed radial init
(P = 0.25, seed 0).  One step = one optimize() iteration on the device: fused K1+K2
N-body, gradient combine + BB dots, step + K3 projection (FISTA 100 it + polish),
feasibility residuals, position all-gather.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's CPU path (the
bit-exact C port in oracle/, all host threads) on bounded row samples of the same
workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# Workloads (SURVEY 8 shapes).  The bench line is C2 (BASELINE configs[1], the config
# the metric is quoted on for one GPU); the others are selectable with --config.
WORKLOADS = {
    "c2": dict(name="C2: 3D SPARKLING 1024 shots x 1024 samples, 129^3 density grid",
               n_c=1024, n_s=1024, dims=3, grid_n=(64, 64, 64), pert=0.25,
               fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dwell=2e-6),
    "c4": dict(name="C4: full 3D SPARKLING 4096 shots x 2048 samples (8.4M), "
                    "385x385x209 density grid (384x384x208 matrix)",
               n_c=4096, n_s=2048, dims=3, grid_n=(192, 192, 104), pert=0.75,
               fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dwell=2e-6),
    "c1": dict(name="C1: 2D SPARKLING 64 shots x 512 samples, 257^2 density grid",
               n_c=64, n_s=512, dims=2, grid_n=(128, 128), pert=0.25,
               fov=0.192, matrix=64, dwell=2e-6),
    "c4t": dict(name="C4 with treecodes: full 3D SPARKLING 4096 shots x 2048 samples (8.4M), "
                     "385x385x209 density grid; repulsion backend=tree at tree_precision "
                     "1e-3 (the reference's pkg/configs/full3d.cfg), attraction treecode "
                     "at 1e-4 over the static lattice tree",
                n_c=4096, n_s=2048, dims=3, grid_n=(192, 192, 104), pert=0.75,
                fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dwell=2e-6, tree=True,
                rep_prec=1e-3, att_prec=1e-4),
    "c2t": dict(name="C2 with treecodes: 3D SPARKLING 1024 shots x 1024 samples, 129^3 "
                     "density grid; repulsion tree 1e-3, attraction treecode 1e-4",
                n_c=1024, n_s=1024, dims=3, grid_n=(64, 64, 64), pert=0.25,
                fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dwell=2e-6, tree=True,
                rep_prec=1e-3, att_prec=1e-4),
    "c3": dict(name="C3: stack-of-SPARKLING, 64 independent 2D problems of 64 shots x 512 "
                    "samples, 257^2 density grid (one device batch)",
               n_c=64, n_s=512, dims=2, grid_n=(128, 128), pert=0.25,
               fov=0.192, matrix=64, dwell=2e-6, stack=64),
}
W = dict(WORKLOADS["c2"])
EPS_REP = 1e-3


def select_workload(key: str) -> None:
    global N_C, N_S, DIMS, GRID_NS, GRID_N
    W.clear()
    W.update(WORKLOADS[key])
    W["key"] = key
    N_C, N_S, DIMS, GRID_NS = W["n_c"], W["n_s"], W["dims"], W["grid_n"]
    GRID_N = max(GRID_NS)


select_workload("c2")


def density():
    import paper_2108_02991_b200 as spk

    params = spk.DensityParams(0.25, 2.0)
    if len(set(GRID_NS)) == 1:
        return spk.discretize(params, GRID_NS[0], DIMS)
    return spk.discretize_anisotropic(params, GRID_NS, DIMS)
FLOPS = {3: (17, 19), 2: (12, 14)}  # (repulsion, attraction) flops per pair
METRIC = "pair-interactions/s"


def workload_config():
    return {"workload": W["name"] + " (exact attraction + exact repulsion + projection)",
            "n_c": N_C, "n_s": N_S, "p": N_C * N_S, "grid": [2 * n + 1 for n in GRID_NS],
            "grad_mode": "exact", "eps_rep": EPS_REP, "eps_att": 1.0 / (2 * GRID_N),
            "n_pit": 100,
            "hardware": f"G 40 mT/m, S 180 T/m/s, raster 10 us, matrix {W['matrix']}, "
                        f"fov {W['fov']} m",
            "l2": "flushed between steps (256 MiB memset outside the per-step events)"}


def hardware():
    import paper_2108_02991_b200 as spk

    return spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=W["dwell"], fov=W["fov"], matrix=W["matrix"], dims=DIMS)


def start_pattern():
    import paper_2108_02991_b200 as spk

    return spk.perturb(spk.init_radial(N_C, N_S, DIMS), W["pert"], 0)


def proj_config():
    import paper_2108_02991_b200 as spk

    lim = spk.normalized_limits(hardware())
    pin = spk.LinearConstraint(pinned_index=N_S // 2, pinned_value=np.zeros(DIMS))
    return spk.ProjectionConfig(alpha=lim.alpha, beta=lim.beta, raster_dt=1e-5, n_pit=100,
                                pin=pin)


def pairs_per_step():
    p = N_C * N_S
    g = int(np.prod([2 * n + 1 for n in GRID_NS]))
    return p, g, p * p, p * g


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- helpers
def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError:
        return {}


def fp32_peak_tflops(sm_mhz):
    # 148 SMs x 128 FP32 lanes x 2 flop (FMA) x clock
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def measured_fp32_peak():
    """FP32 TFLOP/s measured by scripts/micro/fp32_peak.cu (profiles/fp32_peak.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "fp32_peak.json")) as fh:
            d = json.load(fh)
        return float(d["fp32_tflops"]), float(d["sm_mhz"])
    except (OSError, ValueError, KeyError):
        return None, None


def sfu_pairs_per_s(mhz):
    """Measured MUFU.RSQ throughput x 148 SMs (one rsqrt per pair)."""
    per_clk = 15.87
    try:
        with open(os.path.join(REPO, "profiles", "fp32_peak.json")) as fh:
            per_clk = float(json.load(fh)["mufu_rsq_per_clk_per_sm"])
    except (OSError, ValueError, KeyError):
        pass
    return per_clk * 148 * mhz * 1e6


def committed_traffic():
    path = os.path.join(REPO, "profiles", "nbody_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(rows: int, threads: int = 0):
    """Reference CPU path (bit-exact C port of direct_sums / the weighted attraction sum
    / _project_all, OpenMP over all host threads) on bounded row samples of the workload.
    Returns pairs/s and an extrapolated s/iteration."""
    from oracle import oracle as orc
    import paper_2108_02991_b200 as spk

    pts = start_pattern().points().copy()
    rho = density()
    p, g, rep_pairs, att_pairs = pairs_per_step()
    idx = np.linspace(0, p - 1, rows).astype(np.int64)
    t0 = time.perf_counter()
    orc.direct_sums_subset(pts, idx, EPS_REP * EPS_REP, threads)
    t_rep = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.grid_sums(pts[idx], rho.grid, (1.0 / (2 * GRID_N)) ** 2, threads)
    t_att = time.perf_counter() - t0
    rate = (rows * p + rows * g) / (t_rep + t_att)
    # projection: a bounded shot sample at full size, scaled to all shots
    cfg = proj_config()
    n_sh = 16
    shots = start_pattern().coords[:n_sh]
    tau = 1.0 / spk.projection.stacked_operator_norm(N_S, N_S // 2)
    t0 = time.perf_counter()
    orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, N_S // 2, np.zeros(DIMS), 100,
                    tau, 0.1 * cfg.feas_tol, nthreads=threads)
    t_proj = (time.perf_counter() - t0) * (N_C / n_sh)
    s_per_it = rep_pairs / (rows * p / t_rep) + att_pairs / (rows * g / t_att) + t_proj
    return {"pairs_per_s": rate, "s_per_iteration": s_per_it, "t_sample": t_rep + t_att,
            "rows": rows, "proj_s_extrapolated": t_proj}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    use_dist = world > 1 or os.environ.get("SPK_BENCH_DIST") == "1"
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _native, engine
    from paper_2108_02991_b200.optimizer import _bb_step, default_eta0

    class TimedOps(engine.CudaOps):
        def __init__(self):
            super().__init__()
            self.record = False
            self.ev = []

        def sums(self, *a, **k):
            if not self.record:
                return super().sums(*a, **k)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = super().sums(*a, **k)
            e.record()
            self.ev.append((s, e))
            return out

    hw = hardware()
    cfg = spk.OptimizerConfig(n_c=N_C, n_s=N_S, dims=DIMS, n_pit=100, grad_mode="exact",
                              grid_n=GRID_N, seed=0, perturbation=W["pert"])
    rho = density()
    fld = spk.precompute_field(rho)
    pcfg = proj_config()
    ops = TimedOps()
    run = engine.ShardedRun(np.ascontiguousarray(start_pattern().coords), cfg, fld, ops=ops)
    run.project(pcfg)
    eta0 = default_eta0(run.p, EPS_REP)
    state = {"eta": eta0, "it": 0, "have": False}

    def step():
        state["it"] += 1
        att, rep, bad, dots = run.evaluate()
        if bad or not np.isfinite(att - rep):
            raise RuntimeError("non-finite during bench")
        state["eta"] = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                                eta0, cfg.fixed_step_iters)
        state["have"] = True
        run.step_project(pcfg, state["eta"])
        run.residual_max(pcfg)
        return att - rep

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    ops.record = True
    _native.reset_launch_count()
    times = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            times.append((s, e))
        torch.cuda.synchronize()
    launches = _native.launch_count()
    if use_dist:
        dist.barrier()
    total_ms = sum(s.elapsed_time(e) for s, e in times)
    nb_ms = [s.elapsed_time(e) for s, e in ops.ev]
    if use_dist:
        t = torch.tensor([total_ms, float(np.mean(nb_ms))], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, nb_mean = float(t[0]), float(t[1])
    else:
        nb_mean = float(np.mean(nb_ms))
    p, g, rep_pairs, att_pairs = pairs_per_step()
    value = (rep_pairs + att_pairs) * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel (fused K1+K2 launch on this rank)
    local_t = run.local * N_S
    f_rep, f_att = FLOPS[DIMS]
    flops = local_t * p * f_rep + local_t * g * f_att
    achieved = flops / (nb_mean / 1e3) / 1e12
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak, peak_mhz = measured_fp32_peak()
    if peak is None:
        peak, peak_mhz = fp32_peak_tflops(sm_max), sm_max
        peak_source = (f"nominal 148 SM x 128 FP32 lanes x 2 x {sm_max} MHz "
                       f"(MEASURED_PEAKS.json clock)")
    else:
        peak_source = (f"measured FFMA2 throughput {peak:.2f} TFLOP/s at {peak_mhz:.0f} MHz "
                       f"(scripts/micro/fp32_peak.cu, profiles/fp32_peak.json); "
                       f"MEASURED_PEAKS.json has no FP32 entry")
    clocks = clk.summary()
    # hardware-bound time of the launch: repulsion pairs at the FP32 roofline (f_rep flops
    # per pair), attraction pairs at the measured SFU rate (the lattice kernel spends 6
    # FP32 lane-ops + 1 MUFU per pair, so the SFU binds, profiles/fp32_peak.json)
    sfu_rate = sfu_pairs_per_s(peak_mhz)
    bound_ms = (local_t * p / (peak * 1e12 / f_rep) + local_t * g / sfu_rate) * 1e3

    # end-to-end through the public drop-in API with host buffers
    if args.no_e2e:
        e2e = None
    elif not use_dist:
        e2e = run_e2e(args, spk, fld, pcfg) if rank == 0 else None
    else:
        e2e = run_e2e_sharded(args, run, step, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "s_per_iteration": total_ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
            "config": workload_config() | {"parallelism": f"shots sharded over {world} GPU(s)"},
            "roofline": {"bound": "fp32+sfu", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_at_measured_clock": (
                             achieved / (peak * clocks["sm_mhz"] / peak_mhz)
                             if clocks.get("sm_mhz") else None),
                         "traffic": committed_traffic(),
                         "kernel": "nbody_kernel (fused K1+K2) + finalize",
                         "flops_per_pair": {"repulsion": f_rep, "attraction": f_att},
                         "launch_ms": nb_mean,
                         "peak_source": peak_source,
                         "hw_bound_ms": bound_ms,
                         "frac_of_hw_bound": bound_ms / nb_mean,
                         "hw_bound_note": "repulsion pairs at the FP32 peak / 17 flops, "
                                          "attraction pairs at the measured MUFU.RSQ rate "
                                          f"({sfu_rate:.3g}/s): the lattice kernel does fewer "
                                          "than the algorithmic 19 flops per pair, so "
                                          "'frac' (algorithmic flops / FP32 peak) can "
                                          "approach 1 while frac_of_hw_bound stays honest"},
            "clocks": clocks,
            "gpu_launches": launches,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_reference_sample(args.cpu_rows)
            line["cpu_baseline"] = {
                "value": cb["pairs_per_s"], "unit": "pairs/s", "cores": os.cpu_count(),
                "kind": "port", "cpu": cpu_model(),
                "sample": f"{cb['rows']} target rows x all p={p} sources (repulsion) + "
                          f"{cb['rows']} rows x all {g} grid cells (attraction), fp64, "
                          f"{cb['t_sample']:.1f} s; projection 16 shots scaled to {N_C}",
                "s_per_iteration_extrapolated": cb["s_per_iteration"]}
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def run_tree(args):
    """Treecode workloads (c2t, c4t): s/iteration of the full optimizer iteration with
    RepulsionConfig(backend="tree") and the treecode attraction, through ShardedRun."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    use_dist = world > 1 or os.environ.get("SPK_BENCH_DIST") == "1"
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _native, engine
    from paper_2108_02991_b200.optimizer import _bb_step, default_eta0

    hw = hardware()
    cfg = spk.OptimizerConfig(n_c=N_C, n_s=N_S, dims=DIMS, n_pit=100, grad_mode="exact",
                              grid_n=GRID_N, seed=0, perturbation=W["pert"],
                              attraction_tree_precision=W["att_prec"],
                              repulsion=spk.RepulsionConfig(backend="tree",
                                                            tree_precision=W["rep_prec"]))
    fld = spk.precompute_field(density())
    pcfg = proj_config()
    t0 = time.perf_counter()
    fld.source_tree()
    from paper_2108_02991_b200 import tree as _tree
    fld.source_tree().static_proxies(_tree.auto_params(W["att_prec"], DIMS)[0])
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    run = engine.ShardedRun(np.ascontiguousarray(start_pattern().coords), cfg, fld)
    run.project(pcfg)
    eta0 = default_eta0(run.p, EPS_REP)
    state = {"eta": eta0, "it": 0, "have": False}

    def step():
        state["it"] += 1
        att, rep, bad, dots = run.evaluate()
        if bad or not np.isfinite(att - rep):
            raise RuntimeError("non-finite during bench")
        state["eta"] = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                                eta0, cfg.fixed_step_iters)
        state["have"] = True
        run.step_project(pcfg, state["eta"])
        run.residual_max(pcfg)
        return att - rep

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    _native.reset_launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            times.append((s, e))
        torch.cuda.synchronize()
    launches = _native.launch_count()
    total_ms = sum(s.elapsed_time(e) for s, e in times)
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    p, g, rep_pairs, att_pairs = pairs_per_step()
    s_it = total_ms / args.steps / 1e3
    if rank == 0:
        line = {
            "metric": "s/iteration", "value": s_it, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s_it * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
            "config": workload_config() | {
                "parallelism": f"shots sharded over {world} GPU(s)",
                "workload": W["name"], "repulsion": f"tree, tree_precision {W['rep_prec']}",
                "attraction": f"treecode, precision {W['att_prec']}"},
            "equivalent_direct_pairs_per_s": (rep_pairs + att_pairs) / s_it,
            "setup_s": {"lattice_tree_and_proxies": t_setup},
            "roofline": None,
            "roofline_note": "treecode lists vary per iteration; the kernel roofline is "
                             "reported on the exact C2 line",
            "clocks": clk.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def run_stack(args):
    """C3: one stacked optimize iteration of G independent problems per step (1 GPU)."""
    import torch

    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _native, stack
    from paper_2108_02991_b200.optimizer import _bb_step, default_eta0

    torch.cuda.set_device(0)
    G = W["stack"]
    cfg = spk.OptimizerConfig(n_c=N_C, n_s=N_S, dims=DIMS, n_pit=100, grad_mode="exact",
                              grid_n=GRID_N, seed=0, perturbation=W["pert"])
    fld = spk.precompute_field(density())
    pcfg = proj_config()
    base = spk.init_radial(N_C, N_S, DIMS)
    starts = np.stack([spk.perturb(base, W["pert"], q).coords for q in range(G)])
    run = stack.StackedRun(starts, cfg, fld)
    run.project(pcfg)
    eta0 = default_eta0(run.p, EPS_REP)
    st = {"etas": np.full(G, eta0), "it": 0, "have": False}
    nb_events = []
    orig_call = _native.call

    def timed_call(name, *a):
        if name == "spk_fused_sums_batched" and st.get("record"):
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            orig_call(name, *a)
            e0.record()
            nb_events.append((s0, e0))
            return
        orig_call(name, *a)

    _native.call = timed_call

    def step():
        st["it"] += 1
        att, rep, bad, dkdg, dgdg = run.evaluate()
        if bad.any() or not np.isfinite(att - rep).all():
            raise RuntimeError("non-finite during bench")
        for q in range(G):
            st["etas"][q] = _bb_step(st["it"], st["etas"][q], dkdg[q], dgdg[q], st["have"],
                                     eta0, cfg.fixed_step_iters)
        st["have"] = True
        run.step_project(pcfg, st["etas"])
        run.residual_max(pcfg)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st["record"] = True
    _native.reset_launch_count()
    times = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            step()
            e0.record()
            times.append((s0, e0))
        torch.cuda.synchronize()
    _native.call = orig_call
    total_ms = sum(a.elapsed_time(b) for a, b in times)
    nb_ms = float(np.mean([a.elapsed_time(b) for a, b in nb_events]))
    p, g, rep_pairs, att_pairs = pairs_per_step()
    pairs = G * (rep_pairs + att_pairs)
    f_rep, f_att = FLOPS[DIMS]
    peak, peak_mhz = measured_fp32_peak() if measured_fp32_peak()[0] else (
        fp32_peak_tflops(1965.0), 1965.0)
    achieved = G * (rep_pairs * f_rep + att_pairs * f_att) / (nb_ms / 1e3) / 1e12
    bound_ms = G * (rep_pairs / (peak * 1e12 / f_rep) + att_pairs / sfu_pairs_per_s(peak_mhz)) * 1e3
    line = {
        "metric": METRIC, "value": pairs * args.steps / (total_ms / 1e3), "unit": "pairs/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "s_per_iteration": total_ms / args.steps / 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
        "config": workload_config() | {"stack": G, "parallelism": "one device batch"},
        "roofline": {"bound": "fp32+sfu", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "launch_ms": nb_ms,
                     "hw_bound_ms": bound_ms, "frac_of_hw_bound": bound_ms / nb_ms,
                     "kernel": "nbody_kernel batched (spk_fused_sums_batched)"},
        "clocks": clk.summary(), "gpu_launches": _native.launch_count(),
    }
    print(json.dumps(line), flush=True)


def run_e2e_sharded(args, run, step, world):
    """N > 1: the sharded optimize iteration with this rank's shots copied H2D from pinned
    host memory before, and the projected shots + scalars copied D2H after, every step
    (device-timed per step, max over ranks)."""
    import torch
    import torch.distributed as dist

    host_in = torch.empty(run.coords.shape, dtype=torch.float64, pin_memory=True)
    host_in.copy_(run.coords)
    host_out = torch.empty_like(host_in, pin_memory=True)
    steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    dist.barrier()
    total = 0.0
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run.coords.copy_(host_in, non_blocking=True)
        step()
        host_out.copy_(run.coords, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        total += s.elapsed_time(e)
        host_in.copy_(host_out)
    t = torch.tensor([total], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    p, g, rep_pairs, att_pairs = pairs_per_step()
    nbytes = host_in.numel() * 8
    return {"value": (rep_pairs + att_pairs) * steps / (float(t[0]) / 1e3), "unit": "pairs/s",
            "s_per_iteration": float(t[0]) / 1e3 / steps, "steps": steps,
            "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world + 48,
            "api": "sharded optimize iteration (engine.ShardedRun) with per-step pinned "
                   "H2D of every rank's shots and D2H of the projected shots"}


def run_e2e(args, spk, fld, pcfg):
    """The reference's loop body (optimizer.py:301-344) through the public API with numpy
    host arrays; every call copies its inputs H2D and results D2H."""
    import torch
    from paper_2108_02991_b200.optimizer import default_eta0, step_size

    pattern = spk.project_pattern(start_pattern(), pcfg)
    rcfg = spk.RepulsionConfig(kernel_eps=EPS_REP)
    eta0 = default_eta0(pattern.n_samples, EPS_REP)
    prev_c = prev_g = None
    eta = eta0
    steps = max(1, min(args.steps, args.e2e_steps))
    bi = bo = 0
    nbytes = pattern.coords.nbytes
    for it in range(1, steps + 2):  # first iteration is warm-up
        if it == 2:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        att = spk.eval_attraction(pattern, fld, "exact")
        rep_cost, rep_grad = spk.eval_repulsion(pattern, rcfg)
        grad = (att.grad - rep_grad).reshape(pattern.coords.shape)
        dk = None if prev_c is None else pattern.coords - prev_c
        dg = None if prev_g is None else grad - prev_g
        eta = step_size(it, eta, dk, dg, eta0, 20)
        prev_c, prev_g = pattern.coords.copy(), grad
        pattern = spk.project_pattern(spk.SamplingPattern(pattern.coords - eta * grad), pcfg)
        spk.feasibility_residuals(pattern, pcfg)
        if it >= 2:
            bi += 4 * nbytes          # coords to att, rep, project, residuals
            bo += 3 * nbytes + 2 * pattern.n_samples * 8 + 40  # grads, vals, coords, resid
    dt = time.perf_counter() - t0
    p, g, rep_pairs, att_pairs = pairs_per_step()
    return {"value": (rep_pairs + att_pairs) * steps / dt, "unit": "pairs/s",
            "s_per_iteration": dt / steps, "steps": steps,
            "h2d_bytes_per_step": bi // steps, "d2h_bytes_per_step": bo // steps,
            "api": "eval_attraction(exact) + eval_repulsion + step_size + project_pattern + "
                   "feasibility_residuals on numpy host arrays"}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.build()
    threads = orc.max_threads()
    samples = []
    for i in range(args.warmup + args.steps):
        cb = cpu_reference_sample(args.ref_rows, threads)
        if i >= args.warmup:
            samples.append(cb)
    rate = float(np.mean([c["pairs_per_s"] for c in samples]))
    p, g, _, _ = pairs_per_step()
    s_it = float(np.mean([c["s_per_iteration"] for c in samples]))
    line = {
        "metric": METRIC, "value": rate, "unit": "pairs/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s_it * 1e3, "s_per_iteration": s_it, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config() | {"parallelism": "host CPU threads"},
        "cpu_baseline": {"value": rate, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"per step {args.ref_rows} target rows x all {p} sources "
                                   f"+ {args.ref_rows} rows x {g} grid cells, fp64, plus 16 "
                                   f"shots of projection; s/iteration extrapolated"},
        "e2e": {"value": rate, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=16384)
    ap.add_argument("--ref-rows", type=int, default=2048)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    select_workload(args.config)
    if args.impl == "reference":
        run_reference(args)
    elif W.get("stack"):
        run_stack(args)
    elif W.get("tree"):
        run_tree(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
