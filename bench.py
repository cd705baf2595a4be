"""Benchmark: pair-interactions/s and s/iteration of the SPARKLING hot path.

Headline workload (BASELINE.json configs[1], "C2"): 3D, 1024 shots x 1024 samples
(p = 2^20), 129^3 density grid (N = 64, "128^3"), exact attraction (north star),
eps_rep = 1e-3, eps_att = 1/(2N), full3d hardware limits, pin at N_s/2, perturbed radial
init (P = 0.25, seed 0).  One step = one optimize() iteration on the device: fused K1+K2
N-body, gradient combine + BB dots, step + K3 projection (FISTA 100 it + polish),
feasibility residuals, position all-gather.

The metric is quoted at ~10^7 samples (configs[3], "C4": 4096 x 2048), so the default run
appends two sub-records measured in the same invocation: ``c4`` (exact sums, as the
headline) and ``c4t`` (the reference's full3d.cfg backends: repulsion treecode 1e-3,
attraction treecode 1e-4).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` is authoritative: without torchrun's WORLD_SIZE and N > 1 the script
re-launches itself under ``torch.distributed.run`` with N ranks (failing loudly when the
node has fewer than N GPUs); under torchrun WORLD_SIZE must equal N.  Prints ONE JSON
line (rank 0).  ``--impl reference`` times the reference's CPU path (the bit-exact C
port in oracle/, all host threads) on bounded samples of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# Workloads (SURVEY 8 shapes).  The bench line is C2 (BASELINE configs[1], the largest
# config whose exact step fits the per-run budget at 20+5 steps); C4 / C4t ride along as
# sub-records; the others are selectable with --config.
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
# sub-records of the default (c2) run: key -> (timed steps, warm-up steps); None = the
# run's own --steps / --warmup
SUBRECORDS = {"c4": (2, 3), "c4t": (None, None)}
W = dict(WORKLOADS["c2"])
EPS_REP = 1e-3
FLOPS = {3: (17, 19), 2: (12, 14)}  # (repulsion, attraction) algorithmic flops per pair
# executed FP32 lane-ops per pair (csrc/nbody.cu): positions 3D 3 FADD + 3 FFMA (r2) +
# 4 FFMA (value, gradient); 2D 2 + 2 + 3; lattice 6 (dl, r2, w/h, value, S, g_last) in
# both; one MUFU.RSQ per pair everywhere
LANE_OPS = {3: (10, 6), 2: (7, 6)}
# FMA-pipe cost of one rsqrt evaluated without the SFU (integer seed + 2 Newton steps):
# 8 lane-ops; used for the balanced-pipe bound below
RSQRT_FMA_LANE_OPS = 8
METRIC = "pair-interactions/s"


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


def workload_config():
    """The workload keys, identical in both arms (the parallelism is a top-level key)."""
    cfg = {"workload": W["name"] + (" (exact attraction + exact repulsion + projection)"
                                    if not W.get("tree") else ""),
           "n_c": N_C, "n_s": N_S, "p": N_C * N_S, "grid": [2 * n + 1 for n in GRID_NS],
           "grad_mode": "exact", "eps_rep": EPS_REP, "eps_att": 1.0 / (2 * GRID_N),
           "n_pit": 100,
           "hardware": f"G 40 mT/m, S 180 T/m/s, raster 10 us, matrix {W['matrix']}, "
                       f"fov {W['fov']} m",
           "l2": "flushed between steps (256 MiB memset outside the per-step events)"}
    if W.get("tree"):
        cfg["repulsion"] = f"tree, tree_precision {W['rep_prec']}"
        cfg["attraction"] = f"treecode, precision {W['att_prec']}"
    if W.get("stack"):
        cfg["stack"] = W["stack"]
    return cfg


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
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def measured_fp32_peak():
    """(FP32 TFLOP/s, MUFU.RSQ per clk per SM, clock MHz) measured by
    scripts/micro/fp32_peak.cu on a B200 (profiles/fp32_peak.json); MEASURED_PEAKS.json
    has HBM and bf16 entries only."""
    try:
        with open(os.path.join(REPO, "profiles", "fp32_peak.json")) as fh:
            d = json.load(fh)
        return (float(d["fp32_tflops"]), float(d.get("mufu_rsq_per_clk_per_sm", 15.87)),
                float(d["sm_mhz"]), "measured (scripts/micro/fp32_peak.cu, "
                                    "profiles/fp32_peak.json)")
    except (OSError, ValueError, KeyError):
        mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
        return (148 * 128 * 2 * mhz * 1e6 / 1e12, 16.0, mhz,
                "nominal 148 SM x 128 FP32 lanes x 2 and 16 MUFU/clk/SM at the max clock")


def committed_traffic(key: str):
    """DRAM bytes per fused N-body launch for this workload from an ncu capture
    (profiles/nbody_traffic.json, keyed by workload), or None when not captured."""
    try:
        with open(os.path.join(REPO, "profiles", "nbody_traffic.json")) as fh:
            d = json.load(fh)
    except (OSError, ValueError):
        return None, None
    rec = d.get("workloads", {}).get(key)
    if rec is None:
        return None, None
    return rec.get("dram_bytes_per_launch"), rec.get("source")


def co_issue_ceiling(key):
    """Measured FFMA2 + MUFU co-issue ceiling of this workload's instruction mix
    (profiles/mix_peak.json, scripts/micro/mix_peak.cu), or None if not measured."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "mix_peak.json")) as fh:
            return json.load(fh)["co_issue_ceiling"].get(key)
    except (OSError, ValueError, KeyError):
        return None


def nbody_roofline(key, dims, rep_pairs, att_pairs, launch_ms, clocks):
    """Roofline of the fused N-body launch.

    The path is rsqrt-bound: each pair costs FP32 lane-ops on the FMA pipe and
    one MUFU.RSQ on the SFU.  The bound is the FP32 + SFU time of the EXECUTED mix: FMA
    work L = rep * lane_rep + att * lane_att lane-ops at the measured FP32 rate and SFU work
    M = rep + att rsqrts at the measured MUFU rate, the two pipes overlapping perfectly:
    T = max(L / fma_rate, M / sfu_rate) (``hw_bound_ms``).  ``peak`` is the algorithmic
    TFLOP/s the launch would reach at that bound (17/19 flops per pair), so
    frac = achieved / peak = T / launch time <= 1.  Secondary: the balanced bound if the
    hardware also moved x rsqrts to the FMA pipe at RSQRT_FMA_LANE_OPS each,
    min_x max((L + c x)/fma_rate, (M - x)/sfu_rate) -- that offload measured slower in this
    kernel (profiles/r02_ab_nbody_fma_rsqrt.txt), so it is a ceiling, not a target."""
    f_rep, f_att = FLOPS[dims]
    l_rep, l_att = LANE_OPS[dims]
    tflops, mufu_clk, mhz, src = measured_fp32_peak()
    fma_rate = tflops * 1e12 / 2.0            # lane-ops/s
    sfu_rate = mufu_clk * 148 * mhz * 1e6     # rsqrt/s
    lanes = rep_pairs * l_rep + att_pairs * l_att
    mufu = rep_pairs + att_pairs
    c = RSQRT_FMA_LANE_OPS
    x = max(0.0, min(mufu, (mufu * fma_rate / sfu_rate - lanes) / (c + fma_rate / sfu_rate)))
    balanced_s = max((lanes + c * x) / fma_rate, (mufu - x) / sfu_rate)
    bound_s = max(lanes / fma_rate, mufu / sfu_rate)
    flops = rep_pairs * f_rep + att_pairs * f_att
    achieved = flops / (launch_ms / 1e3) / 1e12
    peak = flops / bound_s / 1e12
    traffic, tsrc = committed_traffic(key)
    ceiling = co_issue_ceiling(key)
    sm = clocks.get("sm_mhz") if clocks else None
    return {
        "bound": "fp32+sfu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak,
        "frac_at_measured_clock": (achieved / (peak * sm / mhz)) if sm else None,
        "traffic": traffic,
        "traffic_source": tsrc if traffic is not None else
        "no ncu DRAM capture for this workload (the kernel reads ~0 bytes per pair)",
        "kernel": "nbody_kernel (fused K1+K2) + finalize", "launch_ms": launch_ms,
        "hw_bound_ms": bound_s * 1e3,
        "co_issue_ceiling": ceiling,
        "frac_of_co_issue_ceiling": (bound_s / (launch_ms / 1e3) / ceiling) if ceiling else None,
        "frac_of_balanced_offload_bound": balanced_s / (launch_ms / 1e3),
        "balanced_offload_bound_ms": balanced_s * 1e3,
        "algorithmic_tflops_vs_fp32_peak": achieved / tflops,
        "peak_source": f"{src}: FP32 {tflops:.2f} TFLOP/s and MUFU.RSQ {mufu_clk:.2f}/clk/SM "
                       f"at {mhz:.0f} MHz",
        "work": {"repulsion_pairs": rep_pairs, "attraction_pairs": att_pairs,
                 "flops_per_pair": {"repulsion": f_rep, "attraction": f_att},
                 "lane_ops_per_pair": {"repulsion": l_rep, "attraction": l_att},
                 "mufu_per_pair": 1, "rsqrt_on_fma_lane_ops": c},
        "note": "peak = algorithmic flops at the FP32+SFU bound of the executed mix "
                "(max of FMA-pipe and SFU time, hw_bound_ms); frac = hw_bound_ms / "
                "launch_ms.  frac_of_balanced_offload_bound also lets rsqrts move to the "
                "FMA pipe (measured slower here).  co_issue_ceiling = the fraction of "
                "that bound a dependency-free FFMA2 + MUFU stream of the same mix reaches "
                "on this GPU (profiles/mix_peak.json).  algorithmic_tflops_vs_fp32_peak is "
                "secondary: the lattice segment runs fewer lane-ops than its 19 "
                "algorithmic flops, so it can exceed 1.",
    }


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def inloop_shots():
    """In-loop shots for the CPU projection sample: the stepped (pre-projection) shots of
    optimize iteration 6 of this workload, recorded on a B200 by
    scripts/make_inloop_shots.py (bench_data/).  Fresh-init shots need several times more
    polish sweeps than in-loop ones and would inflate the CPU time."""
    key = "c4" if W["key"].startswith("c4") else W["key"]
    path = os.path.join(REPO, "bench_data", f"inloop_{key}.npz")
    if os.path.exists(path):
        d = np.load(path)
        return d["shots"], f"{d['shots'].shape[0]} in-loop shots (optimize iteration " \
                           f"{int(d['iteration'])}, bench_data/inloop_{key}.npz)"
    return start_pattern().coords[:16], "16 fresh-init shots (no in-loop fixture)"


def cpu_reference_sample(rows: int, threads: int = 0):
    """Reference CPU path (bit-exact C port of direct_sums / the weighted attraction sum
    / _project_all, OpenMP over the host threads) on bounded samples of the workload:
    ``rows`` target rows against all sources, and a sample of in-loop shots through the
    projection.  Returns pairs/s and an extrapolated s/iteration."""
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
    cfg = proj_config()
    shots, what = inloop_shots()
    tau = 1.0 / spk.projection.stacked_operator_norm(N_S, N_S // 2)
    t0 = time.perf_counter()
    orc.project_all(shots, cfg.speed_bound, cfg.accel_bound, N_S // 2, np.zeros(DIMS), 100,
                    tau, 0.1 * cfg.feas_tol, nthreads=threads)
    t_proj = (time.perf_counter() - t0) * (N_C / shots.shape[0])
    s_per_it = rep_pairs / (rows * p / t_rep) + att_pairs / (rows * g / t_att) + t_proj
    return {"pairs_per_s": rate, "s_per_iteration": s_per_it, "t_sample": t_rep + t_att,
            "rows": rows, "proj_s_extrapolated": t_proj, "proj_sample": what}


def cpu_baseline_record(rows):
    cb = cpu_reference_sample(rows)
    p, g, _, _ = pairs_per_step()
    return {"value": cb["pairs_per_s"], "unit": "pairs/s", "cores": os.cpu_count(),
            "kind": "port", "cpu": cpu_model(),
            "sample": f"{cb['rows']} target rows x all p={p} sources (repulsion) + "
                      f"{cb['rows']} rows x all {g} grid cells (attraction), fp64, "
                      f"{cb['t_sample']:.1f} s; projection: {cb['proj_sample']}, scaled to "
                      f"{N_C} shots",
            "s_per_iteration_extrapolated": cb["s_per_iteration"],
            "proj_s_extrapolated": cb["proj_s_extrapolated"]}


# ---------------------------------------------------------------- process group
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def ensure_world(args) -> None:
    """Make ``--gpus N`` authoritative for our arm (one process per GPU)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank "
                     f"per GPU (torchrun --nproc-per-node {args.gpus})")
        if args.gpus > 1:
            # rank 0's NCCL INIT lines show the N-rank communicator; the other ranks stay
            # quiet so that nothing can follow rank 0's JSON line on the shared stdout
            if os.environ.get("RANK", "0") == "0":
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            else:
                os.environ["NCCL_DEBUG"] = "WARN"
        return
    if args.gpus <= 1:
        return
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} requested but this node has {have} CUDA "
                 f"device(s); refusing to report a {args.gpus}-GPU number")
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr,
          flush=True)
    os.execve(sys.executable, cmd, env)


class Ctx:
    """This process's rank / device / process group."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # test hooks (tests/test_gpu_multirank.py): every rank on one device over gloo, a
        # functional check of the N-rank path on a one-GPU box -- never a measurement
        backend = os.environ.get("SPK_BENCH_BACKEND", "nccl")
        if "SPK_BENCH_DEVICE" in os.environ:
            self.local = int(os.environ["SPK_BENCH_DEVICE"])
        torch.cuda.set_device(self.local)
        self.dist = self.world > 1 or os.environ.get("SPK_BENCH_DIST") == "1"
        if self.dist:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(backend)

    def barrier(self):
        if self.dist:
            import torch.distributed as dist

            dist.barrier()

    def max(self, *vals):
        if not self.dist:
            return vals
        import torch
        import torch.distributed as dist

        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return tuple(float(x) for x in t.tolist())

    def close(self):
        if self.dist:
            import torch.distributed as dist

            dist.destroy_process_group()


def timed_loop(ctx, step, steps, warmup, on_record=None):
    """W untimed warm-up steps, then K device-timed steps (CUDA events on the launching
    stream, L2 flushed before each step outside the events), barrier + synchronize on
    both sides.  Returns (total_ms max over ranks, clocks, our kernel launches)."""
    import torch
    from paper_2108_02991_b200 import _native

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.barrier()
    if on_record:
        on_record()
    _native.reset_launch_count()
    times = []
    with ClockSampler(ctx.local) as clk:
        torch.cuda.synchronize()
        for _ in range(steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            times.append((s, e))
        torch.cuda.synchronize()
    launches = _native.launch_count()
    ctx.barrier()
    total_ms = sum(s.elapsed_time(e) for s, e in times)
    del flush
    return total_ms, clk.summary(), launches


def optimizer_step(run, cfg):
    """One optimizer iteration on the device (optimizer.py:301-344 through ShardedRun)."""
    from paper_2108_02991_b200.optimizer import _bb_step, default_eta0

    state = {"eta0": default_eta0(run.p, EPS_REP), "it": 0, "have": False}
    state["eta"] = state["eta0"]
    pcfg = proj_config()

    def step():
        state["it"] += 1
        att, rep, bad, dots = run.evaluate()
        if bad or not np.isfinite(att - rep):
            raise RuntimeError("non-finite during bench")
        state["eta"] = _bb_step(state["it"], state["eta"], dots[0], dots[1], state["have"],
                                state["eta0"], cfg.fixed_step_iters)
        state["have"] = True
        run.step_project(pcfg, state["eta"])
        run.residual_max(pcfg)
        return att - rep

    return step, state


# ---------------------------------------------------------------- our arm: exact sums
def measure_exact(args, ctx, steps, warmup, with_e2e, with_cpu):
    import torch

    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import engine

    cfg = spk.OptimizerConfig(n_c=N_C, n_s=N_S, dims=DIMS, n_pit=100, grad_mode="exact",
                              grid_n=GRID_N, seed=0, perturbation=W["pert"])
    fld = spk.precompute_field(density())
    pcfg = proj_config()
    class TimedOps(engine.CudaOps):
        """Records CUDA events around fused N-body launches (launching stream)."""

        record = False
        ev = []

        def sums(self, *a, **k):
            if not self.record:
                return super().sums(*a, **k)
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            out = super().sums(*a, **k)
            e0.record()
            self.ev.append((s0, e0))
            return out

    ops = TimedOps()
    ops.ev = []
    run = engine.ShardedRun(np.ascontiguousarray(start_pattern().coords), cfg, fld, ops=ops)
    run.project(pcfg)
    step, _ = optimizer_step(run, cfg)
    overlapped = []

    def counted_step():
        out = step()
        overlapped.append(run.att_pre is not None)
        return out

    def on_record():
        ops.record = True

    total_ms, clocks, launches = timed_loop(ctx, counted_step, steps, warmup, on_record)
    n_ovl = sum(overlapped[warmup:])
    # roofline of the N-body kernel: the fused K1 + K2 launch, CUDA events on its stream.
    # When the schedule split every timed step into K1 + per-group K2 under the polish
    # (ShardedRun.overlap), the fused launch is timed alone on the final positions.
    timed = list(ops.ev)
    if not timed:
        tgt = run.pos4_local[:run.local * N_S]
        for _ in range(3):
            ops.sums(tgt, run.pos4_all, run.coords, fld, cfg)
        timed = ops.ev[1:]
    torch.cuda.synchronize()
    nb_mean = float(np.mean([a.elapsed_time(b) for a, b in timed]))
    total_ms, nb_mean = ctx.max(total_ms, nb_mean)
    p, g, rep_pairs, att_pairs = pairs_per_step()
    local_t = run.local * N_S
    rec = {
        "metric": METRIC, "value": (rep_pairs + att_pairs) * steps / (total_ms / 1e3),
        "unit": "pairs/s", "n_gpus": ctx.world, "steps": steps, "warmup": warmup,
        "ms_per_step": total_ms / steps, "s_per_iteration": total_ms / steps / 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
        "config": workload_config(),
        "parallelism": f"shots sharded over {ctx.world} GPU(s)",
        "roofline": nbody_roofline(W["key"], DIMS, local_t * p, local_t * g, nb_mean, clocks),
        "schedule": {"timed_steps_with_k2_under_polish": n_ovl,
                     "note": "steps whose lattice sums (K2) ran per polish group on side "
                             "streams under the slower shots' polish, followed by K1 alone "
                             "(engine.ShardedRun.overlap); the roofline times the fused "
                             "K1 + K2 launch alone"},
        "clocks": clocks, "gpu_launches": launches,
    }
    del run, ops
    torch.cuda.empty_cache()
    if with_e2e:
        rec["e2e"] = run_e2e_step_api(ctx, cfg, fld, max(1, min(steps, args.e2e_steps)))
        if not ctx.dist:
            rec["e2e_numpy_api"] = run_e2e(args, spk, fld, pcfg, steps)
    del fld
    if with_cpu and ctx.world == 1 and ctx.rank == 0:
        rec["cpu_baseline"] = cpu_baseline_record(args.cpu_rows if W["key"] == "c2" else
                                                  args.cpu_rows // 16)
    return rec


# ---------------------------------------------------------------- our arm: treecodes
def measure_tree(args, ctx, steps, warmup):
    """Treecode workloads (c2t, c4t): s/iteration of the full optimizer iteration with
    RepulsionConfig(backend="tree") and the treecode attraction, through ShardedRun."""
    import torch

    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import engine
    from paper_2108_02991_b200 import tree as _tree

    cfg = spk.OptimizerConfig(n_c=N_C, n_s=N_S, dims=DIMS, n_pit=100, grad_mode="exact",
                              grid_n=GRID_N, seed=0, perturbation=W["pert"],
                              attraction_tree_precision=W["att_prec"],
                              repulsion=spk.RepulsionConfig(backend="tree",
                                                            tree_precision=W["rep_prec"]))
    fld = spk.precompute_field(density())
    t0 = time.perf_counter()
    fld.source_tree().static_proxies(_tree.auto_params(W["att_prec"], DIMS)[0])
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    run = engine.ShardedRun(np.ascontiguousarray(start_pattern().coords), cfg, fld)
    run.project(proj_config())
    step, _ = optimizer_step(run, cfg)
    total_ms, clocks, launches = timed_loop(ctx, step, steps, warmup)
    (total_ms,) = ctx.max(total_ms)
    p, g, rep_pairs, att_pairs = pairs_per_step()
    s_it = total_ms / steps / 1e3
    del run, fld
    return {
        "metric": "s/iteration", "value": s_it, "unit": "s", "n_gpus": ctx.world,
        "steps": steps, "warmup": warmup, "ms_per_step": s_it * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
        "config": workload_config(),
        "parallelism": f"shots sharded over {ctx.world} GPU(s)",
        "equivalent_direct_pairs_per_s": (rep_pairs + att_pairs) / s_it,
        "setup_s": {"lattice_tree_and_proxies": t_setup},
        "roofline": None,
        "roofline_note": "treecode interaction lists change every iteration; the kernel "
                         "roofline is reported on the exact lines",
        "clocks": clocks, "gpu_launches": launches,
    }


# ---------------------------------------------------------------- our arm: C3 stack
def measure_stack(args, ctx, steps, warmup):
    """C3: one stacked optimize iteration of G independent problems per step (1 GPU)."""
    import torch

    import paper_2108_02991_b200 as spk
    from paper_2108_02991_b200 import _native, stack
    from paper_2108_02991_b200.optimizer import _bb_step, default_eta0

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
        # fused launches only (a[4] = lattice weights; None when K2 ran under the polish)
        if name == "spk_fused_sums_batched" and st.get("record") and a[4] is not None:
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

    def on_record():
        st["record"] = True

    try:
        total_ms, clocks, launches = timed_loop(ctx, step, steps, warmup, on_record)
        last_split = run.att_pre is not None
        if not nb_events:
            # every timed step split the N-body (K2 under the polish): time the fused
            # batched launch alone for the roofline
            for _ in range(3):
                run.att_pre = None
                run.evaluate()
            torch.cuda.synchronize()
            nb_events[:] = nb_events[1:]
    finally:
        _native.call = orig_call
    nb_ms = float(np.mean([a.elapsed_time(b) for a, b in nb_events]))
    p, g, rep_pairs, att_pairs = pairs_per_step()
    pairs = G * (rep_pairs + att_pairs)
    return {
        "metric": METRIC, "value": pairs * steps / (total_ms / 1e3), "unit": "pairs/s",
        "n_gpus": 1, "steps": steps, "warmup": warmup,
        "ms_per_step": total_ms / steps, "s_per_iteration": total_ms / steps / 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 pair math, f64 accumulation / projection", "data": "synthetic",
        "config": workload_config(), "parallelism": "one device batch",
        "schedule": {"k2_under_polish_in_last_step": last_split},
        "roofline": nbody_roofline("c3", DIMS, G * rep_pairs, G * att_pairs, nb_ms, clocks)
        | {"kernel": "nbody_kernel batched (spk_fused_sums_batched)"},
        "clocks": clocks, "gpu_launches": launches,
    }


# ---------------------------------------------------------------- end to end
def run_e2e_step_api(ctx, cfg, fld, steps):
    """The public per-iteration API -- ``optimizer.start`` once, then ``optimizer.step``
    (optimize's loop body: evaluate, guards, step size, step + projection, residuals,
    TraceRecord) -- with the pattern round-tripping through pinned host memory every step:
    this rank's shots copied H2D into the run before the call, the projected shots copied
    D2H after it (the step's TraceRecord scalars come back inside the call).  Each step is
    device-timed with CUDA events around the copies and the call; max over ranks.  The
    shots a step receives are the previous step's output, so the run progresses like
    ``optimize``."""
    import dataclasses

    import torch

    from paper_2108_02991_b200 import optimizer as om

    warm = 2  # the first step has no previous sweep counts (plain schedule)
    cfg_e = dataclasses.replace(cfg, n_decim=0, n_git=warm + steps)
    state = om.start(cfg_e, hardware(), rho=density(), fld=fld)
    run = state.run
    host_in = torch.empty(run.coords.shape, dtype=torch.float64, pin_memory=True)
    host_out = torch.empty_like(host_in, pin_memory=True)
    for _ in range(warm):
        om.step(state)
    host_in.copy_(run.coords)
    torch.cuda.synchronize()
    ctx.barrier()
    total = 0.0
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run.coords.copy_(host_in, non_blocking=True)
        rec = om.step(state)
        host_out.copy_(run.coords, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        total += s.elapsed_time(e)
        if rec is None or not np.isfinite(rec.cost):
            raise RuntimeError("e2e: optimizer.step did not return a finite record")
        host_in.copy_(host_out)
    (total,) = ctx.max(total)
    p, g, rep_pairs, att_pairs = pairs_per_step()
    nbytes = host_in.numel() * 8
    del state, run
    torch.cuda.empty_cache()
    return {"value": (rep_pairs + att_pairs) * steps / (total / 1e3), "unit": "pairs/s",
            "s_per_iteration": total / 1e3 / steps, "steps": steps,
            "h2d_bytes_per_step": nbytes * ctx.world,
            "d2h_bytes_per_step": nbytes * ctx.world + 64 * ctx.world,
            "api": "optimizer.start + optimizer.step (the public per-iteration entry point, "
                   "optimize's loop body) with every rank's shots H2D from pinned host "
                   "memory before and D2H after each step, plus the TraceRecord scalars"}


def run_e2e(args, spk, fld, pcfg, steps):
    """The reference's loop body (optimizer.py:301-344) through the public API with numpy
    host arrays; every call copies its inputs H2D and results D2H."""
    import torch
    from paper_2108_02991_b200.optimizer import default_eta0, step_size

    pattern = spk.project_pattern(start_pattern(), pcfg)
    rcfg = spk.RepulsionConfig(kernel_eps=EPS_REP)
    eta0 = default_eta0(pattern.n_samples, EPS_REP)
    prev_c = prev_g = None
    eta = eta0
    steps = max(1, min(steps, args.e2e_steps))
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
        "config": workload_config(), "parallelism": f"{threads} host CPU threads",
        "cpu_baseline": {"value": rate, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"per step {args.ref_rows} target rows x all {p} sources "
                                   f"+ {args.ref_rows} rows x {g} grid cells, fp64, plus "
                                   f"{samples[0]['proj_sample']} through the projection; "
                                   f"s/iteration extrapolated"},
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
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true",
                    help="skip the c4 / c4t sub-records of the default c2 run")
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    select_workload(args.config)
    if args.impl == "reference":
        run_reference(args)
        return
    ensure_world(args)
    ctx = Ctx()
    from paper_2108_02991_b200 import _device

    if W.get("stack"):
        line = measure_stack(args, ctx, args.steps, args.warmup)
    elif W.get("tree"):
        line = measure_tree(args, ctx, args.steps, args.warmup)
    else:
        line = measure_exact(args, ctx, args.steps, args.warmup, not args.no_e2e,
                             not args.no_cpu_baseline)
    if args.config == "c2" and not args.no_sub:
        line["subrecords"] = {}
        for key, (k, w) in SUBRECORDS.items():
            _device.release_workspaces()
            select_workload(key)
            k = args.steps if k is None else min(k, args.steps)
            w = args.warmup if w is None else w
            t0 = time.perf_counter()
            if W.get("tree"):
                rec = measure_tree(args, ctx, k, w)
            else:
                rec = measure_exact(args, ctx, k, w, False, not args.no_cpu_baseline)
            rec["wall_s"] = time.perf_counter() - t0
            line["subrecords"][key] = rec
            if ctx.rank == 0:
                print(f"bench.py: {key}: {rec['ms_per_step'] / 1e3:.3f} s/it "
                      f"({rec['wall_s']:.0f} s wall)", file=sys.stderr, flush=True)
        select_workload(args.config)
    # after the process group is destroyed: NCCL's INIT-subsystem INFO lines (which go to
    # stdout, N > 1) then all precede the JSON line, which stays the last line
    ctx.close()
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
