"""Stack-of-SPARKLING: many independent problems optimised as ONE device batch
(BASELINE.json configs[2]: a 2D pattern designed for each of 64 kz partitions).

Every problem runs exactly the reference's ``optimize`` algorithm
(/root/reference/pkg/src/vdtraj/optimizer.py:239-349) with its own seed, costs, guards,
Barzilai-Borwein step and trace; the batch shares the kernel launches:

* one ``spk_fused_sums_batched`` launch for all problems (problem q's targets see only
  problem q's positions; the density lattice is shared);
* one ``spk_combine_gradient_batched`` launch -> per-problem cost and BB scalars;
* one ``spk_project_all`` launch over all shots with a per-shot step size;
* one batched residual launch.

With exact sums and a polish that is heavy next to the N-body (the engine's rule,
engine.ShardedRun), the lattice sums run per polish group under the slower shots' polish
(projection.project_overlap_device) and the next evaluation launches the batched K1
alone.

A single problem of C1 size (32k samples) leaves most of the 148 SMs idle; 64 of them
fill the GPU.
"""

from __future__ import annotations

import time
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device, _native
from .attraction import KernelField, field_eval_device, precompute_field
from .core import HardwareSpec, LinearConstraint, normalized_limits
from .density import TargetDensity, default_grid_n, discretize
from .optimizer import (
    DivergenceError,
    OptimizeResult,
    OptimizerConfig,
    RunTrace,
    TraceRecord,
    _bb_step,
    default_eta0,
    init_radial,
    perturb,
)
from .core import SamplingPattern
from .projection import (
    ProjectionConfig,
    _pin_arrays,
    project_device,
    project_overlap_device,
)


class StackedRun:
    """Device state of G independent problems of identical shape."""

    def __init__(self, starts: np.ndarray, cfg: OptimizerConfig, fld: KernelField):
        self.dev = _device.device()
        self.G, self.n_c, n_s, self.d = starts.shape
        self.cfg, self.fld = cfg, fld
        self.coords = _device.h2d(starts.reshape(self.G * self.n_c, n_s, self.d))
        self._level(n_s)

    def _empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.dev)

    def _level(self, n_s):
        self.n_s = n_s
        self.p = self.n_c * n_s  # samples per problem
        shots = self.G * self.n_c
        self.pos4 = self._empty((self.G * self.p, 4), torch.float32)
        self.next = self._empty((shots, n_s, self.d))
        self.prev = self._empty((shots, n_s, self.d))
        self.grad = self._empty((shots, n_s, self.d))
        self.prev_grad = self._empty((shots, n_s, self.d))
        self.flag = self._empty(1, torch.int32)
        self.have_prev = False
        # K2-under-polish (see the module docstring): lattice sums of the last
        # projection's positions, and the sweep counts that decide and order the next
        self.overlap = self.cfg.grad_mode == "exact"
        self.att_pre = None
        self.sweeps = self._empty(shots, torch.int32)
        self.sweeps_prev = None
        if self.overlap:
            self.att_val = self._empty(self.G * self.p)
            self.att_grad = self._empty((self.G * self.p, self.d))

    def project(self, pcfg):
        out = project_device(self.coords, pcfg, out=self.next, pos4=self.pos4)
        self.coords, self.next = out, self.coords
        self.have_prev = False
        self.att_pre = None

    def _use_overlap(self) -> bool:
        import os

        from .engine import ShardedRun

        env = os.environ.get("SPK_OVERLAP")
        if env is not None:
            return self.overlap and env == "1"
        if not self.overlap or self.sweeps_prev is None:
            return False
        n_src = self.p + int(np.prod(self.fld.sides))
        mean = float(self.sweeps_prev.to(torch.float64).mean().item())
        return mean >= ShardedRun.OVERLAP_MIN_SWEEPS_PER_SOURCE * n_src

    def evaluate(self):
        """Per-problem (att_cost, rep_cost, n_nonfinite, dkdg, dgdg) arrays."""
        G, p, d, cfg = self.G, self.p, self.d, self.cfg
        n = G * p
        va, vr = self._empty(n), self._empty(n)
        ga, gr = self._empty((n, d)), self._empty((n, d))
        eps2_rep = float(cfg.repulsion.kernel_eps ** 2)
        k2_events = []
        if self.att_pre is not None:
            # K2 ran under the last polish: the batched launch sums the positions only
            va, ga, k2_events = self.att_pre
            self.att_pre = None
            n_cells = 0
            args = (None, None, 0.0)
        elif cfg.grad_mode == "exact":
            w = self.fld.device_sources()
            sides = self.fld.sides
            n_cells = int(np.prod(sides))
            args = (w.data_ptr(), _native.i64_array(sides), float(self.fld.kernel_eps ** 2))
        else:
            va, ga, _ = field_eval_device(self.coords.reshape(-1, d), self.fld, cfg.grad_mode)
            n_cells = 0
            args = (None, None, 0.0)
        ws = _device.workspace(_native.query("spk_nbody_batched_workspace_bytes", G, p,
                                             n_cells, p), "nbody")
        _native.call("spk_fused_sums_batched", self.pos4.data_ptr(), G, p, d, *args,
                     self.pos4.data_ptr(), p, eps2_rep,
                     va.data_ptr() if n_cells else None, ga.data_ptr() if n_cells else None,
                     vr.data_ptr(), gr.data_ptr(), ws.data_ptr(), ws.numel(),
                     _device.stream())
        cur = torch.cuda.current_stream()
        for ev in k2_events:
            cur.wait_event(ev)
        out = self._empty((G, 6))
        cws = _device.workspace(_native.query("spk_combine_batched_workspace_bytes", G, p),
                                "combine")
        prev_c = self.prev if self.have_prev else None
        prev_g = self.prev_grad if self.have_prev else None
        _native.call("spk_combine_gradient_batched", G, p, d, va.data_ptr(), ga.data_ptr(),
                     float(p), vr.data_ptr(), gr.data_ptr(), float(p), self.coords.data_ptr(),
                     _device.ptr(prev_c), _device.ptr(prev_g), self.grad.data_ptr(),
                     out.data_ptr(), cws.data_ptr(), cws.numel(), _device.stream())
        o = _device.d2h(out)
        return (o[:, 0] / p, o[:, 1] / (2.0 * p * p), o[:, 4].astype(np.int64), o[:, 2],
                o[:, 3])

    def step_project(self, pcfg, etas: np.ndarray) -> np.ndarray:
        """coords <- P(coords - eta_q * grad) per problem; returns a non-finite flag."""
        eta_shot = _device.h2d(np.repeat(np.asarray(etas, dtype=np.float64), self.n_c))
        self.flag.zero_()
        if self._use_overlap():
            from .engine import CudaOps

            ops = getattr(self, "_ops", None) or CudaOps()
            self._ops = ops
            order = None
            if self.sweeps_prev is not None:
                order = torch.argsort(self.sweeps_prev, descending=True,
                                      stable=True).to(torch.int32)
            ps, ks = ops._overlap_streams()
            out, k2_events = project_overlap_device(
                self.coords, pcfg, grad=self.grad, eta=0.0, out=self.next, pos4=self.pos4,
                nonfinite=self.flag, field=self.fld, att_val=self.att_val,
                att_grad=self.att_grad, sweeps=self.sweeps, order=order, polish_streams=ps,
                k2_streams=ks, eta_per_shot=eta_shot)
            self.att_pre = (self.att_val, self.att_grad, k2_events)
        else:
            out = project_device(self.coords, pcfg, grad=self.grad, eta=0.0, out=self.next,
                                 pos4=self.pos4, nonfinite=self.flag, eta_per_shot=eta_shot,
                                 sweeps=self.sweeps if self.overlap else None)
        if self.overlap:
            self.sweeps_prev = self.sweeps.clone()
        self.prev, self.coords, self.next = self.coords, out, self.prev
        self.prev_grad, self.grad = self.grad, self.prev_grad
        self.have_prev = True
        return bool(self.flag.item())

    def residual_max(self, pcfg) -> np.ndarray:
        pin_idx, pin_val = _pin_arrays(pcfg, self.d)
        out = self._empty((self.G, 5))
        ws = _device.workspace(_native.query("spk_residuals_workspace_bytes",
                                             self.G * self.n_c), "resid")
        pv = _native.f64_array(list(pin_val) + [0.0] * (3 - self.d))
        _native.call("spk_feasibility_residuals_batched", self.coords.data_ptr(), self.G,
                     self.n_c, self.n_s, self.d, pcfg.speed_bound, pcfg.accel_bound, pin_idx,
                     pv, out.data_ptr(), ws.data_ptr(), ws.numel(), _device.stream())
        return _device.d2h(out)[:, 4]

    def upsample(self):
        shots = self.G * self.n_c
        out = self._empty((shots, 2 * self.n_s, self.d))
        _native.call("spk_upsample_shots", self.coords.data_ptr(), out.data_ptr(), shots,
                     self.n_s, self.d, _device.stream())
        self.coords = out
        self._level(2 * self.n_s)

    def coords_host(self) -> np.ndarray:
        return _device.d2h(self.coords).reshape(self.G, self.n_c, self.n_s, self.d).copy()


def optimize_stack(cfg: OptimizerConfig, hw: HardwareSpec, n_stack: int,
                   seeds: Optional[Sequence[int]] = None, rho: Optional[TargetDensity] = None,
                   fld: Optional[KernelField] = None) -> list:
    """Run ``n_stack`` independent ``optimize`` problems (seeds ``cfg.seed + q`` unless
    given) as one device batch; returns one OptimizeResult per problem."""
    if cfg.dims != hw.dims:
        raise ValueError(f"config dims {cfg.dims} != hardware dims {hw.dims}")
    if n_stack < 1:
        raise ValueError("n_stack must be >= 1")
    seeds = list(seeds) if seeds is not None else [cfg.seed + q for q in range(n_stack)]
    if len(seeds) != n_stack:
        raise ValueError("need one seed per problem")
    limits = normalized_limits(hw)
    if rho is None:
        grid_n = cfg.grid_n if cfg.grid_n is not None else default_grid_n(hw.matrix)
        rho = discretize(cfg.density, grid_n, cfg.dims)
    if fld is None:
        fld = precompute_field(rho, cfg.attraction_eps)
    if cfg.grad_mode == "exact" and fld.density is None:
        fld.density = rho
    base = init_radial(cfg.n_c, cfg.n_s, cfg.dims)
    fulls = [perturb(base, cfg.perturbation, s) for s in seeds]
    stride = 2 ** cfg.n_decim
    starts = np.stack([np.ascontiguousarray(f.coords[:, ::stride, :]) for f in fulls])
    pin_full = cfg.resolved_pin()

    run = StackedRun(starts, cfg, fld)
    traces = [RunTrace() for _ in range(n_stack)]
    t0 = time.perf_counter()
    for level in range(cfg.n_decim + 1):
        scale = 2.0 ** (cfg.n_decim - level)
        pin = None
        if pin_full is not None:
            pin = LinearConstraint(pinned_index=pin_full // (2 ** (cfg.n_decim - level)),
                                   pinned_value=np.zeros(cfg.dims))
        pcfg = ProjectionConfig(alpha=limits.alpha * scale, beta=limits.beta * scale,
                                raster_dt=hw.raster_dt, n_pit=cfg.n_pit, pin=pin)
        run.project(pcfg)
        eta0 = cfg.eta0 if cfg.eta0 is not None else default_eta0(run.p,
                                                                   cfg.repulsion.kernel_eps)
        etas = np.full(n_stack, eta0)
        level_min = np.full(n_stack, np.inf)
        have_prev = False
        for it in range(1, cfg.n_git + 1):
            att, rep, bad, dkdg, dgdg = run.evaluate()
            cost = att - rep
            for q in range(n_stack):
                if not np.isfinite(cost[q]) or bad[q]:
                    raise DivergenceError(
                        f"problem {q}: non-finite cost or gradient at level {level} "
                        f"iteration {it}; reduce eta0 (current {etas[q]:.3g})")
                level_min[q] = min(level_min[q], cost[q])
                guard = level_min[q] + cfg.divergence_factor * max(abs(level_min[q]), 1e-6)
                if cost[q] > guard:
                    raise DivergenceError(
                        f"problem {q}: cost {cost[q]:.6g} exceeded divergence guard "
                        f"{guard:.6g} at level {level} iteration {it}; reduce eta0 "
                        f"(current {etas[q]:.3g})")
                etas[q] = _bb_step(it, etas[q], dkdg[q], dgdg[q], have_prev, eta0,
                                   cfg.fixed_step_iters)
            have_prev = True
            if run.step_project(pcfg, etas):
                raise DivergenceError(f"gradient step overflowed at level {level} "
                                      f"iteration {it}: coords must be finite")
            feas = run.residual_max(pcfg)
            wall = time.perf_counter() - t0
            for q in range(n_stack):
                traces[q].append(TraceRecord(level=level, iteration=it,
                                             samples_per_shot=run.n_s, cost=float(cost[q]),
                                             attraction=float(att[q]),
                                             repulsion=float(rep[q]), step=float(etas[q]),
                                             feas_residual=float(feas[q]), wall_time=wall))
        if level < cfg.n_decim:
            run.upsample()
    final = run.coords_host()
    return [OptimizeResult(pattern=SamplingPattern(final[q]), trace=traces[q], density=rho,
                           field=fld, initial=fulls[q]) for q in range(n_stack)]
