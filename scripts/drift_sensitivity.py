"""Sensitivity of the REFERENCE optimize to 1e-6 relative noise in the repulsion gradient
(authoring container only: imports /root/reference).  Result recorded in DESIGN.md."""
import sys, numpy as np
sys.path.insert(0,'/root/reference/pkg/src')
import vdtraj.optimizer as om
from vdtraj import core
from vdtraj.repulsion import eval_repulsion as er
hw = core.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=1e-5, fov=0.192, matrix=32, dims=2)
for mode in ("consistent","smooth"):
    cfg = om.OptimizerConfig(n_c=8, n_s=64, dims=2, n_decim=1, n_git=6, n_pit=100, perturbation=0.25, seed=3, grad_mode=mode, repulsion=om.RepulsionConfig(backend="direct"))
    base = om.optimize(cfg, hw)
    rng = np.random.default_rng(0)
    def noisy(k, c):
        cost, g = er(k, c)
        return cost*(1+1e-7*rng.standard_normal()), g*(1+1e-6*rng.standard_normal(g.shape))
    om.eval_repulsion = noisy
    pert = om.optimize(cfg, hw)
    om.eval_repulsion = er
    print(mode, 'coords drift', np.abs(pert.pattern.coords-base.pattern.coords).max(), 'cost rel', np.abs(pert.trace.costs()-base.trace.costs()).max()/np.abs(base.trace.costs()).max())
    print('  steps', [f"{r.step:.4g}" for r in base.trace.records][-4:], 'feas', [f"{r.feas_residual:.2g}" for r in base.trace.records][-3:])
