"""The README quick-start, shortened (n_git = 2), so that its API calls are checked."""
import os
import sys
import tempfile

sys.path.insert(0, ".")
import paper_2108_02991_b200 as vdtraj  # noqa: E402

hw = vdtraj.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                         dwell_dt=2e-6, fov=(0.23, 0.23, 0.1248), matrix=(384, 384, 208), dims=3)
rho = vdtraj.discretize_anisotropic(vdtraj.DensityParams(0.25, 2.0), (192, 192, 104), 3)
cfg = vdtraj.OptimizerConfig(n_c=4096, n_s=2048, dims=3, n_decim=6, n_git=2, n_pit=100,
                             perturbation=0.75, grad_mode="exact", attraction_tree_precision=1e-4,
                             repulsion=vdtraj.RepulsionConfig(backend="tree", tree_precision=1e-3))
res = vdtraj.optimize(cfg, hw, rho=rho)
st = vdtraj.start(cfg, hw, rho=rho)
vdtraj.step(st)
vdtraj.finish(st)
d = tempfile.mkdtemp()
vdtraj.io.write_spkt(os.path.join(d, "traj.spkt"), res.pattern, hw.k_max, hw.raster_dt)
try:
    vdtraj.optimize(vdtraj.OptimizerConfig(n_c=4096, n_s=2048, dims=3, n_decim=6, n_git=1,
                                           grad_mode="exact"), hw)
except MemoryError as e:
    print("default-grid guard:", str(e)[:80])
print("readme quick-start ok", res.pattern.coords.shape, len(res.trace.records))
