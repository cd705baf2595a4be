"""Guard paths (eps^2 below FLT_MIN) of the treecode and the lattice kernel: coincident
pairs / targets on lattice nodes must stay finite and match the exact sums."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk  # noqa: E402
from paper_2108_02991_b200 import _device  # noqa: E402
from paper_2108_02991_b200.attraction import grid_sums_device, tree_grid_sums_device  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from test_gpu_fuzz import _cloud  # noqa: E402

for dims in (2, 3):
    pts = _cloud(dims, 200_000, "duplicates", 3)
    for eps in (0.0, 1e-20):
        cfg = spk.RepulsionConfig(backend="tree", tree_precision=1e-4, kernel_eps=eps)
        ct, gt = spk.eval_repulsion_tree(pts, cfg)
        cd, gd = spk.eval_repulsion_direct(pts, eps)
        print(f"tree dims={dims} eps={eps}: finite {np.isfinite(ct) and np.all(np.isfinite(gt))} "
              f"cost {abs(ct-cd)/abs(cd):.2e} grad {np.linalg.norm(gt-gd)/np.linalg.norm(gd):.2e}")
    n = 20 if dims == 2 else 8
    rho = spk.discretize(spk.DensityParams(0.25, 2.0), n, dims)
    fld = spk.precompute_field(rho, kernel_eps=1e-20)
    ax = np.arange(-n, n + 1) / n
    nodes = np.stack(np.meshgrid(*([ax] * dims), indexing="ij"), -1).reshape(-1, dims)
    p4 = _device.pack_positions(_device.h2d(nodes))
    v, g = (_device.d2h(x) for x in grid_sums_device(p4, fld, 1e-40))
    vr, gr = orc.grid_sums(nodes, rho.grid, 1e-40)
    print(f"lattice dims={dims} eps=1e-20 on nodes: finite {np.all(np.isfinite(v)) and np.all(np.isfinite(g))} "
          f"val {np.linalg.norm(v-vr)/np.linalg.norm(vr):.2e} grad {np.linalg.norm(g-gr)/np.linalg.norm(gr):.2e}")
