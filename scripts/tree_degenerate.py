import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2108_02991_b200 as spk
from oracle import oracle as orc
cfg = spk.RepulsionConfig(backend="tree")
rng = np.random.default_rng(0)
n = 200000
pts = np.tile(np.array([[0.3, -0.2, 0.1]]), (n, 1))
t0 = time.time(); c_t, g_t = spk.eval_repulsion_tree(pts, cfg); print("coincident", c_t, np.abs(g_t).max(), time.time()-t0, flush=True)
c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps); print("direct", c_d, abs(c_t-c_d)/c_d, flush=True)
t = rng.uniform(-1, 1, n)
pts = np.stack([t, 1e-6 * rng.normal(size=n), np.zeros(n)], axis=1)
t0 = time.time(); c_t, g_t = spk.eval_repulsion_tree(pts, cfg); print("needle", time.time()-t0, flush=True)
c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
print("needle err", abs(c_t-c_d)/abs(c_d), np.linalg.norm(g_t-g_d)/np.linalg.norm(g_d), flush=True)
# two clusters of coincident points
pts = np.concatenate([np.tile([[0.5, 0.5, 0.5]], (n//2, 1)), np.tile([[-0.5, 0.1, 0.0]], (n//2, 1))])
c_t, g_t = spk.eval_repulsion_tree(pts, cfg); c_d, g_d = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
print("two clusters err", abs(c_t-c_d)/abs(c_d), np.linalg.norm(g_t-g_d)/np.linalg.norm(g_d), flush=True)
