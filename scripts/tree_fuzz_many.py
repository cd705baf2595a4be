import sys, itertools, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2108_02991_b200 as spk
from test_gpu_fuzz import _cloud
rng = np.random.default_rng(12345)
worst = {}
fails = []
for trial in range(160):
    dims = int(rng.choice([2, 3])); kind = str(rng.choice(["uniform", "radial", "clustered", "duplicates"]))
    prec = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-5])); seed = int(rng.integers(0, 2**31 - 1))
    n = int(rng.choice([140_000, 300_000, 1_000_000]))
    pts = _cloud(dims, n, kind, seed)
    cfg = spk.RepulsionConfig(backend="tree", tree_precision=prec)
    ct, gt = spk.eval_repulsion_tree(pts, cfg)
    cd, gd = spk.eval_repulsion_direct(pts, cfg.kernel_eps)
    eg = np.linalg.norm(gt - gd) / np.linalg.norm(gd); ec = abs(ct - cd) / abs(cd)
    key = (dims, kind, prec)
    worst[key] = max(worst.get(key, 0), eg / prec)
    if eg > prec or ec > prec:
        fails.append((dims, kind, prec, n, seed, eg, ec))
print("fails", len(fails))
for f in fails[:10]: print(f)
for k, v in sorted(worst.items()): print(k, f"worst err/prec {v:.2f}")
