#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python scripts/e2e_profile.py > gpurun_out/e2e_profile.json 2>&1; echo "rc=$?"; cat gpurun_out/e2e_profile.json
timeout 300 python - <<'PY' > gpurun_out/copy_rates.txt 2>&1
import time, numpy as np, torch
x = np.random.default_rng(0).uniform(-1, 1, (1024, 1024, 3))
torch.cuda.synchronize()
for name, fn in (("h2d pageable", lambda: torch.from_numpy(x).to("cuda")),):
    for r in range(3):
        t0 = time.perf_counter(); y = fn(); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(name, f"{x.nbytes / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
y = torch.from_numpy(x).to("cuda")
for r in range(3):
    t0 = time.perf_counter(); z = y.cpu().numpy(); t1 = time.perf_counter()
    print("d2h pageable", f"{x.nbytes / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
pin = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
for r in range(3):
    t0 = time.perf_counter(); pin.numpy()[...] = x; g = pin.to("cuda", non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("h2d via pinned staging", f"{x.nbytes / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
for r in range(3):
    t0 = time.perf_counter(); pin.copy_(y, non_blocking=True); torch.cuda.synchronize(); z = pin.numpy().copy(); t1 = time.perf_counter()
    print("d2h via pinned staging", f"{x.nbytes / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
for r in range(3):
    t0 = time.perf_counter(); ok = np.isfinite(x).all(); t1 = time.perf_counter()
    print("np.isfinite 24 MB", f"{(t1 - t0) * 1e3:.1f} ms", flush=True)
PY
cat gpurun_out/copy_rates.txt
