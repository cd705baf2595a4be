#!/bin/bash
# fp64 NUDFT adjoint on the FP64 tensor cores (DMMA) vs the DFMA kernel: tests + throughput.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_analysis.py tests/test_gpu_acceptance.py -q -x > gpurun_out/gputest_dmma.log 2>&1; echo "pytest (dmma) rc=$?"; tail -2 gpurun_out/gputest_dmma.log
SPK_NUDFT_DMMA=0 timeout 900 python -m pytest tests/test_gpu_analysis.py -q -x > gpurun_out/gputest_dfma.log 2>&1; echo "pytest (dfma) rc=$?"; tail -2 gpurun_out/gputest_dfma.log
for m in 1; do echo "== SPK_NUDFT_DMMA=$m"; SPK_NUDFT_DMMA=$m timeout 900 python scripts/nudft_bench.py > gpurun_out/nudft_bench_dmma$m.jsonl 2>&1; python - $m <<'PY'
import json, sys
for l in open(f"gpurun_out/nudft_bench_dmma{sys.argv[1]}.jsonl"):
    if not l.startswith("{"): print(l.strip()); continue
    d = json.loads(l)
    print(d["case"], "adjoint fp64 %.3e/s" % d["fp64"]["adjoint_products_per_s"], "forward fp64 %.3e/s" % d["fp64"]["forward_products_per_s"], "psf %.2fs" % d["compute_psf_wall_s"])
PY
done
