#!/bin/bash
# Could the polish hide under the whole fused N-body (K1 + K2)?
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for n in 1 2 8; do timeout 600 python scripts/overlap_probe.py $n fused; done > gpurun_out/overlap_fused.txt 2>&1; echo rc=$?; cat gpurun_out/overlap_fused.txt | grep N=
