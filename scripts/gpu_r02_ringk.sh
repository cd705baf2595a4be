#!/bin/bash
# Polish barrier spacing (RING_K) for a rank's few-shot share (128 C2 shots, the N = 8 tail)
# and the full 1024.
mkdir -p gpurun_out
for v in "k4|" "k8|-DSPK_RING_K=8" "k2|-DSPK_RING_K=2"; do
  name=${v%%|*}; flags=${v#*|}
  bash scripts/ab_build.sh $name "$flags"
  echo "== $name ($flags)"
  (cd /tmp/ab_$name && for n in 128 1024; do timeout 600 python scripts/polish_inloop_once.py $n 3 c2 | tail -2; done)
done
