#!/bin/bash
# Polish 8-warp instantiation register budget (CTAs/SM) for few shots (a rank's share at
# N = 8: 128 C2 shots) and for the full 1024.
mkdir -p gpurun_out
for v in "m3|" "m2|-DSPK_POLISH_MINB=2" "m1|-DSPK_POLISH_MINB=1"; do
  name=${v%%|*}; flags=${v#*|}
  bash scripts/ab_build.sh $name "$flags"
  echo "== $name ($flags)"
  (cd /tmp/ab_$name && for n in 128 1024; do timeout 600 python scripts/polish_inloop_once.py $n 3 c2 | tail -2; done)
done
