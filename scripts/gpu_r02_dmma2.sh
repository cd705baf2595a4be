#!/bin/bash
# (historical: NM_CH_CFG / NM_MINB_CFG variants predate the transposed-table kernel, which fixes 64-sample chunks)
# DMMA adjoint variants: table chunk x CTAs per SM (built on the box with scripts/ab_build.sh).
mkdir -p gpurun_out
for v in "base|" "ch32_m3|-DNM_CH_CFG=32 -DNM_MINB_CFG=3" "ch32_m4|-DNM_CH_CFG=32 -DNM_MINB_CFG=4" "ch32_m2|-DNM_CH_CFG=32 -DNM_MINB_CFG=2"; do
  name=${v%%|*}; flags=${v#*|}
  bash scripts/ab_build.sh $name "$flags"
  echo "== $name ($flags)"
  (cd /tmp/ab_$name && timeout 600 python scripts/nudft_bench.py 2>&1 | python -c "
import json, sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d = json.loads(l)
    print(d['case'], 'adjoint fp64 %.3e/s' % d['fp64']['adjoint_products_per_s'])
")
done
