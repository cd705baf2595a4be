#!/bin/bash
# Polish timing vs RING_K (steps between CTA barriers in the polish ring), one build each.
# usage: bash scripts/ring_k_sweep.sh "1 2 4 8"
mkdir -p gpurun_out
for K in $1; do
  rm -rf /tmp/rk$K && mkdir -p /tmp/rk$K && cp -r paper_2108_02991_b200 include oracle tests scripts bench.py __graft_entry__.py /tmp/rk$K/
  (cd /tmp/rk$K && SPK_NVCC_EXTRA="-DSPK_RING_K=$K" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1) || echo "build K=$K failed"
  echo "== RING_K=$K"
  (cd /tmp/rk$K && timeout 300 python scripts/polish_c2.py 2>&1 | tail -4; timeout 300 python scripts/polish_c4.py 2>&1 | tail -3)
done
