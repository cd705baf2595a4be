#!/bin/bash
# diagnostic: polish cycles/step with single components removed (results are wrong on purpose)
FLAGS=("" NOSPEED NOACCEL NOSNAP NOXFER NOBOX NOSYNC)
for F in "${FLAGS[@]}"; do
  D=/tmp/pexp_$F; rm -rf $D && mkdir -p $D && cp -r paper_2108_02991_b200 include scripts bench.py __graft_entry__.py $D/
  EXTRA="-DSPK_POLISH_PROF"; [ -n "$F" ] && EXTRA="$EXTRA -DSPK_EXP_$F"
  (cd $D && SPK_NVCC_EXTRA="$EXTRA" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1) &
done
wait
for F in "${FLAGS[@]}"; do
  echo "== ${F:-baseline}: $(cd /tmp/pexp_$F && timeout 300 python scripts/polish_profile.py 1 2>&1 | sed -n 2p)"
done
