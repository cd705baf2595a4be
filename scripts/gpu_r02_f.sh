#!/bin/bash
# Round-2 GPU session F: what bounds the polish ring step (fixed sweeps, experiments).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
bash scripts/ab_build.sh indep "-DSPK_EXP_SA_INDEP"
bash scripts/ab_build.sh noacc "-DSPK_EXP_NOACCEL"
bash scripts/ab_build.sh nospd "-DSPK_EXP_NOSPEED"
bash scripts/ab_build.sh nosync "-DSPK_EXP_NOSYNC"
for v in base indep noacc nospd nosync base; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v"
  (cd $d && timeout 300 python scripts/polish_fixed.py 16 3200 && timeout 300 python scripts/polish_fixed.py 1024 1600) 2>&1
done > gpurun_out/polish_exp_f.txt
cat gpurun_out/polish_exp_f.txt
