#!/bin/bash
# Round-2 GPU session S: polish register budget in the tail-bound regime (MINB 1 vs 3);
# overlap group count; projected full3d scaling with both target layouts.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
bash scripts/ab_build.sh minb1 "-DSPK_POLISH_MINB=1"
for v in base minb1 base minb1; do
  if [ $v = base ]; then d=.; else d=/tmp/ab_$v; fi
  echo "== $v"; (cd $d && timeout 300 python scripts/polish_inloop_once.py 128 2 && timeout 300 python scripts/polish_inloop_once.py 1024 2)
done > gpurun_out/ab_minb.txt 2>&1
cat gpurun_out/ab_minb.txt
for g in 4 8 16; do echo "== groups $g"; SPK_OVERLAP_GROUPS=$g timeout 600 python bench.py --steps 10 --warmup 5 --no-sub --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])"; done > gpurun_out/ab_groups.txt 2>&1
cat gpurun_out/ab_groups.txt
timeout 2400 python scripts/rank_share_schedule.py > gpurun_out/rank_share_full3d_sp.json 2> gpurun_out/rank_share_full3d_sp.err; echo "schedule rc=$?"
