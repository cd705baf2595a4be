mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/profile_step.py --iters 4 > gpurun_out/profile_step.json 2> gpurun_out/profile_step.err
echo "profile exit $?"
cat gpurun_out/profile_step.json | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['mean_ms'] if isinstance(v,dict) else v) for k,v in d.items()]"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --iters 2 > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/launches.csv')))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            agg[d['Kernel Name'][:60]].append(float(d['Metric Value'].replace(',', '')))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/1e6:10.2f} ms  n={len(v):4d}  {k}")
PY
