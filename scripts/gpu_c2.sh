# C2 iteration: parity tests, bench (with extras), Jacobi launch list
cd $GRAFT_REPO_ROOT
TAG=${1:-c2}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | head
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python -c "
import json
d=json.load(open('gpurun_out/${TAG}_bench.json')); print('C2', d['value'], 'jac us', d['roofline']['avg_launch_us'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])
for k,v in d.get('extra',{}).items(): print('  ', k, {kk: vv for kk, vv in v.items() if kk in ('steps_per_s','solves_per_s','avg_launch_us','achieved_GBps','frac','iterations_per_s','error')})
"
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/prof_c2.py 2 > /dev/null 2>&1; echo ncu rc=$?
python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/${TAG}_launches.csv')))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(list)
for d in data: agg[d['Kernel Name'].split('(')[0][:50]].append(float(d['Metric Value']))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])): print(f"{k:50s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.2f}us min={min(v)/1e3:.2f}")
PY
