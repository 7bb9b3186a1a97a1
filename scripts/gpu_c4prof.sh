cd $GRAFT_REPO_ROOT
TAG=${1:-c4p}
timeout 600 python scripts/mpm_time.py > gpurun_out/${TAG}_time_bin.json 2> gpurun_out/${TAG}_time_bin.err; echo time rc=$?
python - <<PY
import json
d = json.load(open("gpurun_out/${TAG}_time_bin.json"))
for k in ("c3", "c4"):
    v = d.get(k, {})
    print(k, {kk: vv for kk, vv in v.items() if kk in ("steps_per_s", "ms_per_step", "iterations_per_s", "ms_per_iteration", "error")})
    print("   ", v.get("avg_us_per_launch_kind"))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/prof_c4.py 8 2 > /dev/null 2>&1; echo ncu rc=$?
python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/${TAG}_launches.csv')))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(list)
for d in data[len(data)//2:]:
    agg[d['Kernel Name'].split('(')[0]].append(float(d['Metric Value']))
tot=sum(sum(v) for v in agg.values())
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    print(f"{k:40s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.2f}us tot={sum(v)/1e3:9.1f}us {100*sum(v)/tot:5.1f}%")
PY
