# one build-measure iteration on the GPU box (outputs under gpurun_out/)
cd $GRAFT_REPO_ROOT
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('C2', d['value'], 'jac us', d['roofline']['avg_launch_us'], 'share', d['roofline']['share_of_step'], 'e2e', d['e2e']['value'])
for k,v in d.get('extra',{}).items(): print(k, {kk: vv for kk, vv in v.items() if kk in ('steps_per_s','solves_per_s','launches_per_step','avg_launch_us','achieved_GBps','frac','error','vcycles_per_s','launches_per_solve','avg_us_per_launch_kind','result_s','iterations_per_s','launches_per_iteration','ms_per_iteration','loss','dead_removed')})
PY
[ -n "$SKIP_NCU" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/prof_c2.py 2 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_struct_for -s 60 -c 1 -o gpurun_out/${TAG}_sf python scripts/prof_c2.py 3 > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
