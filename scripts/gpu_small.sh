# small-list listgen: full GPU suite, C2 bench with and without k_listgen_small, launch list
cd $GRAFT_REPO_ROOT
TAG=${1:-sm}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_pytest.log
for v in 1 0; do SG_LG_SMALL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$v.json 2> gpurun_out/${TAG}_bench_$v.err; echo "small=$v rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/${TAG}_bench_$v.json')); print('C2', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1))
print({k:(v.get('steps_per_s') or v.get('solves_per_s') or v.get('iterations_per_s')) for k,v in d['extra'].items()})
"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
