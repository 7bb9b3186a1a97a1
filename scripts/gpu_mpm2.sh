cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as E; E.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_mpm.py tests/test_gpu_c4.py tests/test_gpu_parallel.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mpm2_bench.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/mpm2_bench.json')); print('C2', round(d['value'],1))
for k in ('c3','c4','mg','mgpcg','c1'): v=d['extra'][k]; print(k, {kk:vv for kk,vv in v.items() if not isinstance(vv,dict)})
"
