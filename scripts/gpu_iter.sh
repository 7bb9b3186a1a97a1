# one build-measure iteration on the GPU box (outputs under gpurun_out/)
cd $GRAFT_REPO_ROOT
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
head -c 2500 gpurun_out/${TAG}_bench.json; echo
SG_SF_PAIR=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_nopair.json 2>&1; echo bench0 rc=$?
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_nopair.json'));print('nopair', d['value'], d['roofline']['avg_launch_us'])"
timeout 600 python scripts/xl_bench.py > gpurun_out/${TAG}_xl.json 2> gpurun_out/${TAG}_xl.err; echo xl rc=$?
cat gpurun_out/${TAG}_xl.json; tail -3 gpurun_out/${TAG}_xl.err
SG_SF_PAIR=0 timeout 600 python scripts/xl_bench.py jac > gpurun_out/${TAG}_xl_nopair.json 2>&1; echo xl0 rc=$?
cat gpurun_out/${TAG}_xl_nopair.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/prof_c2.py 2 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_struct_for -s 60 -c 1 -o gpurun_out/${TAG}_sf python scripts/prof_c2.py 3 > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
tail -1 gpurun_out/${TAG}_ncu.log
