# round-end style check on one GPU: smoke, full -m gpu suite, default bench, profiles
cd $GRAFT_REPO_ROOT
TAG=${1:-rnd}
timeout 300 python -c "import __graft_entry__ as E; E.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref rc=$?
bash scripts/prof_all.sh > gpurun_out/${TAG}_prof.log 2>&1; echo prof rc=$?
