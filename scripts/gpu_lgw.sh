# warp-tile listgen: parity tests (default variant + the others on the warp tests), LG-XL A/B, ncu of the default
cd $GRAFT_REPO_ROOT
TAG=${1:-lgw}
timeout 600 python -m pytest tests/test_gpu_listgen_warp.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/${TAG}_pytest.log
for v in "0 0" "0 1" "1 0"; do set -- $v; SG_LG_AHEAD=$1 SG_LG_DIRECT=$2 timeout 300 python -m pytest tests/test_gpu_listgen_warp.py -m gpu -x -q 2>&1 | tail -1; done
for v in "1 1" "0 1" "1 0" "0 0"; do set -- $v; SG_LG_AHEAD=$1 SG_LG_DIRECT=$2 timeout 300 python scripts/xl_bench.py lg > gpurun_out/${TAG}_xl_$1$2.json 2>&1; echo "ahead=$1 direct=$2"; python -c "import json; d=json.load(open('gpurun_out/${TAG}_xl_$1$2.json')); print(d['avg_launch_us'], d['frac'])"; done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_listgen -s 1 -c 1 -o gpurun_out/${TAG}_xl env SG_PROFILE_FROM_HERE=1 python scripts/xl_bench.py lg > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
python scripts/ncu_brief.py gpurun_out/${TAG}_xl.ncu-rep 20 > gpurun_out/${TAG}_brief.txt 2>&1
