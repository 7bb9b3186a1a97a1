# warp-tile listgen: parity tests, LG-XL A/B (CTA tiles / single-pass warp tiles / two-pass warp tiles), ncu
cd $GRAFT_REPO_ROOT
TAG=${1:-lgw}
timeout 600 python -m pytest tests/test_gpu_listgen_warp.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${TAG}_pytest.log
for v in 0 -1; do SG_LG_WARP=$v timeout 300 python scripts/xl_bench.py lg > gpurun_out/${TAG}_xl_$v.json 2>&1; echo "SG_LG_WARP=$v"; cut -c1-330 gpurun_out/${TAG}_xl_$v.json; done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_listgen -s 1 -c 1 -o gpurun_out/${TAG}_xl env SG_PROFILE_FROM_HERE=1 python scripts/xl_bench.py lg > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:k_listgen --csv --log-file gpurun_out/${TAG}_launches.csv env SG_PROFILE_FROM_HERE=1 python scripts/xl_bench.py lg > /dev/null 2>&1; echo launches rc=$?
