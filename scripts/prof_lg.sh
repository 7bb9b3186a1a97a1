# LG-XL listgen: one full ncu capture with source counters + launch time list
cd $GRAFT_REPO_ROOT
TAG=${1:-lg}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_listgen -s 1 -c 1 -o gpurun_out/${TAG}_xl env SG_PROFILE_FROM_HERE=1 python scripts/xl_bench.py lg > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
python scripts/hot_sass.py gpurun_out/${TAG}_xl.ncu-rep 60 > gpurun_out/${TAG}_hot.txt 2>&1
ncu -i gpurun_out/${TAG}_xl.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
timeout 300 python scripts/xl_bench.py lg > gpurun_out/${TAG}_xl.json 2>&1; cat gpurun_out/${TAG}_xl.json
