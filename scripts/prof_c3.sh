cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/prof_c3.py 2 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_range_for -s 2 -c 2 -o gpurun_out/c3_rf python scripts/prof_c3.py 1 > gpurun_out/c3_ncu.log 2>&1; echo ncu rc=$?
