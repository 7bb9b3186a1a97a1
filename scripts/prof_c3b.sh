cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3b_launches.csv python scripts/prof_c3b.py 4 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g_bin|k_g2p_bin" -s 2 -c 2 -o gpurun_out/c3b_mpm python scripts/prof_c3b.py 4 > gpurun_out/c3b_ncu.log 2>&1; echo ncu rc=$?
