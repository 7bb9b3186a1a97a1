cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_listgen -s 0 -c 2 -o gpurun_out/xl_lg python scripts/xl_bench.py lg > gpurun_out/xl_lg_ncu.log 2>&1; echo lg rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_struct_for -s 2 -c 1 -o gpurun_out/xl_jac python scripts/xl_bench.py jac > gpurun_out/xl_jac_ncu.log 2>&1; echo jac rc=$?
tail -2 gpurun_out/xl_lg_ncu.log gpurun_out/xl_jac_ncu.log
