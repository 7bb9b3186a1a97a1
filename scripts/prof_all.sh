# Round profile capture (one GPU): launch list of the bench command + full captures of the hot kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_struct_for -s 60 -c 1 -o gpurun_out/prof/c2_jacobi python scripts/prof_c2.py 3 > /dev/null 2>&1; echo c2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_struct_for -s 6 -c 1 -o gpurun_out/prof/jac_xl python scripts/xl_bench.py jac > /dev/null 2>&1; echo jacxl rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_listgen -s 1 -c 1 -o gpurun_out/prof/lg_xl python scripts/xl_bench.py lg > /dev/null 2>&1; echo lgxl rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_g2p" -s 2 -c 2 -o gpurun_out/prof/c3_mpm python scripts/prof_c3.py 1 > /dev/null 2>&1; echo c3 rc=$?
ls -la gpurun_out/prof
