# Round profile capture (one GPU): launch list of the bench command + full captures of the hot kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > /dev/null 2>&1; echo launches rc=$?
# C2 JACOBI with warm L2 (the timed step's condition after the first iteration)
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_jacobi8 -s 60 -c 1 -o gpurun_out/prof/c2_jacobi python scripts/prof_c2.py 3 > /dev/null 2>&1; echo c2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi8 -s 6 -c 1 -o gpurun_out/prof/jac_xl python scripts/xl_bench.py jac > /dev/null 2>&1; echo jacxl rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_listgen -s 1 -c 1 -o gpurun_out/prof/lg_xl env SG_PROFILE_FROM_HERE=1 python scripts/xl_bench.py lg > /dev/null 2>&1; echo lgxl rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g_bin|k_g2p_bin" -s 2 -c 2 -o gpurun_out/prof/c3_mpm python scripts/prof_c3.py 1 > /dev/null 2>&1; echo c3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g2p_adj_bin|k_p2g_adj_bin" -s 4 -c 2 -o gpurun_out/prof/c4_adj python scripts/prof_c4.py 4 1 > /dev/null 2>&1; echo c4 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c4.csv python scripts/prof_c4.py 8 2 > /dev/null 2>&1; echo c4 launches rc=$?
ls -la gpurun_out/prof
# summaries on the box (the .ncu-rep files are ~30 MB each; gpurun copies back <= 64 MiB)
cd gpurun_out/prof
python ../../scripts/ncu_summary.py c2_jacobi=c2_jacobi.ncu-rep jac_xl=jac_xl.ncu-rep lg_xl=lg_xl.ncu-rep \
  c3_mpm=c3_mpm.ncu-rep c4_adj=c4_adj.ncu-rep > ncu_summary.md 2> ncu_summary.err
for r in c2_jacobi jac_xl lg_xl c3_mpm c4_adj; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > $r.details.csv 2>/dev/null
done
rm -f c3_mpm.ncu-rep c4_adj.ncu-rep lg_xl.ncu-rep jac_xl.ncu-rep
ls -la
