cd $GRAFT_REPO_ROOT
for cfg in none shared equal l1; do
  if [ $cfg = none ]; then unset SG_CACHECFG; else export SG_CACHECFG=$cfg; fi
  timeout 300 python scripts/mpm_time.py > gpurun_out/cc_$cfg.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cc_$cfg.json')); print('$cfg', 'c3', round(d['c3']['ms_per_step'],4), 'c4', round(d['c4']['ms_per_iteration'],3), 'c4 listgen', d['c4']['avg_us_per_launch_kind']['listgen'])"
  timeout 300 python scripts/host_time.py
done
