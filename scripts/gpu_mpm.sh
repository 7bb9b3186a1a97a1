# MPM iteration on the GPU box: parity tests, then C3/C4 timings binned and per-particle
cd $GRAFT_REPO_ROOT
TAG=${1:-mpm}
timeout 900 python -m pytest tests/test_gpu_mpm.py tests/test_gpu_c4.py tests/test_gpu_parallel.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Error|assert" gpurun_out/${TAG}_pytest.log | head -20
timeout 600 python scripts/mpm_time.py > gpurun_out/${TAG}_time_bin.json 2> gpurun_out/${TAG}_time_bin.err; echo time rc=$?
SG_NO_BIN=1 timeout 600 python scripts/mpm_time.py > gpurun_out/${TAG}_time_nobin.json 2> gpurun_out/${TAG}_time_nobin.err; echo time rc=$?
python - <<PY
import json
for f in ("bin", "nobin"):
    try:
        d = json.load(open("gpurun_out/${TAG}_time_%s.json" % f))
    except Exception as e:
        print(f, "no result", e); continue
    for k in ("c3", "c4"):
        v = d.get(k, {})
        print(f, k, {kk: vv for kk, vv in v.items() if kk in ("steps_per_s", "ms_per_step", "iterations_per_s", "ms_per_iteration", "error")})
        print("   ", v.get("avg_us_per_launch_kind"))
PY
