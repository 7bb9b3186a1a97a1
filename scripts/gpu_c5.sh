cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parallel.py -x -q > gpurun_out/c5_pytest.log 2>&1; echo c5 rc=$?
tail -30 gpurun_out/c5_pytest.log
