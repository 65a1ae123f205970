cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_symmetric.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist exit $?"
tail -3 gpurun_out/pytest_dist.log; grep -E "FAILED|Error" gpurun_out/pytest_dist.log | head -5
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo "full exit $?"
tail -3 gpurun_out/pytest_full.log; grep -E "FAILED|Error|assert" gpurun_out/pytest_full.log | head -10
