cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
RSRS_DEBUG_SYNC=1 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head
