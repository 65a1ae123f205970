cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
RSRS_DEBUG_SYNC=1 timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist exit $?"
tail -40 gpurun_out/pytest_dist.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
