cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
RSRS_DEBUG_SYNC=1 timeout 900 python -m pytest tests/test_gpu_gram_blocks.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gb.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gb.log
bash tools/gpu_r1q.sh
