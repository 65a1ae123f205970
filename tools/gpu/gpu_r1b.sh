set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -C paper_2311_01451_b200/csrc > gpurun_out/make.log 2>&1
RSRS_DEBUG_SYNC=1 timeout 900 python -m pytest tests -m gpu -x -q -k "c4 or sampler" > gpurun_out/pytest_c4.log 2>&1; echo "pytest c4 exit $?"
tail -30 gpurun_out/pytest_c4.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
CFG=c4 RUNS=768:2 ITERS=2 timeout 900 python tools/quick_c2.py > gpurun_out/c4.log 2>&1; echo "c4 exit $?"
tail -30 gpurun_out/c4.log
