cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
CFG=c2 RUNS=768:2 ITERS=3 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c2_q.log 2>&1
CFG=c3 RUNS=1216:2 ITERS=3 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c3_q.log 2>&1
cat gpurun_out/c2_q.log gpurun_out/c3_q.log | grep -v "^sample"
