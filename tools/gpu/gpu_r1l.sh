cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=c5 RUNS=1216:2 ITERS=2 PROF=last RSRS_TRACE=1 timeout 1500 python tools/quick_c2.py > gpurun_out/c5_q.log 2>&1; echo "c5 exit $?"
cat gpurun_out/c5_q.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
