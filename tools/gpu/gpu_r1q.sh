cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=c2 RUNS=768:2 ITERS=3 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c2_q.log 2>&1
CFG=c3 RUNS=1216:2 ITERS=2 PROF=last RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/c3_q.log 2>&1
CFG=c4 RUNS=768:2 ITERS=2 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c4_q.log 2>&1
cat gpurun_out/c2_q.log gpurun_out/c3_q.log gpurun_out/c4_q.log | grep -v "^sample"
