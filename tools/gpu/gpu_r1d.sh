cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export RSRS_TRACE=1
CFG=c2 RUNS=768:2 ITERS=5 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/c2_trace.log 2>&1
CFG=c3 RUNS=1216:2 ITERS=3 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/c3_trace.log 2>&1
grep -E "iter|trace" gpurun_out/c2_trace.log gpurun_out/c3_trace.log
