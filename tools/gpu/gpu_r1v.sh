cd $GRAFT_REPO_ROOT
CFG=c3 RUNS=1216:2 ITERS=2 PROF=none RSRS_TRACE=1 timeout 900 python tools/quick_c2.py 2>&1 | grep -E "trace|iter"
CFG=c2 RUNS=768:2 ITERS=2 PROF=none RSRS_TRACE=1 timeout 900 python tools/quick_c2.py 2>&1 | grep -E "trace|iter"
