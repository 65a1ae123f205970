cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tm in 64 32; do
RSRS_UPD_TM=$tm CFG=c2 RUNS=768:2 ITERS=3 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c2_tm$tm.log 2>&1
echo "TM=$tm"; grep -E "iter 2|lu_update" gpurun_out/c2_tm$tm.log
done
