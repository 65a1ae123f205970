set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
tail -30 gpurun_out/smoke.log
