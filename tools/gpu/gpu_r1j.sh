cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=c2 RUNS=768:2 ITERS=3 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c2_q.log 2>&1
grep -v "^sample" gpurun_out/c2_q.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chol_diag -s 0 -c 1 -o gpurun_out/prof_diag $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_nn_kernel -s 3 -c 1 -o gpurun_out/prof_nn $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?"
ls -la gpurun_out/*.ncu-rep
