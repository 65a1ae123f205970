cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_blocks.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gb.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_gb.log; grep -E "FAILED|Error" gpurun_out/pytest_gb.log | head -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c2.log | cut -c1-400
RSRS_TRACE=1 CFG=c3 RUNS=1216:2 ITERS=2 timeout 900 python tools/quick_c2.py > gpurun_out/c3_q.log 2>&1
RSRS_TRACE=1 CFG=c5 RUNS=1216:2 ITERS=2 timeout 900 python tools/quick_c2.py > gpurun_out/c5_q.log 2>&1
cat gpurun_out/c3_q.log gpurun_out/c5_q.log | grep -v "^sample" | tail -30
