#!/bin/bash
# round 2, call 9: 8-row / 8-column DMMA predication; parity subset; c3 / c5 traces; c2 solve timings; bench c5
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py tests/test_gpu_triangular.py -x -q > gpurun_out/r2_pytest_call9.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call9.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_pred.log 2>&1
CFG=c5 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c5_pred.log 2>&1
echo "traces exit $?" >> gpurun_out/r2_call9.txt
CFG=c2 python tools/solve_bench.py > gpurun_out/r2_solve_c2.json 2> gpurun_out/r2_solve_c2.err
echo "solve exit $?" >> gpurun_out/r2_call9.txt
python bench.py > gpurun_out/r2_bench_c5_v4.json 2> gpurun_out/r2_bench_c5_v4.err
echo "bench exit $?" >> gpurun_out/r2_call9.txt
