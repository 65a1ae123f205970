#!/bin/bash
# round 2, call 8: flat 16-row warp layout in the TM = 32 DMMA tiles; c3 / c5 traces; bench c5 (host-mode e2e)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py -x -q > gpurun_out/r2_pytest_call8.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call8.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_flat.log 2>&1
echo "c3 exit $?" >> gpurun_out/r2_call8.txt
python bench.py > gpurun_out/r2_bench_c5_v3.json 2> gpurun_out/r2_bench_c5_v3.err
echo "bench exit $?" >> gpurun_out/r2_call8.txt
