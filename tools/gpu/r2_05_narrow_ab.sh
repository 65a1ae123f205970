#!/bin/bash
# round 2, call 5: narrow small-box tiles + per-box Gram-block update + wide skinny E/F:
# correctness (parity subset), A/B per-level traces on c3 and c5, c3 launch list
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py tests/test_gpu_coupling.py tests/test_gpu_triangular.py -x -q > gpurun_out/r2_pytest_narrow.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call5.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_levels_narrow.log 2>&1
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 RSRS_WIDE_NT=1 python tools/quick_c2.py > gpurun_out/r2_c3_levels_wide.log 2>&1
echo "c3 traces exit $?" >> gpurun_out/r2_call5.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_launches_c3.log 2>&1
echo "launches exit $?" >> gpurun_out/r2_call5.txt
CFG=c5 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c5_levels_narrow.log 2>&1
echo "c5 trace exit $?" >> gpurun_out/r2_call5.txt
