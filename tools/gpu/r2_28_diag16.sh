#!/bin/bash
# round 2, call 28: two-level (16 x 16 warp sub-block) Cholesky diagonal blocks: parity, A/B on c3
mkdir -p gpurun_out
O=gpurun_out/r2_call28.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -k "not t11" > gpurun_out/r2_c28_pytest.log 2>&1
echo "pytest exit $?" > $O
CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c28_c3.log 2>&1
echo "c3 exit $?" >> $O
RSRS_DIAG16=0 CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c28_c3_d64.log 2>&1
echo "c3 diag64 exit $?" >> $O
CFG=c2 RUNS=768:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c28_c2.log 2>&1
echo "c2 exit $?" >> $O
