#!/bin/bash
# round 2, call 21: 16-row NT / NN tiles for the small-box descriptors of small-box levels (A/B on c3,
# c2 check), parity + kernel-variant tests
mkdir -p gpurun_out
O=gpurun_out/r2_call21.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c21_c3.log 2>&1
echo "c3 exit $?" > $O
RSRS_TM16=0 CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c21_c3_notm16.log 2>&1
echo "c3 notm16 exit $?" >> $O
CFG=c2 RUNS=768:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c21_c2.log 2>&1
echo "c2 exit $?" >> $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_variants.py -q > gpurun_out/r2_c21_pytest.log 2>&1
echo "pytest exit $?" >> $O
