#!/bin/bash
# round 2, call 26: packed Gram-block row blocks on small-box levels (A/B on c3), parity
mkdir -p gpurun_out
O=gpurun_out/r2_call26.txt
CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c26_c3.log 2>&1
echo "c3 exit $?" > $O
RSRS_GRAM_PACK=0 CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c26_c3_nopack.log 2>&1
echo "c3 nopack exit $?" >> $O
python -m pytest tests/test_gpu_gram_blocks.py tests/test_gpu_parity.py -q -x -k "sphere or gram or ragged or c1" > gpurun_out/r2_c26_pytest.log 2>&1
echo "pytest exit $?" >> $O
