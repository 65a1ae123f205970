#!/bin/bash
# round 2, call 31: no stream drain after the level setup / compaction (host planning of the next
# level overlaps the compaction): A/B on c3 and c2, parity tests, c5 per-level trace
mkdir -p gpurun_out
O=gpurun_out/r2_call31.txt
CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/r2_c31_c3.log 2>&1
echo "c3 exit $?" > $O
RSRS_LEVEL_SYNC=1 CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/r2_c31_c3_sync.log 2>&1
echo "c3 sync exit $?" >> $O
CFG=c2 RUNS=768:2 ITERS=3 RSRS_TRACE=1 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/r2_c31_c2.log 2>&1
echo "c2 exit $?" >> $O
RSRS_LEVEL_SYNC=1 CFG=c2 RUNS=768:2 ITERS=3 RSRS_TRACE=1 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/r2_c31_c2_sync.log 2>&1
echo "c2 sync exit $?" >> $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_gram_blocks.py tests/test_gpu_determinism.py -q -x > gpurun_out/r2_c31_pytest.log 2>&1
echo "pytest exit $?" >> $O
CFG=c5 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 1200 python tools/quick_c2.py > gpurun_out/r2_c31_c5.log 2>&1
echo "c5 exit $?" >> $O
