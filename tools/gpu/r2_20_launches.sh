#!/bin/bash
# round 2, call 20: c3 timing after the per-level Gram-block update sizing; launch list of one c3
# factorization + solve (per-kernel device time; ncu serialises launches)
mkdir -p gpurun_out
O=gpurun_out/r2_call20.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c20_c3.log 2>&1
echo "c3 exit $?" > $O
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c20_launches_c3.csv \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c20_launches_c3.log 2>&1
echo "launches exit $?" >> $O
