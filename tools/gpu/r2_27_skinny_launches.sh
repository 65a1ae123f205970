#!/bin/bash
# round 2, call 27: skinny E/F shared memory sized per launch (A/B on c3), launch list of one c3 factor
mkdir -p gpurun_out
O=gpurun_out/r2_call27.txt
CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c27_c3.log 2>&1
echo "c3 exit $?" > $O
RSRS_SKINNY_FIXED=1 CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c27_c3_fixed.log 2>&1
echo "c3 fixed exit $?" >> $O
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c27_launches_c3.csv \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c27_launches_c3.log 2>&1
echo "launches exit $?" >> $O
