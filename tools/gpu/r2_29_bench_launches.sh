#!/bin/bash
# round 2, call 29: default bench (c5) on the current tree, then the ncu launch list of the same
# command (1 timed step, 1 warm-up, no CPU leg; per-launch times are cold-cache and serialised)
mkdir -p gpurun_out
O=gpurun_out/r2_call29.txt
timeout 1800 python bench.py > gpurun_out/r2_c29_bench_c5.json 2> gpurun_out/r2_c29_bench_c5.err
echo "bench c5 exit $?" > $O
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c29_launches_c5.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_c29_launches_c5.log 2>&1
echo "launches exit $?" >> $O
gzip -f gpurun_out/r2_c29_launches_c5.csv
