#!/bin/bash
# round 2, call 30: compact multi-GPU solve merge (emulated-rank tests, both merge modes); ncu source
# capture of one c3 leaf-level fused Cholesky launch and one blocked-path diagonal launch
mkdir -p gpurun_out
O=gpurun_out/r2_call30.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/r2_c30_dist.log 2>&1
echo "dist exit $?" > $O
RSRS_MERGE_COMPACT=0 timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "c1_bit_exact or sphere" > gpurun_out/r2_c30_dist_full.log 2>&1
echo "dist (full-vector merge) exit $?" >> $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_fused -s 3 -c 1 -o gpurun_out/r2_c30_cholf \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c30_ncu_cholf.log 2>&1
echo "ncu cholf exit $?" >> $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_diag_kernel -s 40 -c 1 -o gpurun_out/r2_c30_diag \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c30_ncu_diag.log 2>&1
echo "ncu diag exit $?" >> $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c30_launches_c3_bench.csv \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_c30_launches_c3_bench.log 2>&1
echo "launches c3 bench exit $?" >> $O
gzip -f gpurun_out/r2_c30_launches_c3_bench.csv
