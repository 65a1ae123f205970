#!/bin/bash
# round 2, call 17: extract ILP + per-level 32-row tiles (parity + c2/c3 timing), packed-solve A/B
# with a launch list, fused Cholesky on every level (A/B), t11 sample-count / tolerance exploration
mkdir -p gpurun_out
O=gpurun_out/r2_call17.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py -q -x > gpurun_out/r2_c17_pytest.log 2>&1
echo "pytest exit $?" > $O
for sp in 0 1; do
  RSRS_SOLVE_PACKED=$sp CFG=c3 timeout 600 python tools/solve_bench.py > gpurun_out/r2_c17_solve_c3_p$sp.json 2>&1
  echo "solve c3 packed=$sp exit $?" >> $O
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"solve|top_|permute" \
  --launch-skip 600 --launch-count 520 --csv --log-file gpurun_out/r2_c17_solve_launches.csv \
  env CFG=c3 RSRS_SWEEP_GRAPH=0 python tools/solve_bench.py > gpurun_out/r2_c17_ncu_solve.log 2>&1
echo "ncu solve exit $?" >> $O
CFG=c2 RUNS=768:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c17_c2.log 2>&1
echo "c2 exit $?" >> $O
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c17_c3.log 2>&1
echo "c3 exit $?" >> $O
RSRS_CHOL_FUSE_RMAX=100000 CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c17_c3_fuseall.log 2>&1
echo "c3 fuseall exit $?" >> $O
CFG=t11 RUNS=1536:2,2048:2 ITERS=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c17_t11_5e-6.log 2>&1
echo "t11 5e-6 exit $?" >> $O
EPS=5e-4 CFG=t11 RUNS=1024:2,768:2 ITERS=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c17_t11_5e-4.log 2>&1
echo "t11 5e-4 exit $?" >> $O
