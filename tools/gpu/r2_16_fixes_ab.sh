#!/bin/bash
# round 2, call 16: t11 / emulated-rank fixes, packed solve v2 (predicated chunked loads),
# NN epilogue prefetch, skinny D prefetch; 32-row tiles everywhere (A/B on c2, c3)
mkdir -p gpurun_out
O=gpurun_out/r2_call16.txt
python -m pytest tests/test_gpu_dist.py tests/test_gpu_t11.py tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py -q > gpurun_out/r2_c16_pytest.log 2>&1
echo "pytest exit $?" > $O
for c in c2 c3; do
  CFG=$c timeout 600 python tools/solve_bench.py > gpurun_out/r2_c16_solve_$c.json 2> gpurun_out/r2_c16_solve_$c.err
  echo "solve $c exit $?" >> $O
done
for c in c2 c3; do
  CFG=$c RUNS=$([ $c = c2 ] && echo 768:2 || echo 1216:2) ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c16_${c}_default.log 2>&1
  echo "$c default exit $?" >> $O
  RSRS_TM32_NT=100000 RSRS_TM32_NN=100000 CFG=$c RUNS=$([ $c = c2 ] && echo 768:2 || echo 1216:2) ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c16_${c}_tm32.log 2>&1
  echo "$c tm32 exit $?" >> $O
done
