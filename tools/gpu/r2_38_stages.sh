#!/bin/bash
# round 2, call 38: nn_stream_kernel ring depth 3 (2 CTAs / SM) vs 2 (3 CTAs / SM) on c3, bit-identity with 2 stages
mkdir -p gpurun_out
O=gpurun_out/r2_call38.txt
: > $O
run() {
  local name=$1; shift
  env "$@" CFG=c3 RUNS=1216:2 ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c38_$name.log 2>&1
  echo "$name exit $?" >> $O
  grep -E "iter 2|gemm_nn_lu_update|residual" gpurun_out/r2_c38_$name.log | cut -c1-150 >> $O
}
run st3 RSRS_NS_STAGES=3
run st2 RSRS_NS_STAGES=2
RSRS_NS_STAGES=2 timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "bit_identical" > gpurun_out/r2_c38_pytest.log 2>&1
echo "pytest bit-identical (2 stages) exit $?" >> $O
