#!/bin/bash
# round 2, call 33: nn_stream_kernel (streaming L/U push for n_r <= 32) A/B on c3 / c2, E/F through
# the same kernel (RSRS_EF_STREAM=1), parity tests on the new default
mkdir -p gpurun_out
O=gpurun_out/r2_call33.txt
: > $O
run() {  # name, env...
  local name=$1; shift
  env "$@" CFG=${CFG:-c3} RUNS=${RUNS:-1216:2} ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c33_$name.log 2>&1
  echo "$name exit $?" >> $O
  grep -E "iter 2|gemm_nn_lu_update|gemm_nn_ef|residual" gpurun_out/r2_c33_$name.log >> $O
}
run c3_off RSRS_NS_KMAX=0
run c3_on RSRS_NS_KMAX=128
run c3_on_ch4 RSRS_NS_KMAX=128 RSRS_NS_CHUNKS=4
run c3_on_ch19 RSRS_NS_KMAX=128 RSRS_NS_CHUNKS=19
run c3_on_ef RSRS_NS_KMAX=128 RSRS_EF_STREAM=1
run c3_on32 RSRS_NS_KMAX=32
CFG=c2 RUNS=768:2 run c2_off RSRS_NS_KMAX=0
CFG=c2 RUNS=768:2 run c2_on RSRS_NS_KMAX=128
CFG=c2 RUNS=768:2 run c2_on_ef RSRS_NS_KMAX=128 RSRS_EF_STREAM=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_dist.py -q -x > gpurun_out/r2_c33_pytest.log 2>&1
echo "pytest exit $?" >> $O
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "nn_stream or ef_stream" > gpurun_out/r2_c33_pytest_var.log 2>&1
echo "pytest variants exit $?" >> $O
