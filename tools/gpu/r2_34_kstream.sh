#!/bin/bash
# round 2, call 34: nn_kstream_kernel (column-walking projection / pulled update) A/B on c3 / c2,
# parity of the forced variants
mkdir -p gpurun_out
O=gpurun_out/r2_call34.txt
: > $O
run() {  # name, env...
  local name=$1; shift
  env "$@" CFG=${CFG:-c3} RUNS=${RUNS:-1216:2} ITERS=3 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c34_$name.log 2>&1
  echo "$name exit $?" >> $O
  grep -E "iter 2|gemm_nn_lu_update|gemm_nn_proj|gemm_nn_ef|residual" gpurun_out/r2_c34_$name.log >> $O
}
run c3_off RSRS_KS_MMAX=0
run c3_ks32 RSRS_KS_MMAX=32
run c3_ks128 RSRS_KS_MMAX=128
run c3_ks128_ch10 RSRS_KS_MMAX=128 RSRS_KS_CHUNKS=10
run c3_ks128_ch3 RSRS_KS_MMAX=128 RSRS_KS_CHUNKS=3
CFG=c2 RUNS=768:2 run c2_off RSRS_KS_MMAX=0
CFG=c2 RUNS=768:2 run c2_ks128 RSRS_KS_MMAX=128
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "kstream" > gpurun_out/r2_c34_pytest_var.log 2>&1
echo "pytest variants exit $?" >> $O
RSRS_KS_MMAX=128 timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_dist.py -q -x > gpurun_out/r2_c34_pytest.log 2>&1
echo "pytest ks exit $?" >> $O
