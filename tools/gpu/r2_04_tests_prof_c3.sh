#!/bin/bash
# round 2, call 4: full GPU suite (new sweep kernels, f1/f4/f2 tests), c3 per-level trace, ncu --set full of
# the sphere's leaf Gram precompute, projection and pulled L/U update
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call4.txt
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_levels.log 2>&1
echo "levels exit $?" >> gpurun_out/r2_call4.txt
for spec in "gemm_nt_gram:0" "gemm_nn_proj:0" "gemm_nn_lu_update:3" "cholesky:1"; do
  cls=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "$cls/" \
      --launch-skip $skip --launch-count 1 -o gpurun_out/r2_c3_$cls -f \
      env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_ncu_$cls.log 2>&1
  echo "ncu $cls exit $?" >> gpurun_out/r2_call4.txt
done
