#!/bin/bash
# round 2, call 15: packed solve records + fused Cholesky (real, small near fields): parity, A/B
mkdir -p gpurun_out
O=gpurun_out/r2_call15.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py tests/test_gpu_dist.py -x -q > gpurun_out/r2_c15_pytest_default.log 2>&1
echo "pytest default exit $?" > $O
RSRS_CHOL_FUSE_RMAX=100000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_coupling.py -x -q > gpurun_out/r2_c15_pytest_fuseall.log 2>&1
echo "pytest fuse-all exit $?" >> $O
for c in c2 c3; do
  CFG=$c timeout 600 python tools/solve_bench.py > gpurun_out/r2_c15_solve_$c.json 2> gpurun_out/r2_c15_solve_$c.err
  echo "solve $c exit $?" >> $O
done
RSRS_SWEEP_GRAPH=0 CFG=c2 timeout 600 python tools/solve_bench.py > gpurun_out/r2_c15_solve_c2_nograph.json 2>&1
echo "solve c2 nograph exit $?" >> $O
RSRS_CHOL_FUSE_RMAX=0 CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c15_c3_nofuse.log 2>&1
echo "c3 nofuse exit $?" >> $O
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c15_c3_fuse.log 2>&1
echo "c3 fuse exit $?" >> $O
RSRS_TM32_NT=100000 CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c15_c3_tm32nt.log 2>&1
echo "c3 tm32nt exit $?" >> $O
RSRS_TM32_NT=100000 RSRS_TM32_NN=100000 CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c15_c3_tm32all.log 2>&1
echo "c3 tm32all exit $?" >> $O
# ncu --set full: one leaf-level L/U update GEMM and one fused Cholesky + one skinny E/F launch of c3
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "gemm_nn_lu_update/" \
  --kernel-name regex:gemm_nn_kernel --launch-skip 12 --launch-count 1 -o gpurun_out/r2_c3_luupd -f \
  env CFG=c3 RUNS=1216:2 ITERS=1 python tools/quick_c2.py > gpurun_out/r2_c15_ncu_luupd.log 2>&1
echo "ncu luupd exit $?" >> $O
timeout 900 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"chol_fused|skinny_nn" --launch-skip 8 --launch-count 2 -o gpurun_out/r2_c3_cholf_skinny -f \
  env CFG=c3 RUNS=1216:2 ITERS=1 python tools/quick_c2.py > gpurun_out/r2_c15_ncu_cholf.log 2>&1
echo "ncu cholf exit $?" >> $O
