#!/bin/bash
# round 2, call 10: multi-RHS sweep (16-wide tiles, paired shared loads) correctness + c2 solve timings;
# c5 launch list (per-kernel time split of one factorization)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_t11.py -x -q -k "multiple_rhs or c1_parity or pinned or t11_dense" > gpurun_out/r2_pytest_call10.log 2>&1
python tests/parity_full.py --config t11 --out gpurun_out/r02_parity_t11.json > gpurun_out/r2_parity_t11.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call10.txt
CFG=c2 python tools/solve_bench.py > gpurun_out/r2_solve_c2_v2.json 2> gpurun_out/r2_solve_c2_v2.err
echo "solve exit $?" >> gpurun_out/r2_call10.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv \
   env CFG=c5 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_launches_c5.log 2>&1
echo "launches exit $?" >> gpurun_out/r2_call10.txt
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "gemm_nn_lu_update/" \
    --kernel-name regex:gemm_nn --launch-skip 2 --launch-count 2 -o gpurun_out/r2_c3_luupd -f \
    env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_ncu_luupd.log 2>&1
echo "ncu luupd exit $?" >> gpurun_out/r2_call10.txt
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "cholesky/" \
    --kernel-name regex:chol_diag --launch-skip 4 --launch-count 1 -o gpurun_out/r2_c3_choldiag -f \
    env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_ncu_choldiag.log 2>&1
echo "ncu choldiag exit $?" >> gpurun_out/r2_call10.txt
for v in 0 1; do
  RSRS_NT3=$v CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_nt3_$v.log 2>&1
done
echo "nt3 ab exit $?" >> gpurun_out/r2_call10.txt
