#!/bin/bash
# round 2, call 3: new tests (complex-symmetric shortcut, sampler), c5 per-level profile, bench c5, ncu traffic c5
mkdir -p gpurun_out
python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_pytest_sym.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call3.txt
CFG=c5 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c5_levels.log 2>&1
echo "levels exit $?" >> gpurun_out/r2_call3.txt
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
echo "bench exit $?" >> gpurun_out/r2_call3.txt
ncu --nvtx --nvtx-include "gemm_nt_gram/" --nvtx-include "gemm_nn_lu_update/" --nvtx-include "cholesky/" \
    --print-nvtx-rename kernel --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --csv --log-file gpurun_out/ncu_traffic_c5.csv \
    python tools/ncu_traffic.py run --config c5 --regions gpurun_out/regions_c5_ncu.json > gpurun_out/ncu_traffic_c5.log 2>&1
echo "ncu exit $?" >> gpurun_out/r2_call3.txt
