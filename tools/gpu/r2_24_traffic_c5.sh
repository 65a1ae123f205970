#!/bin/bash
# round 2, call 24: DRAM bytes per kernel-class region of one c5 factorization (bench.py roofline
# `traffic`), ncu with NVTX class ranges; serialised launches, no timing claims
mkdir -p gpurun_out
O=gpurun_out/r2_call24.txt
timeout 3000 ncu --nvtx --nvtx-include "gemm_nt_gram/" --nvtx-include "gemm_nn_lu_update/" --nvtx-include "cholesky/" \
   --nvtx-include "gemm_nn_proj/" --nvtx-include "gemm_nn_ef/" --print-nvtx-rename kernel --clock-control none \
   --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --csv --log-file gpurun_out/r2_ncu_traffic_c5.csv \
   python tools/ncu_traffic.py run --config c5 --regions gpurun_out/r2_regions_c5.json > gpurun_out/r2_c24_ncu.log 2>&1
echo "ncu exit $?" > $O
python tools/ncu_traffic.py parse --config c5 --csv gpurun_out/r2_ncu_traffic_c5.csv \
   --regions gpurun_out/r2_regions_c5.json --out gpurun_out/ncu_traffic_r02.json > gpurun_out/r2_c24_parse.log 2>&1
echo "parse exit $?" >> $O
gzip -kf gpurun_out/r2_ncu_traffic_c5.csv
