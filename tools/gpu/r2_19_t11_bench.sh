#!/bin/bash
# round 2, call 19: t11 at p = 1536 (GPU tests incl. full-size oracle parity), skinny E/F columns per
# CTA A/B on c3, c5 bench line after the round-2 kernel changes
mkdir -p gpurun_out
O=gpurun_out/r2_call19.txt
python -m pytest tests/test_gpu_t11.py -q > gpurun_out/r2_c19_pytest_t11.log 2>&1
echo "pytest t11 exit $?" > $O
for sc in 256 512; do
  RSRS_SKINNY_COLS=$sc CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c19_c3_sk$sc.log 2>&1
  echo "c3 skinny $sc exit $?" >> $O
done
timeout 1800 python bench.py > gpurun_out/r2_c19_bench_c5.json 2> gpurun_out/r2_c19_bench_c5.err
echo "bench c5 exit $?" >> $O
