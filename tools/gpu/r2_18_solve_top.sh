#!/bin/bash
# round 2, call 18: packed solve v3 (rows per warp in flight, explicit top inverse), fused back
# substitution everywhere, kernel-variant parity, t11 exploration (p / tolerance)
mkdir -p gpurun_out
O=gpurun_out/r2_call18.txt
python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_t11.py -q -k "not full_size" > gpurun_out/r2_c18_pytest.log 2>&1
echo "pytest exit $?" > $O
for c in c2 c3; do
  CFG=$c timeout 600 python tools/solve_bench.py > gpurun_out/r2_c18_solve_$c.json 2> gpurun_out/r2_c18_solve_$c.err
  echo "solve $c exit $?" >> $O
done
CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c18_c3.log 2>&1
echo "c3 exit $?" >> $O
CFG=t11 RUNS=1536:2,2048:2 ITERS=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c18_t11_5e-6.log 2>&1
echo "t11 5e-6 exit $?" >> $O
EPS=5e-4 CFG=t11 RUNS=1024:2 ITERS=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c18_t11_5e-4.log 2>&1
echo "t11 5e-4 exit $?" >> $O
