#!/bin/bash
# round 2, call 32: whole GPU suite + smoke on the restored tree, default bench (c5), reference arm
mkdir -p gpurun_out
O=gpurun_out/r2_call32.txt
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2_c32_pytest_gpu.log 2>&1
echo "pytest exit $?" > $O
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_c32_smoke.log 2>&1
echo "smoke exit $?" >> $O
( time timeout 1800 python bench.py > gpurun_out/r2_c32_bench_c5.json 2> gpurun_out/r2_c32_bench_c5.err ) 2>> $O
echo "bench c5 exit $?" >> $O
( time timeout 900 python bench.py --impl reference > gpurun_out/r2_c32_bench_ref.json 2> gpurun_out/r2_c32_bench_ref.err ) 2>> $O
echo "bench ref exit $?" >> $O
