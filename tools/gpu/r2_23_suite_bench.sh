#!/bin/bash
# round 2, call 23: the whole GPU suite + smoke on the current tree, then the default bench (c5)
mkdir -p gpurun_out
O=gpurun_out/r2_call23.txt
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2_c23_pytest_gpu.log 2>&1
echo "pytest exit $?" > $O
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_c23_smoke.log 2>&1
echo "smoke exit $?" >> $O
timeout 1800 python bench.py > gpurun_out/r2_c23_bench_c5.json 2> gpurun_out/r2_c23_bench_c5.err
echo "bench c5 exit $?" >> $O
