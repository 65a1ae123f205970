#!/bin/bash
# round 2, call 14 (re-entry): GPU suite + smoke at HEAD, solve timings, bench lines c2/c3/c4
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2_pytest_gpu_c14.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call14.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_c14.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2_call14.txt
for c in c2 c3; do
  CFG=$c timeout 600 python tools/solve_bench.py > gpurun_out/r2_solve_$c.json 2> gpurun_out/r2_solve_$c.err
  echo "solve $c exit $?" >> gpurun_out/r2_call14.txt
done
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
  echo "bench $c exit $?" >> gpurun_out/r2_call14.txt
done
