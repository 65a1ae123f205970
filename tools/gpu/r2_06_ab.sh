#!/bin/bash
# round 2, call 6: per-box Gram assembly + skinny column A/B, host-input e2e parity test, c3/c5 traces, bench c5
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_triangular.py -x -q > gpurun_out/r2_pytest_call6.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call6.txt
for v in "RSRS_ASSEMBLE=slot RSRS_SKINNY_COLS=128" "RSRS_ASSEMBLE=box RSRS_SKINNY_COLS=128" "RSRS_ASSEMBLE=box RSRS_SKINNY_COLS=512"; do
  tag=$(echo $v | tr ' =' '__')
  env $v CFG=c3 RUNS=1216:2 ITERS=2 RSRS_TRACE=1 python tools/quick_c2.py > gpurun_out/r2_c3_$tag.log 2>&1
done
echo "c3 ab exit $?" >> gpurun_out/r2_call6.txt
python bench.py > gpurun_out/r2_bench_c5_v2.json 2> gpurun_out/r2_bench_c5_v2.err
echo "bench exit $?" >> gpurun_out/r2_call6.txt
