#!/bin/bash
# round 2, call 25: bench lines of the other configurations (no CPU leg) and the f2 / f4 / f1 variants
mkdir -p gpurun_out
O=gpurun_out/r2_call25.txt
for c in c2 c3 c4 t11; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/r2_c25_bench_$c.json 2> gpurun_out/r2_c25_bench_$c.err
  echo "bench $c exit $?" >> $O
done
timeout 900 python bench.py --config c2 --variant symmetric --no-cpu > gpurun_out/r2_c25_bench_c2_sym.json 2> gpurun_out/r2_c25_bench_c2_sym.err
echo "c2 sym exit $?" >> $O
timeout 900 python bench.py --config c3 --variant symmetric --triangular --no-cpu > gpurun_out/r2_c25_bench_c3_tri.json 2> gpurun_out/r2_c25_bench_c3_tri.err
echo "c3 tri exit $?" >> $O
timeout 900 python bench.py --config c3 --noise-factor 4 --no-cpu > gpurun_out/r2_c25_bench_c3_noise.json 2> gpurun_out/r2_c25_bench_c3_noise.err
echo "c3 noise exit $?" >> $O
