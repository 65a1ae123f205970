#!/bin/bash
# round 2, call 12: bench lines of the other configurations and the variants (f1 / f2 / f4)
mkdir -p gpurun_out
for c in c2 c3 c4 t11; do
  python bench.py --config $c > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
  echo "bench $c exit $?" >> gpurun_out/r2_call12.txt
done
python bench.py --config c2 --variant symmetric --no-cpu > gpurun_out/r2_bench_c2_sym.json 2> gpurun_out/r2_bench_c2_sym.err
python bench.py --config c4 --variant symmetric --no-cpu > gpurun_out/r2_bench_c4_sym.json 2> gpurun_out/r2_bench_c4_sym.err
python bench.py --config c3 --variant symmetric --triangular --no-cpu > gpurun_out/r2_bench_c3_tri.json 2> gpurun_out/r2_bench_c3_tri.err
python bench.py --config c3 --noise-factor 4 --no-cpu > gpurun_out/r2_bench_c3_noise.json 2> gpurun_out/r2_bench_c3_noise.err
echo "variants exit $?" >> gpurun_out/r2_call12.txt
