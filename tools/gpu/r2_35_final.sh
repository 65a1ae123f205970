#!/bin/bash
# round 2, call 35: default bench (c5) on the final tree, the ncu launch list of the same command
# (1 timed step, 1 warm-up, no CPU leg), one ncu --set full capture of a leaf-level nn_stream_kernel
# launch on c3, and the c3 / c2 bench lines
mkdir -p gpurun_out
O=gpurun_out/r2_call35.txt
timeout 1800 python bench.py > gpurun_out/r2_c35_bench_c5.json 2> gpurun_out/r2_c35_bench_c5.err
echo "bench c5 exit $?" > $O
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c35_launches_c5.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_c35_launches_c5.log 2>&1
echo "launches exit $?" >> $O
gzip -f gpurun_out/r2_c35_launches_c5.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_stream_kernel -s 30 -c 1 -o gpurun_out/r2_c35_nnstream \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c35_ncu_nnstream.log 2>&1
echo "ncu nn_stream exit $?" >> $O
timeout 900 python bench.py --config c3 --no-cpu > gpurun_out/r2_c35_bench_c3.json 2> gpurun_out/r2_c35_bench_c3.err
echo "bench c3 exit $?" >> $O
timeout 900 python bench.py --config c2 --no-cpu > gpurun_out/r2_c35_bench_c2.json 2> gpurun_out/r2_c35_bench_c2.err
echo "bench c2 exit $?" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/r2_c35_pytest.log 2>&1
echo "pytest exit $?" >> $O
