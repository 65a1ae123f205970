#!/bin/bash
# round 2, call 36: ncu launch list of the bench command on c3 (the c5 command cannot pass the box's
# 300-s pre-run without ncu: its sampling alone takes 250 s) and one ncu --set full capture of a
# leaf-level nn_stream_kernel launch (c3)
mkdir -p gpurun_out
O=gpurun_out/r2_call36.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c36_launches_c3_bench.csv \
   python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_c36_launches_c3_bench.log 2>&1
echo "launches c3 bench exit $?" > $O
gzip -f gpurun_out/r2_c36_launches_c3_bench.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_stream_kernel -s 12 -c 1 -o gpurun_out/r2_c36_nnstream \
   env CFG=c3 RUNS=1216:2 ITERS=1 PROF=none python tools/quick_c2.py > gpurun_out/r2_c36_ncu_nnstream.log 2>&1
echo "ncu nn_stream exit $?" >> $O
ncu -i gpurun_out/r2_c36_nnstream.ncu-rep --page raw --csv > gpurun_out/r2_c36_nnstream_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2_c36_nnstream.ncu-rep > gpurun_out/r2_c36_nnstream_summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/r2_c36_nnstream.ncu-rep >> gpurun_out/r2_c36_nnstream_summary.txt 2>&1
