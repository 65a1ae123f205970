#!/bin/bash
# round 2, call 1: host probe + full-size parity c2 and the deep sphere (c3 family at N=65536)
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r2_host.txt 2>&1
python tests/parity_full.py --config c2 --out gpurun_out/r02_parity_c2.json > gpurun_out/r2_parity_c2.log 2>&1
echo "c2 exit $?" >> gpurun_out/r2_host.txt
python tests/parity_full.py --config c3@65536 --out gpurun_out/r02_parity_c3_65536.json > gpurun_out/r2_parity_c3_65536.log 2>&1
echo "c3@65536 exit $?" >> gpurun_out/r2_host.txt
