#!/bin/bash
# round 2, call 13: ncu --set full of the 1-RHS solve kernels at c2's leaf level
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:solve_fwd_kernel \
    --launch-skip 0 --launch-count 1 -o gpurun_out/r2_c2_solvefwd -f env CFG=c2 python tools/solve_bench.py > gpurun_out/r2_ncu_solvefwd.log 2>&1
echo "ncu fwd exit $?" > gpurun_out/r2_call13.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:solve_bwd_kernel \
    --launch-skip 44 --launch-count 1 -o gpurun_out/r2_c2_solvebwd -f env CFG=c2 python tools/solve_bench.py > gpurun_out/r2_ncu_solvebwd.log 2>&1
echo "ncu bwd exit $?" >> gpurun_out/r2_call13.txt
