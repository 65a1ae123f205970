cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CFG=c3 RUNS=1216:2 ITERS=1 PROF=none
timeout 600 ncu --set full --clock-control none --import-source on -k regex:extract_lu -s 3 -c 1 -o gpurun_out/prof_extract_c3 python tools/quick_c2.py > gpurun_out/ncu_e.log 2>&1; echo "ncu extract exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nn_kernel" -s 40 -c 6 -o gpurun_out/prof_nn_c3b python tools/quick_c2.py > gpurun_out/ncu_n.log 2>&1; echo "ncu nn exit $?"
