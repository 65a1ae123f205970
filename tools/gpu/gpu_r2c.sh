cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_gpu.log; grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -5
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_default.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
export CFG=c3 RUNS=1216:2 ITERS=1 PROF=none
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c3.csv python tools/quick_c2.py > gpurun_out/ncu_l.log 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_diag -s 60 -c 2 -o gpurun_out/prof_diag_c3 python tools/quick_c2.py > gpurun_out/ncu_d.log 2>&1; echo "ncu diag exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_nn -s 80 -c 8 -o gpurun_out/prof_nn_c3 python tools/quick_c2.py > gpurun_out/ncu_n.log 2>&1; echo "ncu nn exit $?"
python tools/launch_summary.py gpurun_out/launches_c3.csv | head -30
