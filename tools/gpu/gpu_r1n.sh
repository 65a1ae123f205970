cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_nt_kernel -s 0 -c 1 -o gpurun_out/prof_nt $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_nt_kernel --csv --log-file gpurun_out/nt_traffic.csv $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?"
python tools/traffic_from_ncu.py gpurun_out/nt_traffic.csv gpurun_out/ncu_traffic.json
