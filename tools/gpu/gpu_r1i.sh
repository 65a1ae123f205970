cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c2_v3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1
echo "ncu exit $?"
python tools/launch_summary.py gpurun_out/launches_c2_v3.csv
