set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=c2 RUNS=768:2 ITERS=4 PROF=last timeout 900 python tools/quick_c2.py > gpurun_out/c2_prof_last.log 2>&1
CFG=c4 RUNS=768:2 ITERS=4 PROF=none timeout 900 python tools/quick_c2.py > gpurun_out/c4_prof_none.log 2>&1
grep iter gpurun_out/c2_prof_last.log gpurun_out/c4_prof_none.log
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1
echo "ncu exit $?"
python tools/launch_summary.py gpurun_out/launches_c2.csv
