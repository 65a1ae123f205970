cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['factor_ms'], d['solve_ms'], d['residual'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'], d['clocks'])
for k,v in d['kernels'].items(): print(k, round(v['ms_per_step'],2), round(v['tflops'],2))"
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c2_v4.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu exit $?"
python tools/launch_summary.py gpurun_out/launches_c2_v4.csv | head -30
