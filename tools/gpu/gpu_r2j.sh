cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 $?"; tail -c 600 gpurun_out/bench_c2.json
timeout 600 python bench.py --variant symmetric --no-cpu > gpurun_out/bench_sym.json 2>/dev/null; echo "sym $?"
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2>/dev/null; echo "c3 $?"
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2>/dev/null; echo "c4 $?"
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2>/dev/null; echo "c5 $?"
for f in c2 sym c3 c4 c5; do python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c2_v6.csv $CMD > gpurun_out/ncu.log 2>&1; echo "ncu $?"
python tools/launch_summary.py gpurun_out/launches_c2_v6.csv | head -32
