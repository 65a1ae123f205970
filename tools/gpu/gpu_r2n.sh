cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2>/dev/null; echo "c4 $?"
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2>/dev/null; echo "c5 $?"
for f in c4 c5; do python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
