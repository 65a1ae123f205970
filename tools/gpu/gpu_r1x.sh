cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 exit $?"
tail -3 gpurun_out/bench_c5.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['solve_ms'], d['residual'], d['e2e']['value'], d['top_size'], d['max_rank'])"
