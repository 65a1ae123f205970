cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --variant symmetric --no-cpu > gpurun_out/bench_sym.json 2> gpurun_out/bench_sym.err; echo "sym exit $?"
tail -3 gpurun_out/bench_sym.err
python -c "import json; d=json.loads(open('gpurun_out/bench_sym.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['residual'], d['e2e']['value'])"
timeout 900 python bench.py --config c3 --no-cpu --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 exit $?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['residual'], d['e2e']['value'])"
timeout 900 python bench.py --config c4 --no-cpu --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 exit $?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['residual'], d['e2e']['value'])"
