cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['factor_ms'], d['solve_ms'], d['residual'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'], d['clocks'])"
for c in c3 c4; do
timeout 900 python bench.py --config $c --no-cpu --steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c exit $?"
python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['residual'], d['e2e']['value'])"
done
timeout 900 python bench.py --variant symmetric --no-cpu --steps 3 > gpurun_out/bench_sym.json 2> gpurun_out/bench_sym.err; echo "sym exit $?"
python -c "import json; d=json.loads(open('gpurun_out/bench_sym.json').read().strip().splitlines()[-1]); print(d['value'], d['factor_ms'], d['residual'], d['e2e']['value'])"
CFG=c5 RUNS=1216:2 ITERS=2 PROF=last RSRS_TRACE=1 timeout 1500 python tools/quick_c2.py > gpurun_out/c5_q.log 2>&1; echo "c5 exit $?"
grep -v "^sample" gpurun_out/c5_q.log | head -20
