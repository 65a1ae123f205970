cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_gpu.log; grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -5
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 $?"
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2>/dev/null; echo "c3 $?"
timeout 600 python bench.py --variant symmetric --no-cpu > gpurun_out/bench_sym.json 2>/dev/null; echo "sym $?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>/dev/null; echo "ref $?"
for f in c2 c3 sym; do python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
tail -c 400 gpurun_out/bench_ref.json
