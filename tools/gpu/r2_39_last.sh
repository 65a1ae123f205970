#!/bin/bash
# round 2, call 39: final defaults (nn_stream ring depth 2): smoke, parity / determinism / stream variants, default bench (c5)
mkdir -p gpurun_out
O=gpurun_out/r2_call39.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_c39_smoke.log 2>&1
echo "smoke exit $?" > $O
timeout 1800 python bench.py > gpurun_out/r2_c39_bench_c5.json 2> gpurun_out/r2_c39_bench_c5.err
echo "bench c5 exit $?" >> $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x > gpurun_out/r2_c39_pytest.log 2>&1
echo "pytest exit $?" >> $O
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "bit_identical or no_nn_stream" > gpurun_out/r2_c39_pytest_var.log 2>&1
echo "pytest variants exit $?" >> $O
