#!/bin/bash
# round 2, call 37: bit-identity of the streaming / column-walking NN kernels against the tiled one,
# the stream variants' parity, and the gram-block / dist tests on the final tree
mkdir -p gpurun_out
O=gpurun_out/r2_call37.txt
timeout 1500 python -m pytest tests/test_gpu_variants.py -q -x -k "stream or bit_identical" --durations=5 > gpurun_out/r2_c37_pytest_var.log 2>&1
echo "pytest variants exit $?" > $O
timeout 900 python -m pytest tests/test_gpu_gram_blocks.py tests/test_gpu_dist.py tests/test_gpu_symmetric.py -q -x > gpurun_out/r2_c37_pytest.log 2>&1
echo "pytest exit $?" >> $O
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_c37_smoke.log 2>&1
echo "smoke exit $?" >> $O
