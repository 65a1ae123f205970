#!/bin/bash
# round 2, call 22: extraction rewrite (thread per near column / row, batched loads), batched loads in
# the Gram assembly and the Gram-block update, 16-row NT tiles only for wide launches: c2/c3 timing,
# parity of every path that runs the extraction (real, complex, symmetric, triangular, estimator)
mkdir -p gpurun_out
O=gpurun_out/r2_call22.txt
for c in c2 c3; do
  CFG=$c RUNS=$([ $c = c2 ] && echo 768:2 || echo 1216:2) ITERS=2 RSRS_TRACE=1 timeout 900 python tools/quick_c2.py > gpurun_out/r2_c22_$c.log 2>&1
  echo "$c exit $?" >> $O
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram_blocks.py tests/test_gpu_symmetric.py tests/test_gpu_triangular.py tests/test_gpu_coupling.py -q -x > gpurun_out/r2_c22_pytest.log 2>&1
echo "pytest exit $?" >> $O
