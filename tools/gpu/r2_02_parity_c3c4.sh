#!/bin/bash
# round 2, call 2: n_r > 64 parity tests, full-size parity c3 and c4
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity_full.py -k redundant -x -q > gpurun_out/r2_pytest_bigbox.log 2>&1
echo "bigbox exit $?" > gpurun_out/r2_call2.txt
for c in c3 c4; do
  python tests/parity_full.py --config $c --out gpurun_out/r02_parity_$c.json > gpurun_out/r2_parity_$c.log 2>&1
  echo "$c exit $?" >> gpurun_out/r2_call2.txt
done
