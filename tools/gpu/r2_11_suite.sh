#!/bin/bash
# round 2, call 11: the whole GPU suite and smoke()
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=25 > gpurun_out/r2_pytest_gpu_full.log 2>&1
echo "pytest exit $?" > gpurun_out/r2_call11.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2_call11.txt
