#!/bin/bash
# One iteration on the B200: parity suite (fast subset unless FULL=1) + device timings.
#   gpurun -- bash scripts/gpu_iter.sh [configs...]
mkdir -p gpurun_out
if [[ ${FULL:-0} == 1 ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/quick_bench.py ${@:-c2 c4 c5} > gpurun_out/quick.log 2>&1
cut -c1-220 gpurun_out/quick.log
