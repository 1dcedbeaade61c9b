#!/bin/bash
# Fast GPU iteration: parity suite + device timings of every BASELINE config.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/quick_bench.py ${@:-c1 c2 c3 c4 c5} > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log | cut -c1-200
