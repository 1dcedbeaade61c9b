#!/bin/bash
# GPU iteration with a profile of the top kernel:  gpu_prof.sh <kernel-regex> <quick_bench args...>
mkdir -p gpurun_out
k=${1:-k2_}; shift
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/quick_bench.py ${@:-c2} > gpurun_out/quick.log 2>&1
cut -c1-200 gpurun_out/quick.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/prof -f python scripts/quick_bench.py c2 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
