#!/bin/bash
# One GPU session: build check, parity suite, quick sweep, bench, launch list, ncu capture.
#   gpurun -- bash scripts/gpu_check.sh [tests|bench|ncu|all]
set -x
mode=${1:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $mode == all || $mode == tests ]]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
if [[ $mode == all || $mode == bench ]]; then
  timeout 900 python scripts/quick_bench.py c1 c2 c3 c4 c5 > gpurun_out/quick.log 2>&1
  timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
fi
if [[ $mode == all || $mode == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 2 -c 1 \
    -o gpurun_out/prof_k2 -f python scripts/quick_bench.py c2 > gpurun_out/ncu_k2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 1 \
    -o gpurun_out/prof_k1 -f python scripts/quick_bench.py c2 > gpurun_out/ncu_k1.log 2>&1
fi
ls -la gpurun_out
