#!/bin/bash
# A/B experiments on c2 (device timing) + refine statistics
mkdir -p gpurun_out
python scripts/stats.py > gpurun_out/stats.log 2>&1
IMF_LIB=scripts/libstats.so IMF_REFINE=1 python scripts/stats.py > gpurun_out/stats_seq.log 2>&1
for v in 0 1; do IMF_REFINE=$v python scripts/quick_bench.py c2 c5 | sed "s/^/REFINE=$v /"; done > gpurun_out/exp.log 2>&1
IMF_REFINE=1 python -m pytest tests/test_gpu_full.py -x -q -k "c1_c2 or acceptance" > gpurun_out/exp_tests.log 2>&1; tail -2 gpurun_out/exp_tests.log
cat gpurun_out/stats.log gpurun_out/stats_seq.log gpurun_out/exp.log | cut -c1-250
