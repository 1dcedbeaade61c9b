#!/bin/bash
# A/B: phase-D refine modes (0 both walks per iteration, 1 in sequence, 2 cooperative tail)
mkdir -p gpurun_out
IMF_REFINE=2 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/exp_tests.log 2>&1; tail -2 gpurun_out/exp_tests.log
for v in 0 1 2; do IMF_REFINE=$v python scripts/quick_bench.py c2 c4 c5 | sed "s/^/REFINE=$v /"; done > gpurun_out/exp.log 2>&1
cut -c1-200 gpurun_out/exp.log
