#!/bin/bash
# env sweep: gpu_sweep.sh "<cfgs>" "VAR=a VAR2=b" "VAR=c" ...
cfgs=$1; shift
mkdir -p gpurun_out; : > gpurun_out/sweep.log
for e in "$@"; do
  echo "== $e" >> gpurun_out/sweep.log
  env $e timeout 300 python scripts/quick_bench.py $cfgs >> gpurun_out/sweep.log 2>&1
done
cut -c1-170 gpurun_out/sweep.log
