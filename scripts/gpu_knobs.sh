#!/bin/bash
# Sweep planner knobs on c2 (device-resident timing): gpurun -- bash scripts/gpu_knobs.sh
mkdir -p gpurun_out
out=gpurun_out/knobs.log; : > $out
for env in "" "IMF_SEED_ROWS=4" "IMF_SEED_ROWS=6" "IMF_SEED_ROWS=4 IMF_PAIR_OMG=1" "IMF_PAIR_OMG=1" \
           "IMF_GROUPED=0" "IMF_REFINE=0" "IMF_SEED_ROWS=4 IMF_GROUPED=0"; do
  echo "== $env" >> $out
  env $env timeout 300 python scripts/quick_bench.py ${CFG:-c2} 2>&1 | cut -c1-260 >> $out
done
cat $out
