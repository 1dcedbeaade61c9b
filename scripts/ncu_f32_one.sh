#!/bin/bash
# ncu --set full of one f32 bucket K1 launch at c3 radius $1 -> gpurun_out/prof_k1f32_r$1.ncu-rep
mkdir -p gpurun_out
cat > /tmp/c3one.py <<PY
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests", "golden"))
import torch, cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.tiling import run_device
r = int(sys.argv[1]); t = torch.from_numpy(C.baseline_input("c3")).cuda().unsqueeze(0)
for _ in range(3): run_device(t, FilterParams(shape=ShapeSpec("circle", r)), batched=True)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_f32 -s 2 -c 1 \
    -o gpurun_out/prof_k1f32_r$1 -f python /tmp/c3one.py $1 > gpurun_out/ncu_f32_r$1.log 2>&1
ls -la gpurun_out/prof_k1f32_r$1.ncu-rep; tail -2 gpurun_out/ncu_f32_r$1.log
