#!/bin/bash
# f32 K1 evidence: bucket statistics + phase cycles (stats build), ncu of the K1 kernels at r=64 / r=100
mkdir -p gpurun_out
for r in 48 64 100; do python scripts/rstats.py $r; done > gpurun_out/rstats.log 2>&1
cat > /tmp/c3one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests", "golden"))
import torch, cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.tiling import run_device
r = int(sys.argv[1]); t = torch.from_numpy(C.baseline_input("c3")).cuda().unsqueeze(0)
for _ in range(3): run_device(t, FilterParams(shape=ShapeSpec("circle", r)), batched=True)
torch.cuda.synchronize()
PY
for r in 64 100; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_f32 -s 2 -c 1 -o gpurun_out/prof_k1f32_r$r -f python /tmp/c3one.py $r > gpurun_out/ncu_f32_r$r.log 2>&1
done
cat gpurun_out/rstats.log
