"""Run one BASELINE configuration a few times (target for ncu captures).

    python scripts/one_config.py c2|c4hex|c4sq|c4dodec|c5|c3r64|c3r100|c1
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.tiling import run_device

CFG = {"c1": ("c1", ("circle", 8, 0)), "c2": ("c2", ("circle", 48, 0)),
       "c4hex": ("c4", ("regular_polygon", 32, 6)), "c4sq": ("c4", ("square", 32, 0)),
       "c4dodec": ("c4", ("regular_polygon", 32, 12)), "c5": ("c5", ("circle", 64, 0)),
       "c3r64": ("c3", ("circle", 64, 0)), "c3r100": ("c3", ("circle", 100, 0))}
name, (src, (kind, r, sides)) = sys.argv[1], CFG[sys.argv[1]]
t = torch.from_numpy(C.baseline_input(src)).cuda().unsqueeze(0)
p = FilterParams(shape=ShapeSpec(kind, r, sides=sides))
for _ in range(3):
    run_device(t, p, batched=True)
torch.cuda.synchronize()
