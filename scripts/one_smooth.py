"""One c2-shaped smooth-field filter call (for ncu; dev aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.tiling import run_device
t = torch.from_numpy(C.smooth_image((2160, 3840, 3), np.uint16, 2)).cuda().unsqueeze(0)
for _ in range(2): run_device(t, FilterParams(shape=ShapeSpec("circle", 48)), batched=True)
torch.cuda.synchronize()
