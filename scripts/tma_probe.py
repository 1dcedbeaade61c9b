"""dev aid: one small planar u8 filter (TMA K1 path) for compute-sanitizer."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_batch, _lib
img = np.random.default_rng(1).integers(0, 256, (1, 256, 256), dtype=np.uint8)
out = filter_batch(torch.from_numpy(img).cuda(), FilterParams(shape=ShapeSpec("circle", 8)))
torch.cuda.synchronize()
print("features", _lib.lib().imf_last_features(), out.float().mean().item())
