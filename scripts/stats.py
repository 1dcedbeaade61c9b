"""Refine step statistics of k2_pair (dev aid; needs scripts/libstats.so, built
with -DIMF_STATS):  python scripts/stats.py [size]"""
import ctypes, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ["IMF_LIB"] = os.path.join(HERE, "libstats.so")
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib
from paper_2505_22938_b200.tiling import run_device
img = C.smooth_image((2160, 3840, 3), np.uint16, 2) if os.environ.get("STATS_IMG") == "smooth" else C.baseline_input("c2")
if len(sys.argv) > 1:
    n = int(sys.argv[1]); img = img[:n, :n]
t = torch.from_numpy(np.ascontiguousarray(img)).cuda().unsqueeze(0)
L = _lib.lib()
L.imf_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 256)()
L.imf_stats(buf, 1)
run_device(t, FilterParams(shape=ShapeSpec("circle", 48)), batched=True)
torch.cuda.synchronize()
L.imf_stats(buf, 0)
lane = np.array(buf[:64], dtype=np.float64); warp = np.array(buf[64:128], dtype=np.float64)
i = np.arange(64)
print("lane iterations per window pair: mean %.2f" % ((lane * i).sum() / lane.sum()))
print("warp trip count per pair-step:   mean %.2f  (lane efficiency %.2f)" % ((warp * i).sum() / warp.sum(), (lane * i).sum() / lane.sum() / ((warp * i).sum() / warp.sum())))
print("lane hist:", {int(k): int(v) for k, v in zip(i, lane) if v})
print("warp hist:", {int(k): int(v) for k, v in zip(i, warp) if v})

x = np.array(buf[128:134], dtype=np.float64)
if x[0]:
    print("pairs %d  same direction %.3f  mean |PA-PB| %.1f  mean walk A %.1f  B %.1f ranks  mean union (same dir) %.1f"
          % (x[0], x[1] / x[0], x[2] / x[0], x[3] / x[0], x[4] / x[0], x[5] / max(x[1], 1)))
