"""Bucket-size statistics of the f32 bucket K1 (dev aid; scripts/libstats.so built
with -DIMF_STATS):  python scripts/rstats.py R"""
import ctypes, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ["IMF_LIB"] = os.path.join(HERE, "libstats.so")
sys.path.insert(0, os.path.dirname(HERE)); sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib
from paper_2505_22938_b200.tiling import run_device
r = int(sys.argv[1])
t = torch.from_numpy(C.baseline_input("c3")).cuda().unsqueeze(0)
L = _lib.lib(); L.imf_rstats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 128)(); L.imf_rstats(buf, 1)
run_device(t, FilterParams(shape=ShapeSpec("circle", r)), batched=True); torch.cuda.synchronize()
L.imf_rstats(buf, 0); h = np.array(buf[:64], dtype=np.float64); ph = np.array(buf[64:88], dtype=np.float64); i = np.arange(64)
print("r", r, "entries", int(h.sum()), "mean bucket size per entry %.2f" % ((h * i).sum() / h.sum()))
print({int(k): int(v) for k, v in zip(i, h) if v})
print("phases (sum Mcycles, max Kcycles):", [(round(ph[2*k]/1e6, 1), round(ph[2*k+1]/1e3, 1)) for k in range(12)])
