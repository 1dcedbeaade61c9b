"""Time one synthetic case (dev aid): quick_one.py DTYPE H W C R [reps]"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib, make_kernel
from paper_2505_22938_b200.tiling import run_device
dt, H, W, C, R = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
rng = np.random.default_rng(3)
shape = (H, W, C) if C > 1 else (H, W)
img = rng.standard_normal(shape).astype(np.float32) if dt == "f32" else \
    rng.integers(0, 65536 if dt == "u16" else 256, shape).astype(np.uint16 if dt == "u16" else np.uint8)
t = torch.from_numpy(img).cuda().unsqueeze(0)
params = FilterParams(shape=ShapeSpec("circle", R)); k = make_kernel(params.shape)
out = run_device(t, params, batched=True, kernel=k)
L = _lib.lib(); k1 = []; k2 = []
for _ in range(reps):
    run_device(t, params, out=out, batched=True, check=False, kernel=k, profile=True)
    a, b, tl = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32()
    L.imf_profile_last(ctypes.byref(a), ctypes.byref(b), None, None, ctypes.byref(tl), None)
    k1.append(a.value); k2.append(b.value)
print(json.dumps({"case": sys.argv[1:6], "k1": round(float(np.median(k1)), 3), "k2": round(float(np.median(k2)), 3), "tile": tl.value}))
