"""Quick device-resident timing of one config (development aid)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_batch

def run(name, img, spec, reps=5):
    t = torch.from_numpy(img).cuda().unsqueeze(0)
    params = FilterParams(shape=ShapeSpec(*spec))
    out = filter_batch(t, params)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); filter_batch(t, params, out=out, check=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    h, w = img.shape[:2]; c = img.shape[2] if img.ndim == 3 else 1
    print(json.dumps({"cfg": name, "ms": round(ms, 3), "MP/s": round(h*w/1e3/ms, 1), "chMP/s": round(h*w*c/1e3/ms, 1)}), flush=True)
    return out

which = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
if "c1" in which: run("c1", C.baseline_input("c1"), ("circle", 8, 0, 0.0))
if "c2" in which: run("c2", C.baseline_input("c2"), ("circle", 48, 0, 0.0))
if "c3" in which:
    img = C.baseline_input("c3")
    for r in (2, 8, 32, 48, 64, 100): run(f"c3 r{r}", img, ("circle", r, 0, 0.0), reps=3)
if "c4" in which:
    img = C.baseline_input("c4")
    for s in C.C4_SHAPES: run(f"c4 {s}", img, s, reps=3)
