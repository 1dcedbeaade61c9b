"""Quick device-resident timing of BASELINE configs (development aid).

    python scripts/quick_bench.py [c1 c2 c3 c4 c5]   (env IMF_TILE / IMF_SEED_ROWS / IMF_SEEDS tune)
"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib, make_kernel
from paper_2505_22938_b200.tiling import run_device

_PEAK = None


def int_peak():
    """Measured int32 add throughput of this GPU (imf_int_peak), ops/s."""
    global _PEAK
    if _PEAK is None:
        pk = ctypes.c_double()
        _lib.lib().imf_int_peak(ctypes.byref(pk), None)
        _PEAK = pk.value
    return _PEAK


def run(name, img, spec, reps=5, gold=None):
    t = torch.from_numpy(img).cuda().unsqueeze(0)
    params = FilterParams(shape=ShapeSpec(*spec))
    k = make_kernel(params.shape)
    out = run_device(t, params, batched=True)
    ok = None if gold is None else C.digest(out[0].cpu().numpy()) == gold
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L = _lib.lib(); ts = []; k1 = []; k2 = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run_device(t, params, out=out, batched=True, check=False, kernel=k); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        run_device(t, params, out=out, batched=True, check=False, kernel=k, profile=True)
        a, b = ctypes.c_float(), ctypes.c_float(); tl = ctypes.c_int32(); qs = ctypes.c_int32()
        L.imf_profile_last(ctypes.byref(a), ctypes.byref(b), None, None, ctypes.byref(tl), ctypes.byref(qs))
        k1.append(a.value); k2.append(b.value)
    ms = float(np.median(ts))
    h, w = img.shape[:2]; c = img.shape[2] if img.ndim == 3 else 1
    W = 4 * len(k.col_dx) + 384
    print(json.dumps({"cfg": name, "ms": round(ms, 3), "k1_ms": round(float(np.median(k1)), 3),
                      "k2_ms": round(float(np.median(k2)), 3), "MP/s": round(h*w/1e3/ms, 1),
                      "chMP/s": round(h*w*c/1e3/ms, 1), "tile": tl.value, "qs": qs.value,
                      "path_frac": round(h*w*c/1e3/ms*1e6*W/int_peak(), 4),
                      "k2_frac": (round(h*w*c/1e3/float(np.median(k2))*1e6*W/int_peak(), 4)
                                  if np.median(k2) > 0 else None),
                      "peak_Tops": round(int_peak()/1e12, 2), "parity": ok,
                      "env": {k_: os.environ.get(k_) for k_ in ("IMF_TILE", "IMF_SEED_ROWS", "IMF_SEEDS") if os.environ.get(k_)}}), flush=True)

which = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["baseline"]
if "c1" in which: run("c1", C.baseline_input("c1"), ("circle", 8, 0, 0.0), gold=gold["c1"])
if "c2" in which: run("c2", C.baseline_input("c2"), ("circle", 48, 0, 0.0), gold=gold["c2"])
if "c3" in which:
    img = C.baseline_input("c3")
    for r in (2, 8, 16, 32, 48, 64, 100): run(f"c3 r{r}", img, ("circle", r, 0, 0.0), reps=3, gold=gold[f"c3/r{r}"])
if "c4" in which:
    img = C.baseline_input("c4")
    for s in C.C4_SHAPES: run(f"c4 {s[0]}{s[2]}", img, s, reps=3, gold=gold["c4/" + json.dumps(list(s))])
if "c2smooth" in which:  # SURVEY 8(d) refine-stress distribution at the c2 shape (parity vs the C oracle)
    import oracle
    img = C.smooth_image((2160, 3840, 3), np.uint16, 2)
    want = oracle.fast_filter(img, ShapeSpec("circle", 48), 0.5)
    run("c2smooth", img, ("circle", 48, 0, 0.0), gold=C.digest(want))
if "c5" in which:
    g5 = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_c5.json")))
    run("c5 img0", C.baseline_input("c5", 0), ("circle", 64, 0, 0.0), reps=3, gold=g5.get("0"))
