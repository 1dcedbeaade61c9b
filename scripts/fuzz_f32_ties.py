"""Large tie-heavy f32 frames (quantized normals, flat corners, circles and
polygons r=32..100) against the C oracle, with and without the f32 footprint
(dev aid):  python scripts/fuzz_f32_ties.py"""
import sys, numpy as np, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
import os
bad = 0
for seed in range(12):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(600, 1100)), int(rng.integers(600, 1100))
    q = float(rng.choice([0.05, 0.5, 4.0]))
    img = (np.round(rng.standard_normal((h, w)) * q) / q).astype(np.float32)
    if seed % 3 == 0: img[:200, :300] = 7.0
    r = int(rng.choice([32, 48, 64, 80, 100]))
    kind = rng.choice(["circle", "regular_polygon"])
    spec = ShapeSpec(kind, r, sides=int(rng.integers(3, 9)), rotation_deg=float(rng.uniform(0, 90))) if kind == "regular_polygon" else ShapeSpec(kind, r)
    for fp in ("1", "2"):
        os.environ["IMF_F32_FOOTPRINT"] = fp
        p = FilterParams(shape=spec, percentile=float(rng.random()))
        t0 = time.time(); got = filter_image(img, p); t1 = time.time()
        want = oracle.fast_filter(img, spec, p.percentile)
        ok = got.tobytes() == want.tobytes(); bad += not ok
        print(seed, (h, w), q, spec.kind, r, fp, "OK" if ok else "MISMATCH", round(t1 - t0, 3), round(time.time() - t1, 2), flush=True)
print("bad", bad)
