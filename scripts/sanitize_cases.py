"""Small cases over every engine path, for compute-sanitizer (dev aid):
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
Each case is also checked against the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image, filter_image_bracket
from paper_2505_22938_b200.tiling import run_host

rng = np.random.default_rng(3)
cases = [
    ("uint16", (150, 170, 3), ("circle", 20, 0, 0.0), {}),
    ("uint16", (150, 170), ("circle", 40, 0, 0.0), {}),                    # TMA (planar)
    ("uint16", (130, 140), ("circle", 62, 0, 0.0), {}),                    # halved ranks, omega in L2
    ("uint16", (270, 260), ("circle", 100, 0, 0.0), {}),                   # k1_count_g, wide circle
    ("uint8", (120, 130, 3), ("regular_polygon", 20, 6, 10.0), {}),
    ("uint8", (120, 130), ("square", 9, 0, 0.0), {}),
    ("uint8", (120, 130, 3), ("regular_polygon", 20, 6, 0.0), {}),         # symmetric polygon (VABSDIFF4 + table)
    ("uint8", (140, 130), ("regular_polygon", 24, 12, 0.0), {}),
    ("uint8", (90, 100), ("regular_polygon", 30, 3, 29.0), {"IMF_PAIR": "0"}),  # general path
    ("float32", (140, 150), ("circle", 2, 0, 0.0), {}),                    # direct
    ("float32", (160, 170), ("circle", 20, 0, 0.0), {}),                   # f32 bucket, footprint
    ("float32", (200, 190), ("circle", 60, 0, 0.0), {}),                   # OWN16
    ("float32", (280, 270), ("circle", 100, 0, 0.0), {}),                  # bucket_g, corner runs
    ("float32", (60, 242), ("regular_polygon", 34, 3, 29.3), {"IMF_MAXSUMSQ_K": "0"}),  # LSD fallback
    ("float32", (150, 160), ("circle", 30, 0, 0.0), {"IMF_RUNMIN": "2", "IMF_F32_FOOTPRINT": "2"}),
]
bad = 0
for dt, shape, spec, env in cases:
    os.environ.update(env)
    img = (rng.standard_normal(shape).astype(np.float32) if dt == "float32"
           else rng.integers(0, 256 if dt == "uint8" else 65536, shape).astype(dt))
    p = FilterParams(shape=ShapeSpec(*spec), percentile=0.4)
    want = oracle.fast_filter(img, p.shape, 0.4)
    ok = filter_image(img, p).tobytes() == want.tobytes()
    ok &= run_host(img, p).tobytes() == want.tobytes()
    ok &= filter_image_bracket(img, p, [0.4])[0].tobytes() == want.tobytes()
    print(dt, shape, spec, env, "OK" if ok else "MISMATCH", flush=True)
    bad += not ok
    for k in env:
        del os.environ[k]
torch.cuda.synchronize()
print("mismatches", bad)
