"""e2e (pinned host -> GPU -> host) per-image time of c5-size images vs batch size (dev aid)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, make_kernel
from paper_2505_22938_b200.tiling import run_host
params = FilterParams(shape=ShapeSpec("circle", 64)); k = make_kernel(params.shape)
base = C.baseline_input("c5", 0)
for nb in [int(x) for x in (sys.argv[1:] or ["1", "4", "16"])]:
    host = torch.from_numpy(np.stack([base] * nb)).pin_memory()
    out = torch.empty_like(host).pin_memory()
    run_host(host, params, out=out, batched=True, kernel=k); torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2): run_host(host, params, out=out, batched=True, kernel=k)
    e1.record(); torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 2 * 1e3
    print(json.dumps({"batch": nb, "ms_per_image_events": round(e0.elapsed_time(e1) / 2 / nb, 3),
                      "ms_per_image_wall": round(wall / nb, 3)}), flush=True)
