"""End-to-end (pinned host -> GPU -> pinned host) timing of c2 through the C-ABI
host entry for stripe settings given as ENV=VAL[,ENV=VAL] arguments (dev aid):
    python scripts/quick_e2e.py "" IMF_STRIPE_MID=12 IMF_STRIPE_MID=16,IMF_STRIPE_EDGE=2"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, make_kernel
from paper_2505_22938_b200.tiling import run_host
img = C.baseline_input("c2")
host = torch.from_numpy(img).pin_memory()
out = torch.empty_like(host).pin_memory()
params = FilterParams(shape=ShapeSpec("circle", 48)); k = make_kernel(params.shape)
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["baseline"]["c2"]
base = dict(os.environ)
for setting in (sys.argv[1:] or [""]):
    os.environ.clear(); os.environ.update(base)
    for kv in filter(None, setting.split(",")):
        kk, vv = kv.split("=")
        os.environ[kk] = vv
    for _ in range(3): run_host(host, params, out=out, kernel=k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run_host(host, params, out=out, kernel=k)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"setting": setting, "e2e_ms": round(ms, 3), "MP/s": round(3840*2160/1e3/ms, 1),
                      "parity": C.digest(out.numpy()) == gold}), flush=True)
