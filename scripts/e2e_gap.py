"""Host->host time of c2 split into the Python prologue, the C call and the gap
between calls (dev aid):  python scripts/e2e_gap.py"""
import os, sys, time, json, ctypes
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, make_kernel, _lib
from paper_2505_22938_b200.tiling import run_host
img = C.baseline_input("c2"); host = torch.from_numpy(img).pin_memory(); out = torch.empty_like(host).pin_memory()
params = FilterParams(shape=ShapeSpec("circle", 48)); k = make_kernel(params.shape)
L = _lib.lib(); f = L.imf_filter_host; tin = []
def wrapped(*a):
    t0 = time.perf_counter(); r = f(*a); tin.append(time.perf_counter() - t0); return r
class LW:
    def __getattr__(self, n): return wrapped if n == "imf_filter_host" else getattr(L, n)
import paper_2505_22938_b200._lib as LL
orig = LL.lib; LL.lib = lambda: LW()
for _ in range(3): run_host(host, params, out=out, kernel=k)
tin.clear()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
walls = []
for a, b in evs:
    t0 = time.perf_counter(); a.record(); run_host(host, params, out=out, kernel=k); b.record(); walls.append(time.perf_counter() - t0)
torch.cuda.synchronize()
per = [a.elapsed_time(b) for a, b in evs]; gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(9)]
print(json.dumps({"event_ms": round(float(np.median(per)), 3), "wall_ms": round(1e3 * float(np.median(walls)), 3),
                  "c_call_ms": round(1e3 * float(np.median(tin)), 3), "gap_between_calls_ms": round(float(np.median(gaps)), 3),
                  "e2e_over_10_ms": round(evs[0][0].elapsed_time(evs[-1][1]) / 10, 3)}))
