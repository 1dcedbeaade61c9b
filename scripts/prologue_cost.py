"""Cost of run_host's Python prologue with the C call stubbed out, plus a
cProfile breakdown (dev aid):  python scripts/prologue_cost.py"""
import sys, time, ctypes
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np, torch
import cases as C
from paper_2505_22938_b200 import FilterParams, ShapeSpec, make_kernel, _lib
import paper_2505_22938_b200.tiling as T
img = C.baseline_input("c2"); host = torch.from_numpy(img).pin_memory().unsqueeze(0); out = torch.empty_like(host).pin_memory()
params = FilterParams(shape=ShapeSpec("circle", 48)); k = make_kernel(params.shape)
L = _lib.lib()
class Fake:
    def __getattr__(self, n):
        if n == "imf_filter_host": return lambda *a: 0
        return getattr(L, n)
orig = _lib.lib; _lib.lib = lambda: Fake()
for _ in range(100): T.run_host(host, params, out=out, batched=True, kernel=k)
t0 = time.perf_counter(); n = 2000
for _ in range(n): T.run_host(host, params, out=out, batched=True, kernel=k)
print("run_host prologue us:", (time.perf_counter() - t0) / n * 1e6)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(2000): T.run_host(host, params, out=out, batched=True, kernel=k)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
