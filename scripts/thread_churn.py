"""300 short-lived host threads each filtering through imf_filter_host (and
filter_multi every 50): per-thread CUDA resources are released at thread
exit (dev aid):  python scripts/thread_churn.py"""
import sys, threading, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_multi
from paper_2505_22938_b200.tiling import run_host
img = np.random.default_rng(0).integers(0, 65536, (300, 260, 3)).astype(np.uint16)
p = FilterParams(shape=ShapeSpec("circle", 12))
want = oracle.fast_filter(img, p.shape, 0.5)
t0 = time.time()
for i in range(300):
    res = {}
    th = threading.Thread(target=lambda: res.setdefault("o", run_host(img, p)))
    th.start(); th.join()
    assert res["o"].tobytes() == want.tobytes()
    if i % 50 == 0:
        assert filter_multi(img, p, devices=[0, 0]).tobytes() == want.tobytes()
print("300 thread lifetimes ok", round(time.time() - t0, 2), "s")
