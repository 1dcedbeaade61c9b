"""Pinned host->device / device->host copy bandwidth with 1..4 concurrent streams (dev aid)."""
import torch
n = 50 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 1, 2, 4, 1):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    for direction in ("h2d", "d2h"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for rep in range(5):
            for i, s in enumerate(ss):
                s.wait_event(e0) if rep == 0 else None
                with torch.cuda.stream(s):
                    a, b = i * n // ns, (i + 1) * n // ns
                    if direction == "h2d": d[a:b].copy_(h[a:b], non_blocking=True)
                    else: h[a:b].copy_(d[a:b], non_blocking=True)
        for s in ss: e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        print(f"{direction} streams={ns}: {5 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
