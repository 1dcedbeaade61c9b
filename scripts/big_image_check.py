"""Large-offset check (dev aid): a 2+ GB frame (BIG_DTYPE u16 / u8) through the device path;
the last rows (byte offsets past 2^31) are compared with the oracle run on a
bottom band of the frame (the filter is local: rows >= r from the band's top
edge see the same windows)."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.tiling import run_device

H, W = int(sys.argv[1]) if len(sys.argv) > 1 else 33000, int(sys.argv[2]) if len(sys.argv) > 2 else 33000
DT = os.environ.get("BIG_DTYPE", "u16")
for r in (5, 40):
    g = torch.Generator(device="cuda").manual_seed(1)
    if DT == "u8":
        t = torch.randint(0, 256, (H, W), device="cuda", dtype=torch.uint8, generator=g)
    else:
        t = torch.randint(0, 65536, (H, W), device="cuda", dtype=torch.int32, generator=g).to(torch.uint16)
    params = FilterParams(shape=ShapeSpec("circle", r))
    t0 = time.time(); out = run_device(t, params); torch.cuda.synchronize(); t1 = time.time()
    band = t[H - 300:].cpu().numpy()
    want = oracle.fast_filter(band, params.shape, 0.5)
    got = out[H - 300:].cpu().numpy()
    ok = np.array_equal(got[r:], want[r:])
    print(f"{H}x{W} {DT} r={r}: {t1 - t0:.2f} s device, {t.numel() / 2**30:.2f} G elements, last-rows parity {ok}",
          flush=True)
    del t, out
    torch.cuda.empty_cache()
