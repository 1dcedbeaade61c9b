"""The launch planner, on the host (no GPU): imf_plan_info reports the plan the
library would use.  The tile footprint -- the input pixels some window of the
tile contains, i.e. the Minkowski sum of the output rectangle and the kernel
(the reference's _footprint_mask, tiling.py:148-162) -- must equal a brute-force
construction from the kernel's own span table, for every convex shape."""
import ctypes

import numpy as np
import pytest

from paper_2505_22938_b200 import ShapeSpec, _lib, make_kernel
from paper_2505_22938_b200.tiling import _kernel_struct

KEYS = ["Tw", "Th", "Sw", "Sh", "N", "Npad", "tiles", "chunk", "lanes", "k2", "fp", "tma", "hs", "G",
        "ws", "k1"]


def plan(shape_hw_c, spec, dtype=1, boundary=0, aligned=True):
    L = _lib.load()
    h, w, c = shape_hw_c
    k = make_kernel(spec)
    ks, keep = _kernel_struct(k)
    img = _lib.ImfImage(0x1000 if aligned else 0x1002, dtype, 1, h, w, c, 0, w * c, c, 1)
    opt = _lib.ImfOptions(boundary, 0, 0, 0)
    info = (ctypes.c_int64 * 16)()
    assert L.imf_plan_info(ctypes.byref(img), ctypes.byref(ks), ctypes.byref(opt), info) == 0
    return dict(zip(KEYS, list(info))), k


def brute_footprint(k, Tw, Th, Sw, Sh, r):
    mask = np.zeros((Sh, Sw), bool)
    for dy, xlo, xhi in zip(k.row_dy, k.row_xlo, k.row_xhi):
        if xhi <= xlo:
            continue
        for cy in range(r, r + Th):
            y = cy + dy
            if 0 <= y < Sh:
                mask[y, max(0, r + xlo):min(Sw, r + Tw - 1 + xhi)] = True
    return int(mask.sum())


@pytest.mark.parametrize("spec", [ShapeSpec("circle", 48), ShapeSpec("circle", 8), ShapeSpec("circle", 64),
                                  ShapeSpec("regular_polygon", 32, sides=6),
                                  ShapeSpec("regular_polygon", 32, sides=12),
                                  ShapeSpec("regular_polygon", 20, sides=5, rotation_deg=17.0),
                                  ShapeSpec("regular_polygon", 40, sides=3, rotation_deg=90.0)])
def test_footprint_is_the_minkowski_sum(spec):
    p, k = plan((2160, 3840, 3), spec)
    assert p["k2"] == 2 and p["fp"] == 1
    assert p["N"] == brute_footprint(k, p["Tw"], p["Th"], p["Sw"], p["Sh"], spec.radius)
    assert p["N"] < p["Sw"] * p["Sh"]


def test_c2_plan():
    p, k = plan((2160, 3840, 3), ShapeSpec("circle", 48))
    assert (p["Tw"], p["Th"], p["Sw"], p["Sh"]) == (64, 64, 160, 160)
    assert p["N"] == 23584 and p["tiles"] == 60 * 34 * 3 and p["lanes"] == 2
    assert p["tma"] == 0  # interleaved HWC: per-lane loads
    assert p["k1"] == 3   # counting sort


def test_planar_u16_uses_tma_when_aligned():
    p, _ = plan((4320, 7680, 1), ShapeSpec("circle", 64))
    assert p["tma"] == 1 and p["hs"] == 1  # c5: TMA tile boxes, halved ranks (N > 32768)
    p, _ = plan((4321, 7681, 1), ShapeSpec("circle", 64))
    assert p["tma"] == 0                   # rows of 15,362 bytes are not 16-byte multiples


def test_square_has_no_footprint():
    p, _ = plan((2160, 3840, 3), ShapeSpec("square", 32), dtype=0)
    assert p["fp"] == 0 and p["N"] == p["Sw"] * p["Sh"]


@pytest.mark.parametrize("r", [8, 32, 64, 100])
def test_f32_bucket_plans_rank_the_footprint(r, monkeypatch):
    spec = ShapeSpec("circle", r)
    p, _ = plan((2048, 2048, 1), spec, dtype=2)
    assert p["fp"] == (0 if r == 64 else 1)  # auto: not on the 16-bit-entry kernel (S 161..192)
    monkeypatch.setenv("IMF_F32_FOOTPRINT", "2")
    p, k = plan((2048, 2048, 1), spec, dtype=2)
    assert p["fp"] == 1 and p["k1"] in (1, 2)
    assert p["N"] == brute_footprint(k, p["Tw"], p["Th"], p["Sw"], p["Sh"], r) < p["Sw"] * p["Sh"]


def test_large_u16_tiles_use_the_global_counting_sort():
    p, _ = plan((1024, 1024, 1), ShapeSpec("circle", 100))
    assert p["k1"] == 4 and p["Sw"] > 192


def test_direct_selection_for_tiny_windows():
    p, _ = plan((512, 512, 1), ShapeSpec("circle", 2), dtype=2)
    assert p["k2"] == 0


def test_kernel_static_shared_memory_within_the_planner_reservations():
    """The planner sizes dynamic shared memory as opt-in minus a per-family
    static reservation (imf_api.cu kStaticK1*): every built kernel's own static
    shared memory (cuobjdump SHARED minus the 1 KB system reserve) must fit."""
    import os
    import re
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-res-usage", _lib.LIB_PATH], capture_output=True, text=True).stdout
    limits = {"k1_sort": 2048, "k1_f32_bucket": 4096, "k1_count": 1024, "k2_": 1024, "k_direct": 1024,
              "k2_select": 1024}
    seen = 0
    for name, shared in re.findall(r"Function (\S+):\s*\n\s*REG:\d+ STACK:\d+ SHARED:(\d+)", out):
        for prefix, lim in limits.items():
            if re.search(r"\d" + prefix, name):
                seen += 1
                assert int(shared) - 1024 <= lim, (name, shared, lim)
                break
    assert seen > 50


def test_random_plans_are_consistent():
    """Seeded random geometries: the plan's tile counts, padding, footprint and
    workspace agree with each other and with imf_workspace_size."""
    import numpy as np
    rng = np.random.default_rng(123)
    L = _lib.load()
    for _ in range(150):
        dt = int(rng.integers(0, 3))
        kind = str(rng.choice(["circle", "square", "regular_polygon"]))
        r = int(rng.integers(0, 125))
        spec = ShapeSpec(kind, r, sides=int(rng.integers(3, 13)), rotation_deg=float(rng.uniform(0, 360))) \
            if kind == "regular_polygon" else ShapeSpec(kind, r)
        h, w, c = int(rng.integers(1, 3000)), int(rng.integers(1, 3000)), int(rng.choice([1, 3]))
        p, k = plan((h, w, c), spec, dtype=dt)
        assert p["N"] <= p["Sw"] * p["Sh"] and p["Npad"] == (p["N"] + 63) // 64 * 64
        assert p["Sw"] <= 255 and p["Sh"] <= 255 and p["Sw"] - p["Tw"] == 2 * r
        tiles = -(-h // p["Th"]) * -(-w // p["Tw"]) * c
        assert p["tiles"] == tiles and 1 <= p["chunk"] <= tiles
        if p["fp"]:
            assert p["N"] == brute_footprint(k, p["Tw"], p["Th"], p["Sw"], p["Sh"], r)
        ks, keep = _kernel_struct(k)
        img = _lib.ImfImage(0x1000, dt, 1, h, w, c, 0, w * c, c, 1)
        opt = _lib.ImfOptions(0, 0, 0, 0)
        assert L.imf_workspace_size(ctypes.byref(img), ctypes.byref(ks), ctypes.byref(opt)) == p["ws"]
