"""Randomized parity sweep: seeded random geometries, dtypes, kernel shapes,
boundaries, percentiles (scalar and per-pixel maps) and engine switches,
every output byte-compared with the C oracle (itself pinned to the
reference's golden outputs, tests/test_oracle.py).  Sized to run in well
under a minute (IMF_FUZZ_CASES=N for a longer sweep); each case prints its
parameters on failure."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ENVS = [{}, {}, {"IMF_F32_FOOTPRINT": "2"}, {"IMF_RUNMIN": "8"}, {"IMF_F32_FOOTPRINT": "0"},
        {"IMF_TILE": "40"}, {"IMF_PAIR": "0"}, {"IMF_MAXSUMSQ_K": "4"}]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    dt = rng.choice(["uint8", "uint16", "float32"])
    kind = rng.choice(["circle", "circle", "square", "regular_polygon"])
    r = int(rng.choice([1, 2, 3, 5, 8, 13, 21, 34, 47, 60, 70]))
    h, w = int(rng.integers(1, 260)), int(rng.integers(1, 260))
    c = int(rng.choice([1, 1, 3]))
    shape = (h, w) if c == 1 else (h, w, c)
    if dt == "float32":
        img = rng.standard_normal(shape).astype(np.float32)
        if rng.random() < 0.3:
            img = np.round(img * 4) / 4  # many ties
    else:
        hi = 256 if dt == "uint8" else int(rng.choice([16, 4096, 65536]))
        img = rng.integers(0, hi, shape).astype(dt)
    if kind == "regular_polygon":
        spec = (kind, r, int(rng.integers(3, 13)), float(rng.uniform(0, 360)))
    else:
        spec = (kind, r, 0, 0.0)
    boundary = "valid" if rng.random() < 0.25 and min(h, w) > 2 * r else "replicate"
    oh, ow = (h - 2 * r, w - 2 * r) if boundary == "valid" else (h, w)
    pct = rng.random((oh, ow)) if rng.random() < 0.2 else float(rng.choice([0.0, 0.5, 1.0, rng.random()]))
    env = ENVS[seed % len(ENVS)]
    return img, spec, boundary, pct, env


@pytest.mark.parametrize("seed", range(int(os.environ.get("IMF_FUZZ_CASES", "96"))))
def test_random_case_bit_exact(seed, monkeypatch):
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    img, spec, boundary, pct, env = _case(seed)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    params = FilterParams(shape=ShapeSpec(*spec), percentile=pct, boundary=boundary)
    got = filter_image(img, params)
    want = oracle.fast_filter(img, params.shape, pct, boundary)
    assert got.tobytes() == want.tobytes(), (seed, img.dtype, img.shape, spec, boundary, env,
                                             "map" if isinstance(pct, np.ndarray) else pct)


def _big_case(seed):
    rng = np.random.default_rng(5000 + seed)
    dt = rng.choice(["uint8", "uint16", "float32"])
    kind = rng.choice(["circle", "circle", "square", "regular_polygon"])
    r = int(rng.choice([8, 24, 48, 64, 90, 124]))
    h, w = int(rng.integers(130, 520)), int(rng.integers(60, 420))
    c = int(rng.choice([1, 3]))
    shape = (h, w) if c == 1 else (h, w, c)
    if dt == "float32":
        img = rng.standard_normal(shape).astype(np.float32)
    else:
        img = rng.integers(0, 256 if dt == "uint8" else int(rng.choice([4096, 65536])), shape).astype(dt)
    spec = (kind, r, int(rng.integers(3, 13)), float(rng.uniform(0, 360))) if kind == "regular_polygon" \
        else (kind, r, 0, 0.0)
    boundary = "valid" if rng.random() < 0.3 and min(h, w) > 2 * r else "replicate"
    return img, spec, boundary


@pytest.mark.parametrize("seed", range(int(os.environ.get("IMF_FUZZ_BIG", "12"))))
def test_random_host_pipeline_and_bracket(seed):
    """Larger random frames (up to r = 124) through the streamed host entry
    (imf_filter_host: row stripes over three streams) and the bracket (one K1
    per tile, one K2 per percentile)."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image_bracket
    from paper_2505_22938_b200.tiling import run_host
    img, spec, boundary = _big_case(seed)
    pcts = [0.1, 0.5, 0.93]
    params = FilterParams(shape=ShapeSpec(*spec), percentile=pcts[1], boundary=boundary)
    want = [oracle.fast_filter(img, params.shape, p, boundary) for p in pcts]
    got = run_host(img, params)
    assert got.tobytes() == want[1].tobytes(), ("host", seed, img.dtype, img.shape, spec, boundary)
    for p, g, wnt in zip(pcts, filter_image_bracket(img, params, pcts), want):
        assert g.tobytes() == wnt.tobytes(), ("bracket", p, seed, img.dtype, img.shape, spec, boundary)


def test_host_pipeline_workspace_covers_every_stripe():
    """Regression (found by the sweep above, seed 14): a one-image stripe plans
    one chunk lane whose chunk can exceed the whole call's two-lane chunks, so
    imf_filter_host sizes each lane's workspace by the largest stripe plan."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec
    from paper_2505_22938_b200.tiling import run_host
    img, spec, boundary = _big_case(14)
    assert img.shape == (430, 306, 3) and spec[:2] == ("square", 124)
    params = FilterParams(shape=ShapeSpec(*spec), boundary=boundary)
    want = oracle.fast_filter(img, params.shape, 0.5, boundary)
    assert run_host(img, params).tobytes() == want.tobytes()
