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

SEED0 = int(os.environ.get("IMF_FUZZ_SEED0", "0"))  # shifts every sweep's seeds
ENVS = [{}, {}, {"IMF_F32_FOOTPRINT": "2"}, {"IMF_RUNMIN": "8"}, {"IMF_F32_FOOTPRINT": "0"},
        {"IMF_TILE": "40"}, {"IMF_PAIR": "0"}, {"IMF_MAXSUMSQ_K": "4"}]


def _case(seed):
    rng = np.random.default_rng(1000 + SEED0 + seed)
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


def _big_case(seed, base=None):
    rng = np.random.default_rng((5000 + SEED0 if base is None else base) + seed)
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
    img, spec, boundary = _big_case(14, base=5000)
    assert img.shape == (430, 306, 3) and spec[:2] == ("square", 124)
    params = FilterParams(shape=ShapeSpec(*spec), boundary=boundary)
    want = oracle.fast_filter(img, params.shape, 0.5, boundary)
    assert run_host(img, params).tobytes() == want.tobytes()


def _layout_case(seed):
    rng = np.random.default_rng(9000 + SEED0 + seed)
    dt = rng.choice(["uint8", "uint16", "float32"])
    r = int(rng.choice([0, 1, 3, 6, 12, 25, 40, 64, 100]))
    b = int(rng.integers(1, 4))
    h, w = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    c = int(rng.choice([1, 2, 3, 4]))
    if dt == "float32":
        img = rng.standard_normal((b, h, w, c)).astype(np.float32)
        special = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 3.4e38, -3.4e38], np.float32)
        m = rng.random((b, h, w, c)) < 0.05
        img[m] = rng.choice(special, int(m.sum()))
    else:
        top = 256 if dt == "uint8" else 65536
        img = rng.integers(0, int(rng.choice([2, 17, top])), (b, h, w, c)).astype(dt)
    kind = rng.choice(["circle", "square", "regular_polygon"])
    spec = (kind, r, int(rng.integers(3, 9)), float(rng.uniform(0, 90))) if kind == "regular_polygon" \
        else (kind, r, 0, 0.0)
    return img, spec, float(rng.choice([0.0, 0.25, 0.5, 0.999, 1.0])), rng


@pytest.mark.parametrize("seed", range(int(os.environ.get("IMF_FUZZ_LAYOUT", "24"))))
def test_random_device_layouts_and_batches(seed):
    """CUDA tensors in random layouts -- channel subsets, transposed (W, H)
    views, batches -- special f32 values (+-0, +-inf, denormals, +-FLT_MAX),
    few-valued integer images, r = 0 .. 100: filter_image on a view and
    filter_batch on the batch equal the oracle image by image."""
    import torch

    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_batch, filter_image
    img, spec, pct, rng = _layout_case(seed)
    params = FilterParams(shape=ShapeSpec(*spec), percentile=pct)
    t = torch.from_numpy(img).cuda()
    want = [oracle.fast_filter(img[i], params.shape, pct) for i in range(img.shape[0])]
    got = filter_batch(t, params).cpu().numpy()
    for i in range(img.shape[0]):
        assert got[i].tobytes() == want[i].tobytes(), ("batch", seed, img.dtype, img.shape, spec, pct, i)
    # one image through a strided view: a channel subset, optionally transposed
    c0 = int(rng.integers(0, img.shape[3]))
    view = t[0, :, :, c0:]
    if rng.random() < 0.5:
        view = view.transpose(0, 1)
        ref = oracle.fast_filter(np.ascontiguousarray(img[0, :, :, c0:].transpose(1, 0, 2)), params.shape, pct)
    else:
        ref = want[0][..., c0:]
    g = filter_image(view, params)
    g = g.cpu().numpy() if hasattr(g, "cpu") else g
    assert np.ascontiguousarray(g).tobytes() == np.ascontiguousarray(ref).tobytes(), ("view", seed, spec, pct)


@pytest.mark.parametrize("seed", range(int(os.environ.get("IMF_FUZZ_MAPS", "12"))))
def test_random_maps_row_ranges_and_multi(seed):
    """Per-pixel percentile maps in both boundary modes through the streamed
    host entry with a random output-row range, and filter_multi over repeated
    device entries (row stripes of one image), against the oracle."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_multi
    from paper_2505_22938_b200.tiling import run_host
    rng = np.random.default_rng(7000 + SEED0 + seed)
    dt = rng.choice(["uint8", "uint16", "float32"])
    r = int(rng.choice([3, 10, 30, 48, 70]))
    h, w = int(rng.integers(2 * r + 2, 2 * r + 400)), int(rng.integers(2 * r + 2, 2 * r + 300))
    shape = (h, w) if rng.random() < 0.5 else (h, w, 3)
    img = (rng.standard_normal(shape).astype(np.float32) if dt == "float32"
           else rng.integers(0, 256 if dt == "uint8" else 65536, shape).astype(dt))
    boundary = rng.choice(["replicate", "valid"])
    oh, ow = (h - 2 * r, w - 2 * r) if boundary == "valid" else (h, w)
    pmap = rng.random((oh, ow))
    spec = ShapeSpec(rng.choice(["circle", "square"]), r)
    params = FilterParams(shape=spec, percentile=pmap, boundary=boundary)
    want = oracle.fast_filter(img, spec, pmap, boundary)
    y0 = int(rng.integers(0, oh))
    y1 = int(rng.integers(y0 + 1, oh + 1))
    out = np.zeros_like(want)
    run_host(img, params, out=out, rows=(y0, y1))
    assert out[y0:y1].tobytes() == want[y0:y1].tobytes(), ("rows", seed, dt, shape, r, boundary, y0, y1)
    assert not out[:y0].any() and not out[y1:].any()
    got = filter_multi(img, params, devices=[0, 0, 0])
    assert got.tobytes() == want.tobytes(), ("multi", seed, dt, shape, r, boundary)
