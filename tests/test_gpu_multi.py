"""Multi-device dispatch, host row ranges, stream safety and the device
scan-defect path (all bit-exact against the oracle / golden digests).

* filter_multi: one process driving several GPU pipelines:
  whole images per device for batches, output-row stripes for single images;
  on a one-GPU box the device list repeats cuda:0 (two pipelines, one GPU);
* run_host(rows=...): imf_filter_host with an output-row range;
* run_device on a side stream (workspace per (device, stream));
* IMF_DEBUG_DEFECT: an inconsistent slide count injected on the device must
  surface as ScanDefectError from every entry point -- the device analog of
  the reference's test_refine_defect_on_inconsistent_count
  (/root/reference/pkg/tests/test_core.py:124-130).
"""
import numpy as np
import pytest

import cases as C
import oracle

pytestmark = pytest.mark.gpu


def _api():
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    return FilterParams, ShapeSpec, filter_image


@pytest.mark.parametrize("ndev", [1, 2, 3])
def test_filter_multi_single_image_stripes(ndev):
    from paper_2505_22938_b200 import filter_multi
    FilterParams, ShapeSpec, _ = _api()
    img = np.random.default_rng(31).integers(0, 65536, (523, 419, 3), dtype=np.uint16)
    params = FilterParams(shape=ShapeSpec("circle", 13))
    got = filter_multi(img, params, devices=[0] * ndev)
    assert np.array_equal(got, oracle.fast_filter(img, params.shape, 0.5))


@pytest.mark.parametrize("boundary", ["replicate", "valid"])
def test_filter_multi_stripes_percentile_map(boundary):
    from paper_2505_22938_b200 import filter_multi
    FilterParams, ShapeSpec, _ = _api()
    rng = np.random.default_rng(32)
    img = rng.integers(0, 256, (300, 211), dtype=np.uint8)
    r = 9
    oh, ow = (300 - 2 * r, 211 - 2 * r) if boundary == "valid" else (300, 211)
    pmap = rng.random((oh, ow))
    params = FilterParams(shape=ShapeSpec("circle", r), percentile=pmap, boundary=boundary)
    got = filter_multi(img, params, devices=[0, 0])
    assert np.array_equal(got, oracle.fast_filter(img, params.shape, pmap, boundary))


def test_filter_multi_batch_whole_images():
    from paper_2505_22938_b200 import filter_multi
    FilterParams, ShapeSpec, _ = _api()
    imgs = np.random.default_rng(33).integers(0, 256, (5, 190, 230), dtype=np.uint8)
    params = FilterParams(shape=ShapeSpec("regular_polygon", 6, sides=6))
    got = filter_multi(imgs, params, devices=[0, 0], batched=True)
    for b in range(5):
        assert np.array_equal(got[b], oracle.fast_filter(imgs[b], params.shape, 0.5)), b


def test_filter_multi_c5_images(golden):
    """Two c5 8K images (r=64) through the multi-device batch path == reference digests."""
    import json
    import os
    from paper_2505_22938_b200 import filter_multi
    FilterParams, ShapeSpec, _ = _api()
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_c5.json")) as f:
        g5 = json.load(f)
    imgs = np.stack([C.baseline_input("c5", i) for i in (5, 6)])
    got = filter_multi(imgs, FilterParams(shape=ShapeSpec("circle", 64)), devices=[0, 0], batched=True)
    assert C.digest(got[0]) == g5["5"] and C.digest(got[1]) == g5["6"]


def test_run_host_row_range_leaves_other_rows():
    from paper_2505_22938_b200.tiling import run_host
    FilterParams, ShapeSpec, _ = _api()
    img = np.random.default_rng(34).integers(0, 65536, (400, 150), dtype=np.uint16)
    params = FilterParams(shape=ShapeSpec("circle", 10))
    out = np.full_like(img, 7)
    run_host(img, params, out=out, rows=(130, 277))
    want = oracle.fast_filter(img, params.shape, 0.5)
    assert np.array_equal(out[130:277], want[130:277])
    assert (out[:130] == 7).all() and (out[277:] == 7).all()


def test_run_host_checks_and_stages_out():
    from paper_2505_22938_b200.tiling import run_host
    FilterParams, ShapeSpec, _ = _api()
    img = np.random.default_rng(35).integers(0, 256, (120, 90, 3), dtype=np.uint8)
    params = FilterParams(shape=ShapeSpec("circle", 5))
    with pytest.raises(ValueError):
        run_host(img, params, out=np.empty((120, 90, 3), np.uint16))
    with pytest.raises(ValueError):
        run_host(img, params, out=np.empty((120, 91, 3), np.uint8))
    rgba = np.full((120, 90, 4), 99, np.uint8)
    run_host(img, params, out=rgba[..., :3])  # non-dense view: staged, alpha untouched
    assert np.array_equal(rgba[..., :3], oracle.fast_filter(img, params.shape, 0.5))
    assert (rgba[..., 3] == 99).all()


def test_run_device_side_stream():
    import torch
    from paper_2505_22938_b200.tiling import run_device
    FilterParams, ShapeSpec, _ = _api()
    img = np.random.default_rng(36).integers(0, 65536, (257, 311), dtype=np.uint16)
    params = FilterParams(shape=ShapeSpec("circle", 12))
    src = torch.from_numpy(img).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a = run_device(src, params, stream=s1)
    b = run_device(src.flip(0).contiguous(), params, stream=s2)
    torch.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), oracle.fast_filter(img, params.shape, 0.5))
    assert np.array_equal(b.cpu().numpy(), oracle.fast_filter(img[::-1].copy(), params.shape, 0.5))


@pytest.mark.parametrize("cfg", [("circle", 9, 0, "u16"), ("square", 6, 0, "u8"),
                                 ("circle", 70, 0, "f32"), ("regular_polygon", 20, 7, "u8")])
def test_device_scan_defect_raises(monkeypatch, cfg):
    """IMF_DEBUG_DEFECT=1 corrupts one slide count in the first tile: the walk
    leaves the rank array, the kernel sets the status word, and the caller
    sees ScanDefectError (core.py:31-36) -- device, host and bracket entries."""
    import torch
    from paper_2505_22938_b200 import ScanDefectError, filter_image_bracket
    from paper_2505_22938_b200.tiling import run_host
    FilterParams, ShapeSpec, filter_image = _api()
    kind, r, sides, dt = cfg
    rng = np.random.default_rng(37)
    img = C.as_dtype(rng.integers(0, 256, (230, 200)), {"u8": np.uint8, "u16": np.uint16}[dt]) if dt != "f32" else \
        rng.standard_normal((300, 300)).astype(np.float32)
    params = FilterParams(shape=ShapeSpec(kind, r, sides=sides))
    monkeypatch.setenv("IMF_DEBUG_DEFECT", "1")
    with pytest.raises(ScanDefectError):
        filter_image(torch.from_numpy(img).cuda(), params)
    with pytest.raises(ScanDefectError):
        run_host(img, params)
    with pytest.raises(ScanDefectError):
        filter_image_bracket(img, params, [0.25, 0.5])
    monkeypatch.delenv("IMF_DEBUG_DEFECT")
    assert np.array_equal(filter_image(img, params), oracle.fast_filter(img, params.shape, 0.5))


@pytest.mark.parametrize("dt,r,boundary", [(np.uint16, 20, "replicate"), (np.uint8, 9, "valid"),
                                           (np.uint16, 64, "replicate")])
def test_k1_tma_tile_loads(dt, r, boundary):
    """Planar (pixel-contiguous) u8/u16 images: K1 loads its tile boxes with TMA
    (cp.async.bulk.tensor, clamped box reads = replicate padding); a row-shifted
    view that breaks the 16-byte alignment falls back to per-lane loads.  Both
    bit-exact against the oracle."""
    import torch
    from paper_2505_22938_b200 import _lib
    FilterParams, ShapeSpec, filter_image = _api()
    rng = np.random.default_rng(38)
    hi = 256 if dt == np.uint8 else 65536
    img = rng.integers(0, hi, (3, 457, 389), dtype=dt)  # batch of planes
    params = FilterParams(shape=ShapeSpec("circle", r), boundary=boundary)
    from paper_2505_22938_b200 import filter_batch
    src = torch.from_numpy(img).cuda()
    pad = torch.zeros((3, 457, 400), dtype=src.dtype, device="cuda")
    pad[:, :, :389] = src  # row stride 400 elements: a 16-byte multiple for u8 and u16
    L = _lib.lib()
    seen_tma = False
    for t in (src, pad[:, :, :389], src[:, :, :384].contiguous()):
        out = filter_batch(t, params).cpu().numpy()
        tma = bool(L.imf_last_features() & _lib.IMF_FEATURE_K1_TMA)
        row_bytes = t.stride(1) * t.element_size()
        assert tma == (row_bytes % 16 == 0 and t.data_ptr() % 16 == 0), (tma, row_bytes)
        seen_tma = seen_tma or tma
        host = t.cpu().numpy()
        for b in range(3):
            assert np.array_equal(out[b], oracle.fast_filter(host[b], params.shape, 0.5, boundary)), b
    assert seen_tma  # the aligned layouts did take the TMA path


@pytest.mark.parametrize("boundary", ["replicate", "valid"])
def test_filter_batch_multi_device_resident(boundary):
    """A device-resident batch scattered to peers (here: cuda:0 listed twice)
    and gathered back equals the single-device batch result."""
    import torch
    from paper_2505_22938_b200 import filter_batch, filter_batch_multi
    FilterParams, ShapeSpec, _ = _api()
    imgs = torch.from_numpy(np.random.default_rng(39).integers(0, 65536, (5, 170, 190, 3),
                                                               dtype=np.uint16)).cuda()
    params = FilterParams(shape=ShapeSpec("circle", 11), boundary=boundary)
    got = filter_batch_multi(imgs, params, devices=[0, 0])
    want = filter_batch(imgs, params)
    assert torch.equal(got, want)


def test_workspace_cache_is_bounded_under_stream_churn():
    """A new stream per call must not pin a workspace per stream."""
    import torch

    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    from paper_2505_22938_b200.tiling import _WS
    img = torch.from_numpy(np.random.default_rng(4).integers(0, 256, (200, 180), dtype=np.uint8)).cuda()
    params = FilterParams(shape=ShapeSpec("circle", 9))
    want = oracle.fast_filter(img.cpu().numpy(), params.shape, 0.5)
    for _ in range(20):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            out = filter_image(img, params)
        s.synchronize()
        assert out.cpu().numpy().tobytes() == want.tobytes()
    assert len(_WS.buf) <= _WS.MAX_ENTRIES
