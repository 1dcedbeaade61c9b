"""GPU parity at full size and through every entry point (bit-exact).

* acceptance criterion 1 matrix (3 dtypes x 13 images x 9 radii x 5 p) vs
  digests of the real reference (test_acceptance.py:62-85);
* BASELINE configs c1..c5 at full size vs reference digests (c3: every radius
  2..100; c5: all 64 8K images through the batch API);
* invariants the reference tests: tile-size invariance, monotone-map
  commutation, r=0 identity, p=0/p=1 erosion/dilation, determinism;
* torch / non-contiguous / planar layouts, and the C ABI host entry point.
"""
import ctypes
import json
import os

import numpy as np
import pytest

import cases as C
import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fi():
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    return FilterParams, ShapeSpec, filter_image


def test_acceptance_matrix(golden):
    FilterParams, ShapeSpec, filter_image = _fi()
    acc = golden["acceptance"]
    bad = []
    for dt in C.ACC_DTYPES:
        for idx, base in enumerate(C.acceptance_images()):
            img = C.as_dtype(base, dt)
            for r in C.ACC_RADII:
                for p in C.ACC_PERCENTILES:
                    out = filter_image(img, FilterParams(shape=ShapeSpec("circle", r), percentile=p))
                    if C.digest(out) != acc[f"{dt}/{idx}/{r}/{p}"]:
                        bad.append((dt, idx, r, p))
    assert not bad, bad[:10]


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_baseline_c1_c2(cfg, golden):
    FilterParams, ShapeSpec, filter_image = _fi()
    r = 8 if cfg == "c1" else 48
    out = filter_image(C.baseline_input(cfg), FilterParams(shape=ShapeSpec("circle", r)))
    assert C.digest(out) == golden["baseline"][cfg]


def test_baseline_c3_radius_sweep(golden):
    import torch
    FilterParams, ShapeSpec, filter_image = _fi()
    img = torch.from_numpy(C.baseline_input("c3")).cuda()
    bad = []
    for r in C.C3_RADII:
        out = filter_image(img, FilterParams(shape=ShapeSpec("circle", r))).cpu().numpy()
        if C.digest(out) != golden["baseline"][f"c3/r{r}"]:
            bad.append(r)
    assert not bad, bad


def test_baseline_c4_shapes(golden):
    FilterParams, ShapeSpec, filter_image = _fi()
    img = C.baseline_input("c4")
    for spec in C.C4_SHAPES:
        out = filter_image(img, FilterParams(shape=ShapeSpec(*spec)))
        assert C.digest(out) == golden["baseline"]["c4/" + json.dumps(list(spec))], spec


def test_baseline_c5_batch():
    import torch
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_batch
    with open(os.path.join(ROOT, "tests", "golden", "golden_c5.json")) as f:
        g5 = json.load(f)
    params = FilterParams(shape=ShapeSpec("circle", 64))
    bad = []
    ids = sorted(int(k) for k in g5)
    for b0 in range(0, len(ids), 8):
        chunk = ids[b0:b0 + 8]
        batch = torch.from_numpy(np.stack([C.baseline_input("c5", i) for i in chunk])).cuda()
        out = filter_batch(batch, params).cpu().numpy()
        bad += [i for k, i in enumerate(chunk) if C.digest(out[k]) != g5[str(i)]]
    assert not bad, bad
    assert len(ids) == 64


@pytest.mark.parametrize("dt", ["uint8", "uint16", "float32"])
def test_tile_size_invariance(dt):
    FilterParams, ShapeSpec, filter_image = _fi()
    img = C.small_input("uniform", (150, 170, 2), dt, 99)
    ref = oracle.fast_filter(img, ShapeSpec("circle", 10), 0.5)
    for ts in (8, 16, 24, 37, 64, 120):
        out = filter_image(img, FilterParams(shape=ShapeSpec("circle", 10), tile_size=ts,
                                             forwarding=False))
        assert out.tobytes() == ref.tobytes(), ts


def test_monotone_map_commutation():
    # acceptance criterion 4 (test_acceptance.py:120-135)
    FilterParams, ShapeSpec, filter_image = _fi()
    rng = np.random.default_rng(0xC0FFEE)
    img = rng.integers(0, 101, (128, 160)).astype(np.uint8)
    params = FilterParams(shape=ShapeSpec("circle", 7), percentile=0.3)
    filtered = filter_image(img, params)
    for _ in range(20):
        lut = np.sort(rng.choice(256, size=101, replace=False)).astype(np.uint8)
        assert np.array_equal(filter_image(lut[img], params), lut[filtered])


def test_identity_erosion_dilation_determinism():
    FilterParams, ShapeSpec, filter_image = _fi()
    rng = np.random.default_rng(4)
    img = rng.integers(0, 65536, (90, 110)).astype(np.uint16)
    assert np.array_equal(filter_image(img, FilterParams(shape=ShapeSpec("circle", 0))), img)
    for p in (0.0, 1.0):
        got = filter_image(img, FilterParams(shape=ShapeSpec("circle", 5), percentile=p))
        want = oracle.brute_filter(img, ShapeSpec("circle", 5), p)
        assert np.array_equal(got, want)
    outs = {filter_image(img, FilterParams(shape=ShapeSpec("circle", 9))).tobytes()
            for _ in range(3)}
    assert len(outs) == 1


def test_torch_layouts_and_noncontiguous():
    import torch
    FilterParams, ShapeSpec, filter_image = _fi()
    rng = np.random.default_rng(8)
    img = rng.integers(0, 65536, (3, 77, 91)).astype(np.uint16)   # planar CHW
    params = FilterParams(shape=ShapeSpec("circle", 6))
    hwc_view = torch.from_numpy(img).cuda().permute(1, 2, 0)       # non-contiguous HWC view
    want = oracle.fast_filter(np.ascontiguousarray(img.transpose(1, 2, 0)), params.shape)
    got = filter_image(hwc_view, params)
    assert got.is_cuda and tuple(got.shape) == want.shape
    assert np.array_equal(got.cpu().numpy(), want)
    t = torch.from_numpy(want.copy())                              # CPU tensor in -> CPU tensor out
    assert not filter_image(t, params).is_cuda
    tr = np.ascontiguousarray(want[..., 0]).T                      # transposed numpy view
    assert np.array_equal(filter_image(tr, params), oracle.fast_filter(np.ascontiguousarray(tr),
                                                                       params.shape))


def test_large_radius_global_omega_path():
    FilterParams, ShapeSpec, filter_image = _fi()
    for dt, r in (("uint8", 120), ("float32", 118), ("uint16", 110)):
        img = C.small_input("uniform", (260, 270), dt, r)
        got = filter_image(img, FilterParams(shape=ShapeSpec("circle", r)))
        want = oracle.fast_filter(img, ShapeSpec("circle", r), 0.5)
        assert got.tobytes() == want.tobytes(), (dt, r)


def test_c_abi_host_entry_point():
    from paper_2505_22938_b200 import ShapeSpec, _lib, make_kernel, target_rank
    from paper_2505_22938_b200.tiling import _kernel_struct
    rng = np.random.default_rng(12)
    src = rng.integers(0, 256, (2, 70, 80, 3), dtype=np.uint8)   # batch of 2 HWC images
    dst = np.zeros_like(src)
    k = make_kernel(ShapeSpec("regular_polygon", 7, sides=8))
    ks, keep = _kernel_struct(k)
    def im(a):
        st = [s // a.itemsize for s in a.strides]
        return _lib.ImfImage(a.ctypes.data, 0, 2, 70, 80, 3, st[0], st[1], st[2], st[3])
    s_im, d_im = im(src), im(dst)
    opt = _lib.ImfOptions(0, 0, 0, 0)
    t = target_rank(k.area, 0.5)
    L = _lib.lib()
    rc = L.imf_filter_host(ctypes.byref(s_im), ctypes.byref(d_im), ctypes.byref(ks), t, None, t, t,
                           ctypes.byref(opt), None)
    assert rc == 0, _lib.strerror(rc)
    for b in range(2):
        assert np.array_equal(dst[b], oracle.fast_filter(src[b], k.spec, 0.5))


def test_scan_defect_is_reported_not_silent():
    # an invalid target (>= area) must be rejected before launch (never a silent wrong answer)
    from paper_2505_22938_b200 import ShapeSpec, _lib, make_kernel
    from paper_2505_22938_b200.tiling import _kernel_struct
    k = make_kernel(ShapeSpec("circle", 3))
    ks, keep = _kernel_struct(k)
    a = np.zeros((1, 20, 20, 1), np.uint8)
    im = _lib.ImfImage(a.ctypes.data, 0, 1, 20, 20, 1, 400, 20, 1, 1)
    out = np.zeros_like(a)
    om = _lib.ImfImage(out.ctypes.data, 0, 1, 20, 20, 1, 400, 20, 1, 1)
    rc = _lib.lib().imf_filter_host(ctypes.byref(im), ctypes.byref(om), ctypes.byref(ks), k.area,
                                    None, k.area, k.area, ctypes.byref(_lib.ImfOptions(0, 0, 0, 0)),
                                    None)
    assert rc == _lib.IMF_ERR_INVALID


@pytest.mark.parametrize("boundary", ["replicate", "valid"])
def test_host_pipeline_stripes(boundary):
    """imf_filter_host pipelines row stripes (upload / filter / download on three
    streams); batch of HWC images, a per-pixel percentile map, both boundaries."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec
    from paper_2505_22938_b200.tiling import run_host
    rng = np.random.default_rng(21)
    src = rng.integers(0, 65536, (2, 421, 333, 3), dtype=np.uint16)
    r = 11
    oh, ow = (421 - 2 * r, 333 - 2 * r) if boundary == "valid" else (421, 333)
    pmap = rng.random((oh, ow))
    params = FilterParams(shape=ShapeSpec("circle", r), percentile=pmap, boundary=boundary)
    got = run_host(src, params, batched=True)
    for b in range(2):
        want = oracle.fast_filter(src[b], params.shape, pmap, boundary)
        assert np.array_equal(got[b], want), b


def test_host_pipeline_ring_batch():
    """Batches longer than two images stream through a ring of two device image
    slots (image b reuses slot b % 2 after image b - 2 is downloaded)."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec
    from paper_2505_22938_b200.tiling import run_host
    rng = np.random.default_rng(23)
    src = rng.integers(0, 256, (5, 290, 270), dtype=np.uint8)
    params = FilterParams(shape=ShapeSpec("circle", 9), percentile=0.3)
    got = run_host(src, params, batched=True)
    for b in range(5):
        want = oracle.fast_filter(src[b], params.shape, 0.3, "replicate")
        assert np.array_equal(got[b], want), b


def test_device_row_range_stripes_assemble():
    """imf_options.row_begin/row_end: disjoint output stripes written by separate
    calls assemble to the whole-image result."""
    import torch
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib, make_kernel, target_rank
    from paper_2505_22938_b200.tiling import _image_struct, _kernel_struct, workspace_for
    rng = np.random.default_rng(22)
    img = rng.integers(0, 256, (300, 257), dtype=np.uint8)
    k = make_kernel(ShapeSpec("circle", 9))
    ks, keep = _kernel_struct(k)
    src = torch.from_numpy(img).cuda()
    out = torch.zeros_like(src)
    s_im, d_im = _image_struct(src, 0, False, False), _image_struct(out, 0, False, False)
    L = _lib.lib()
    t = target_rank(k.area, 0.5)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for y0, y1 in ((0, 37), (37, 200), (200, 300)):
        opt = _lib.ImfOptions(0, 0, 0, 0)
        opt.row_begin, opt.row_end = y0, y1
        need = L.imf_workspace_size(ctypes.byref(s_im), ctypes.byref(ks), ctypes.byref(opt))
        ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        rc = L.imf_filter(ctypes.byref(s_im), ctypes.byref(d_im), ctypes.byref(ks), t, None, t, t,
                          ctypes.byref(opt), ws.data_ptr(), need, stream)
        assert rc == 0, _lib.strerror(rc)
        assert L.imf_workspace_status(ws.data_ptr(), stream) == 0
    assert np.array_equal(out.cpu().numpy(), oracle.fast_filter(img, k.spec, 0.5))
