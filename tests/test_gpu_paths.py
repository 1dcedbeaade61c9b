"""Every alternate engine path stays bit-exact (the planner picks one per
geometry; environment switches force the others on the same inputs).

Paths: pair fast path vs the generic selection kernel (IMF_PAIR), omega in
shared memory vs in L2 (IMF_PAIR_OMG), rounded-rect footprint on/off
(IMF_FOOTPRINT), f32 bucket transform vs LSD radix sort (IMF_F32_BUCKET),
register-resident vs two-pass u16 counting sort (IMF_K1REG), the pair path on
generic-span kernels (IMF_PAIR_ANY), polygons on the general path
(IMF_PAIR_POLY=0), one chunk stream (IMF_LANES), per-group phases (IMF_GROUPED),
direct selection for tiny windows (IMF_DIRECT), TMA vs per-lane K1 tile loads
(IMF_TMA), both phase-D refine loops (IMF_REFINE), rectangular pair tiles
(IMF_PAIR_RECT),
and tile / seed-row overrides.  Compared against the C oracle, which is itself
pinned to the reference's golden outputs (tests/test_oracle.py)."""
import os

import numpy as np
import pytest

import cases as C
import oracle

pytestmark = pytest.mark.gpu

VARIANTS = [
    {},
    {"IMF_PAIR": "0"},
    {"IMF_PAIR_OMG": "1"},
    {"IMF_FOOTPRINT": "0"},
    {"IMF_F32_BUCKET": "0"},
    {"IMF_K1REG": "0"},
    {"IMF_PAIR_ANY": "1"},
    {"IMF_PAIR_POLY": "0"},
    {"IMF_LANES": "1"},
    {"IMF_GROUPED": "0"},
    {"IMF_DIRECT": "0"},
    {"IMF_TMA": "0"},
    {"IMF_K1_BULK": "0"},
    {"IMF_COSTLY_FIRST": "0"},
    {"IMF_REFINE": "0"},
    {"IMF_PAIR_RECT": "1", "IMF_TILE": "64"},
    {"IMF_TILE": "40", "IMF_SEED_ROWS": "4"},
    {"IMF_STRIPE_EDGE": "1", "IMF_STRIPE_MID": "5"},
    {"IMF_RUNMIN": "2"},    # every replicate-copy group ranked as a run (bucket K1)
    {"IMF_RUNMIN": "64"},   # edge groups as runs at large r
    {"IMF_PAIR_WIDE": "0"},  # r > 64 circles on the general select path
    {"IMF_GCOARSE": "2"},    # call-wide coarse bucket table for every adaptive f32 tile
    {"IMF_GCOARSE": "0"},    # per-tile coarse passes only
    {"IMF_K1_COUNT_G": "0"},  # u16 tiles beyond the shared counting sort via the bucket transform
    {"IMF_MAXSUMSQ_K": "0"},  # every run-free f32 tile to the LSD fallback (footprint index map at r=100)
    {"IMF_F32_FOOTPRINT": "2"},  # f32 footprint on the shared-entry bucket kernels too
    {"IMF_F32_FOOTPRINT": "2", "IMF_MAXSUMSQ_K": "0"},
    {"IMF_F32_FOOTPRINT": "2", "IMF_RUNMIN": "2"},  # runs clipped by the footprint
]

CASES = [  # (dtype, shape, kernel spec)
    ("uint16", (211, 301, 3), ("circle", 48, 0, 0.0)),
    ("uint16", (150, 170), ("circle", 62, 0, 0.0)),       # halved ranks (N > 32768)
    ("uint16", (260, 250), ("circle", 100, 0, 0.0)),      # u16 bucket transform (S = 255)
    ("float32", (180, 200), ("circle", 20, 0, 0.0)),
    ("float32", (260, 240), ("circle", 60, 0, 0.0)),      # f32 global-entries bucket
    ("float32", (230, 250), ("circle", 40, 0, 0.0)),      # f32 adaptive buckets, own-pixel ranking
    ("float32", (300, 280), ("circle", 100, 0, 0.0)),     # f32 r=100: corner runs (bucket_g), wide pair K2
    ("uint8", (230, 210, 2), ("circle", 75, 0, 0.0)),     # wide pair K2 (T + r > 128), u8
    ("uint8", (190, 170, 2), ("regular_polygon", 11, 6, 15.0)),
    ("float32", (200, 190), ("regular_polygon", 30, 7, 12.0)),  # f32 polygon footprint
    ("float32", (60, 242), ("regular_polygon", 34, 3, 29.3)),   # empty footprint rows (triangle)
    ("uint8", (120, 130), ("square", 7, 0, 0.0)),
    ("float32", (70, 90), ("circle", 2, 0, 0.0)),         # direct selection (area <= 32)
    ("uint16", (65, 77, 3), ("square", 2, 0, 0.0)),
    ("uint8", (40, 33), ("regular_polygon", 3, 5, 10.0)),
]


def _input(dt, shape, seed):
    rng = np.random.default_rng(seed)
    if dt == "float32":
        img = rng.standard_normal(shape).astype(np.float32)
        img[:, :5] = 0.25  # a flat band: ties and a large bucket
        return img
    hi = np.iinfo(dt).max + 1
    img = rng.integers(0, hi, shape).astype(dt)
    img[:9] = img[0, 0]     # flat rows: ties across the tile
    return img


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: ",".join(f"{k}={x}" for k, x in v.items()) or "default")
def test_variant_bit_exact(variant, monkeypatch):
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    for i, (dt, shape, spec) in enumerate(CASES):
        img = _input(dt, shape, i)
        for boundary in ("replicate", "valid"):
            if boundary == "valid" and min(shape[:2]) <= 2 * spec[1]:
                continue
            for p in (0.5, 0.13):
                params = FilterParams(shape=ShapeSpec(*spec), percentile=p, boundary=boundary)
                got = filter_image(img, params)
                want = oracle.fast_filter(img, params.shape, p, boundary)
                assert got.tobytes() == want.tobytes(), (variant, dt, shape, spec, boundary, p)


@pytest.mark.parametrize("dt", ["uint8", "uint16", "float32"])
def test_direct_selection_maps_bracket_tiny_images(dt):
    """Direct-selection kernel (window area <= 32): per-pixel percentile maps,
    valid boundary, the bracket, and images smaller than one 32-pixel tile."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image, filter_image_bracket
    rng = np.random.default_rng(99)
    for shape in ((1, 1), (3, 5), (31, 33, 2), (77, 45)):
        img = _input(dt, shape, 5)
        for spec in (ShapeSpec("circle", 2), ShapeSpec("square", 1), ShapeSpec("circle", 0)):
            pmap = rng.random(shape[:2])
            got = filter_image(img, FilterParams(shape=spec, percentile=pmap))
            want = oracle.fast_filter(img, spec, pmap, "replicate")
            assert got.tobytes() == want.tobytes(), (dt, shape, spec)
            if min(shape[:2]) > 2 * spec.radius:
                got = filter_image(img, FilterParams(shape=spec, boundary="valid", percentile=0.7))
                want = oracle.fast_filter(img, spec, 0.7, "valid")
                assert got.tobytes() == want.tobytes(), (dt, shape, spec, "valid")
        outs = filter_image_bracket(img, FilterParams(shape=ShapeSpec("circle", 2)), [0.0, 0.5, 1.0])
        for out, p in zip(outs, (0.0, 0.5, 1.0)):
            assert out.tobytes() == oracle.fast_filter(img, ShapeSpec("circle", 2), p).tobytes()


@pytest.mark.parametrize("fp", ["1", "2"])
def test_f32_sentinel_key_collision(fp, monkeypatch):
    """Interior tiles of the bucket K1 mark unranked slots with the entry
    0xffffffff.  A ranked pixel can map to that entry too: values in ONE
    coarse bin (key >> 20) get all 65,536 fine buckets, and +FLT_MAX lands in
    the last one with low key bits 0xffff.  Such tiles must take the LSD
    fallback and stay bit-exact."""
    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image
    monkeypatch.setenv("IMF_F32_FOOTPRINT", fp)
    rng = np.random.default_rng(7)
    fmax = np.finfo(np.float32).max
    # [1.875 * 2^127, FLT_MAX]: one coarse bin (key 0xff7xxxxx)
    img = rng.uniform(1.875 * 2.0 ** 127, float(fmax), (300, 290)).astype(np.float32)
    img[rng.integers(40, 260, 60), rng.integers(40, 250, 60)] = fmax
    assert len(np.unique(img.view(np.uint32) >> 20)) == 1
    for r in (40, 60):
        params = FilterParams(shape=ShapeSpec("circle", r), percentile=0.5)
        got = filter_image(img, params)
        want = oracle.fast_filter(img, params.shape, 0.5, "replicate")
        assert got.tobytes() == want.tobytes(), r


@pytest.mark.parametrize("fp", ["1", "2"])
def test_f32_batch_footprint_runs(fp, monkeypatch):
    """A batch of f32 images (tile index crosses images) through the bucket K1
    with the footprint and clipped corner runs: every image equals the oracle."""
    import torch

    from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_batch
    monkeypatch.setenv("IMF_F32_FOOTPRINT", fp)
    monkeypatch.setenv("IMF_RUNMIN", "64")  # edge copy groups as runs too
    rng = np.random.default_rng(11)
    imgs = rng.standard_normal((3, 170, 190)).astype(np.float32)
    imgs[1, :40, :50] = 1.5  # a flat corner: a long tie run and a large bucket
    for r in (20, 36, 70):
        params = FilterParams(shape=ShapeSpec("circle", r), percentile=0.4)
        out = filter_batch(torch.from_numpy(imgs).cuda(), params).cpu().numpy()
        for b in range(3):
            want = oracle.fast_filter(imgs[b], params.shape, 0.4, "replicate")
            assert out[b].tobytes() == want.tobytes(), (r, b)
