"""The CPU oracle (oracle/, a C restatement of the reference) is pinned to the
real reference's outputs before it is trusted as a checker (CPU only)."""
import json

import numpy as np
import pytest

import cases as C
import oracle
from paper_2505_22938_b200 import ShapeSpec


def _run(which, name, recipe, p):
    img = C.make_input(recipe)
    out_shape = C.out_shape_of(img.shape, p["shape"][1], p["boundary"])
    perc = C.resolve_percentile(p["percentile"], out_shape)
    fn = oracle.fast_filter if which == "fast" else oracle.brute_filter
    return fn(img, ShapeSpec(*p["shape"]), perc, p["boundary"], threads=4)


def test_oracle_kernel_geometry_matches_reference_digests(golden):
    """The oracle rasterizes kernels itself (oracle/kernel_geom.py, not the
    product's make_kernel): every span table equals the real reference's."""
    from oracle.kernel_geom import kernel_of, target_rank
    bad = [spec for key, dig in golden["kernels"].items()
           for spec in [tuple(json.loads(key))]
           if C.kernel_digest(kernel_of(ShapeSpec(*spec))) != dig]
    assert not bad, bad[:5]
    assert len(golden["kernels"]) >= 300
    for area, p, want in [(21, 0.5, 10), (21, 0.0, 0), (21, 1.0, 20), (9, 0.3, 2), (1, 0.7, 0)]:
        assert target_rank(area, p) == want


@pytest.mark.parametrize("which", ["fast", "brute"])
def test_oracle_matches_reference_small(which, golden_small):
    bad = []
    for name, recipe, p in C.small_cases():
        if which == "brute" and p["shape"][1] > 40:
            continue  # brute force at r ~ 100 is slow; the fast port covers them
        got = _run(which, name, recipe, p)
        if got.tobytes() != golden_small[name].tobytes():
            bad.append(name)
    assert not bad, bad


def test_oracle_acceptance_matrix(golden):
    """Acceptance criterion 1 (test_acceptance.py:62-85): 3 dtypes x 13 images x
    9 radii x 5 percentiles at 256^2, byte-identical to the reference."""
    acc = golden["acceptance"]
    bad = []
    for dt in C.ACC_DTYPES:
        for idx, base in enumerate(C.acceptance_images()):
            img = C.as_dtype(base, dt)
            for r in C.ACC_RADII:
                for p in C.ACC_PERCENTILES:
                    out = oracle.fast_filter(img, ShapeSpec("circle", r), p, threads=8)
                    if C.digest(out) != acc[f"{dt}/{idx}/{r}/{p}"]:
                        bad.append((dt, idx, r, p))
    assert not bad, bad[:10]


def test_oracle_c1_digest(golden):
    img = C.baseline_input("c1")
    out = oracle.fast_filter(img, ShapeSpec("circle", 8), 0.5, threads=8)
    assert C.digest(out) == golden["baseline"]["c1"]


def test_oracle_forwarding_and_tiles_neutral():
    img = np.random.default_rng(3).integers(0, 65536, (150, 170)).astype(np.uint16)
    ref = oracle.fast_filter(img, ShapeSpec("circle", 9), 0.5)
    for ts in (16, 32, 64):
        for fwd in (True, False):
            assert np.array_equal(oracle.fast_filter(img, ShapeSpec("circle", 9), 0.5,
                                                     tile_size=ts, forwarding=fwd), ref)


def test_ordinal_known_answers():
    # test_ordinal.py:9-14: [[30,10],[20,5]] -> ranks [[3,1],[2,0]]
    ranks, px, py, vals = oracle.ordinal_transform(np.array([[30, 10], [20, 5]], np.uint8))
    assert ranks.tolist() == [[3, 1], [2, 0]]
    assert vals.tolist() == [5, 10, 20, 30]
    assert list(zip(px.tolist(), py.tolist())) == [(1, 1), (1, 0), (0, 1), (0, 0)]
    # ties take consecutive ranks in row-major order (test_ordinal.py:17-25)
    ranks, *_ = oracle.ordinal_transform(np.array([[29, 29], [1, 50]], np.uint8))
    assert ranks.tolist() == [[1, 2], [0, 3]]
    # constant tile -> row-major ranks (test_ordinal.py:28-30)
    ranks, *_ = oracle.ordinal_transform(np.full((3, 4), 7, np.uint16))
    assert ranks.ravel().tolist() == list(range(12))


def test_ordinal_float_order():
    v = np.array([[-np.inf, -1.0, -0.0, 0.0, 1e-38, 1.0, np.inf]], np.float32)
    ranks, *_ = oracle.ordinal_transform(v)
    assert ranks.ravel().tolist() == list(range(7))


def test_oracle_properties():
    rng = np.random.default_rng(11)
    img = rng.integers(0, 101, (64, 80)).astype(np.uint8)
    out = oracle.fast_filter(img, ShapeSpec("circle", 5), 0.3)
    lut = np.sort(rng.choice(256, size=101, replace=False)).astype(np.uint8)
    assert np.array_equal(oracle.fast_filter(lut[img], ShapeSpec("circle", 5), 0.3), lut[out])
    assert np.array_equal(oracle.fast_filter(img, ShapeSpec("circle", 0), 0.5), img)
