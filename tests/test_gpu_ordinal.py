"""Device-side ordinal transform (K1 of one tile, imf_tile_omega) against the
reference's invariants (/root/reference/pkg/tests/test_ordinal.py:33-63 --
permutation, mutual inverse, sorted reverse map consistent with the source)
and against the oracle's ordinal transform of the same tile (identical sorted
values; tie order is free on the device)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [  # dtype, image shape, kernel, tiles
    (np.uint16, (300, 280, 3), ("circle", 48, 0), [0, 7, 12, 20]),      # c2-like: footprint, HWC
    (np.uint8, (260, 250), ("regular_polygon", 20, 6), [0, 3, 8]),       # polygon footprint
    (np.uint8, (200, 220), ("square", 12, 0), [0, 5]),                   # no footprint (square)
    (np.uint16, (420, 400), ("circle", 64, 0), [0, 4, 13]),              # planar u16: TMA loads
    (np.float32, (300, 300), ("circle", 40, 0), [0, 5, 10]),             # f32 adaptive buckets
    (np.float32, (330, 310), ("circle", 60, 0), [0, 3, 11]),             # f32 16-bit shared entries
    (np.uint16, (180, 170), ("circle", 62, 0), [0, 2]),                  # halved ranks (N > 32768)
]


def _img(rng, dt, shape):
    if dt == np.float32:
        a = rng.standard_normal(shape).astype(np.float32)
        a[rng.random(shape) < 0.2] = np.float32(0.5)  # planted duplicates
        return a
    hi = 256 if dt == np.uint8 else 65536
    a = rng.integers(0, hi, shape).astype(dt)
    a[rng.random(shape) < 0.1] = 7
    return a


@pytest.mark.parametrize("case", range(len(CASES)))
def test_tile_ordinal_invariants(case):
    import torch
    from paper_2505_22938_b200 import FilterParams, ShapeSpec
    from paper_2505_22938_b200.ordinal import tile_ordinal
    dt, shape, (kind, r, sides), tiles = CASES[case]
    rng = np.random.default_rng(100 + case)
    img = _img(rng, dt, shape)
    params = FilterParams(shape=ShapeSpec(kind, r, sides=sides))
    t = torch.from_numpy(img).cuda()
    for tile in tiles:
        ot = tile_ordinal(t, params, tile)
        n = ot.count
        ranked = ot.ranks >= 0
        # permutation of the ranked pixels, and the two maps are mutual inverses
        assert int(ranked.sum()) == n
        assert sorted(ot.ranks[ranked].tolist()) == list(range(n))
        assert np.array_equal(ot.ranks[ot.pos_y, ot.pos_x], np.arange(n))
        # reverse map sorted (by the float order key for f32), consistent with the source
        key = oracle.to_keys(ot.values) if dt == np.float32 else ot.values.astype(np.int64)
        assert np.all(key[:-1] <= key[1:])
        plane = img[..., ot.channel] if img.ndim == 3 else img
        src = ot.tile_values(plane)
        assert np.array_equal(src[ot.pos_y, ot.pos_x].view(np.uint8), ot.values.view(np.uint8))
        # the same sorted values as a sort of the ranked pixels; without a footprint
        # (every pixel ranked) the same as the reference algorithm's transform
        kr = oracle.to_keys(src[ranked]) if dt == np.float32 else src[ranked].astype(np.int64)
        assert np.array_equal(np.sort(kr), key)
        if not ot.footprint:
            ref = oracle.ordinal_transform(src)[3]
            assert np.array_equal(ref.view(np.uint8), ot.values.view(np.uint8))
