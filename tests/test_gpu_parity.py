"""GPU parity: CUDA path vs golden outputs of the real reference (bit-exact)."""
import json

import numpy as np
import pytest

import cases as C

pytestmark = pytest.mark.gpu


def _params(p, out_shape=None):
    from paper_2505_22938_b200 import FilterParams, ShapeSpec
    kind, r, sides, rot = p["shape"]
    return FilterParams(shape=ShapeSpec(kind, r, sides, rot),
                        percentile=C.resolve_percentile(p["percentile"], out_shape),
                        boundary=p["boundary"])


@pytest.mark.parametrize("case", C.small_cases(), ids=lambda c: c[0])
def test_small_golden(case, golden_small):
    from paper_2505_22938_b200 import filter_image
    name, recipe, p = case
    img = C.make_input(recipe)
    out_shape = C.out_shape_of(img.shape, p["shape"][1], p["boundary"])
    got = filter_image(img, _params(p, out_shape))
    want = golden_small[name]
    assert got.dtype == want.dtype and got.shape == want.shape
    if got.tobytes() != want.tobytes():
        bad = np.argwhere(got.view(np.uint8) != want.view(np.uint8))
        raise AssertionError(f"{name}: {len(bad)} mismatching bytes, first at {bad[:5].tolist()}")
