"""Host prologue parity (CPU): kernel rasterization and target ranks.

Mirrors the reference's tests/test_kernels.py known answers and checks every
span table against digests of the REAL reference's make_kernel
(tests/golden/golden.json, produced by make_golden.py in the build container).
"""
import json

import numpy as np
import pytest

import cases as C
from paper_2505_22938_b200 import ShapeSpec, contains, make_kernel, target_rank


def test_span_tables_match_reference_digests(golden):
    bad = []
    for key, dig in golden["kernels"].items():
        spec = tuple(json.loads(key))
        if C.kernel_digest(make_kernel(ShapeSpec(*spec))) != dig:
            bad.append(spec)
    assert not bad, bad[:5]
    assert len(golden["kernels"]) >= 300


def test_known_areas():
    assert make_kernel(ShapeSpec("circle", 2)).area == 21
    k0 = make_kernel(ShapeSpec("circle", 0))
    assert k0.area == 1 and k0.offsets == {(0, 0)}
    assert make_kernel(ShapeSpec("circle", 1)).area == 9
    assert make_kernel(ShapeSpec("square", 2)).area == 25
    assert not contains(ShapeSpec("circle", 2), 2, 2)
    assert contains(ShapeSpec("circle", 2), 2, 1)


def test_baseline_kernel_geometry():
    # areas and row/column counts of the BASELINE kernels
    for spec, area, rows, cols in [(("circle", 8), 225, 17, 17), (("circle", 48), 7393, 97, 97),
                                   (("circle", 64), 13085, 129, 129),
                                   (("circle", 100), 31757, 201, 201),
                                   (("square", 32), 4225, 65, 65),
                                   (("regular_polygon", 32, 6), 2765, 57, 65),
                                   (("regular_polygon", 32, 12), 3177, 65, 65)]:
        k = make_kernel(ShapeSpec(*spec))
        assert (k.area, len(k.row_dy), len(k.col_dx)) == (area, rows, cols), spec


@pytest.mark.parametrize("spec", [ShapeSpec("circle", r) for r in (0, 1, 2, 5, 16, 48, 124)]
                         + [ShapeSpec("square", 4),
                            ShapeSpec("regular_polygon", 9, sides=3, rotation_deg=90.0),
                            ShapeSpec("regular_polygon", 12, sides=12, rotation_deg=7.5)])
def test_slide_round_trip(spec):
    k = make_kernel(spec)
    offs = k.offsets
    h_enter, h_exit = k.h_deltas
    right = {(dx + 1, dy) for dx, dy in offs}
    assert (offs - {tuple(e) for e in h_exit}) | {tuple(e) for e in h_enter} == right
    v_enter, v_exit = k.v_deltas
    down = {(dx, dy + 1) for dx, dy in offs}
    assert (offs - {tuple(e) for e in v_exit}) | {tuple(e) for e in v_enter} == down
    assert k.area == int(np.sum(k.row_xhi - k.row_xlo))


def test_target_rank():
    assert target_rank(49, 0.5) == 24
    assert target_rank(21, 0.5) == 10
    for n in (1, 2, 21, 49):
        assert target_rank(n, 0.0) == 0
        assert target_rank(n, 1.0) == n - 1
    with pytest.raises(ValueError):
        target_rank(21, 1.5)
    with pytest.raises(ValueError):
        target_rank(21, -0.1)


def test_shape_validation():
    with pytest.raises(ValueError):
        ShapeSpec("hexagon", 3)
    with pytest.raises(ValueError):
        ShapeSpec("circle", -1)
    with pytest.raises(ValueError):
        ShapeSpec("regular_polygon", 3, sides=2)
    with pytest.raises(ValueError, match="64 sides"):
        make_kernel(ShapeSpec("regular_polygon", 3, sides=65))
