"""Multi-percentile bracket (core.py:412-426 bracket_filter; test_core.py:254-266):
one ordinal transform per tile, one selection per percentile."""
import numpy as np
import pytest

import oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec, filter_image_bracket


def test_empty_percentile_list_rejected():
    with pytest.raises(ValueError, match="empty"):
        filter_image_bracket(np.zeros((8, 8), np.uint8), FilterParams(shape=ShapeSpec("circle", 1)),
                             [])
    with pytest.raises(ValueError, match="percentile"):
        filter_image_bracket(np.zeros((8, 8), np.uint8), FilterParams(shape=ShapeSpec("circle", 1)),
                             [0.5, 1.5])


@pytest.mark.gpu
def test_bracket_matches_single_percentile_runs():
    # the reference test's case: 40x40 u8 tile, circle r=5, valid mode
    rng = np.random.default_rng(254)
    tile = rng.integers(0, 256, (40, 40)).astype(np.uint8)
    ps = [0.0, 0.25, 0.5, 0.75, 1.0]
    params = FilterParams(shape=ShapeSpec("circle", 5), boundary="valid")
    outs = filter_image_bracket(tile, params, ps)
    assert len(outs) == len(ps)
    for out, p in zip(outs, ps):
        assert out.shape == (30, 30)
        assert np.array_equal(out, oracle.brute_filter(tile, params.shape, p, "valid"))


@pytest.mark.gpu
@pytest.mark.parametrize("dt,shape", [("uint16", ("circle", 20, 0, 0.0)),
                                      ("float32", ("circle", 70, 0, 0.0)),
                                      ("uint8", ("regular_polygon", 9, 6, 0.0))])
def test_bracket_full_images(dt, shape):
    import torch
    rng = np.random.default_rng(7)
    if dt == "float32":
        img = rng.standard_normal((300, 260)).astype(np.float32)
    else:
        img = rng.integers(0, np.iinfo(dt).max + 1, (300, 260, 3)).astype(dt)
    spec = ShapeSpec(*shape)
    ps = [0.1, 0.5, 0.9]
    outs = filter_image_bracket(torch.from_numpy(img).cuda(), FilterParams(shape=spec), ps)
    for out, p in zip(outs, ps):
        assert out.is_cuda
        want = oracle.fast_filter(img, spec, p)
        assert out.cpu().numpy().tobytes() == want.tobytes(), p
