"""Drop-in surface and C ABI checks that need no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2505_22938_b200 import FilterParams, ShapeSpec, _lib, decompose, filter_image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "isomedian_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(imf_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2505_22938_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 9
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED) == set(names)
    L = _lib.load()
    assert L.imf_version() >= 100
    assert L.imf_strerror(3).decode().startswith("segment scan exhausted")


def test_workspace_size_without_gpu():
    L = _lib.load()
    from paper_2505_22938_b200 import make_kernel
    from paper_2505_22938_b200.tiling import _kernel_struct
    ks, keep = _kernel_struct(make_kernel(ShapeSpec("circle", 48)))
    img = _lib.ImfImage(None, 1, 1, 2160, 3840, 3, 0, 3840 * 3, 3, 1)
    opt = _lib.ImfOptions(0, 0, 0, 0)
    need = L.imf_workspace_size(ctypes.byref(img), ctypes.byref(ks), ctypes.byref(opt))
    assert need > 0
    img.height = 0
    assert L.imf_workspace_size(ctypes.byref(img), ctypes.byref(ks), ctypes.byref(opt)) == 0


def _p(r=2, **kw):
    return FilterParams(shape=ShapeSpec("circle", r), **kw)


def test_validation_messages_match_reference():
    # tiling.py:216-226 / test_tiling.py:119-131, raised before any device work
    with pytest.raises(ValueError, match="dtype"):
        filter_image(np.zeros((9, 9), np.int32), _p())
    with pytest.raises(ValueError, match="unsupported image dtype >u2"):
        filter_image(np.zeros((9, 9), ">u2"), _p())
    bad = np.ones((9, 9), np.float32)
    bad[3, 3] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        filter_image(bad, _p())
    with pytest.raises(ValueError, match="non-empty 2D or 3D"):
        filter_image(np.zeros((0, 5), np.uint8), _p())
    with pytest.raises(ValueError, match="non-empty 2D or 3D"):
        filter_image(np.zeros((2, 3, 4, 5), np.uint8), _p())
    with pytest.raises(ValueError, match="radius 125 exceeds the maximum of 124"):
        filter_image(np.zeros((300, 300), np.uint8), _p(125))
    with pytest.raises(ValueError, match="image smaller than the kernel in valid mode"):
        filter_image(np.zeros((6, 6), np.uint8), _p(3, boundary="valid"))
    with pytest.raises(ValueError, match="shape"):
        filter_image(np.zeros((10, 12), np.uint8), _p(percentile=np.zeros((3, 3))))
    with pytest.raises(ValueError, match="percentile"):
        FilterParams(shape=ShapeSpec("circle", 2), percentile=1.5)
    with pytest.raises(ValueError, match="boundary"):
        FilterParams(shape=ShapeSpec("circle", 2), boundary="reflect")


def test_decompose_matches_reference_rules():
    g = decompose((256, 256), _p(16, forwarding=False))
    assert g.tile_size == 64
    assert decompose((400, 400), _p(100, forwarding=False)).tile_size == 56
    assert decompose((400, 400), _p(100, forwarding=True)).tile_size == 55
    with pytest.raises(ValueError, match="radius"):
        decompose((400, 400), _p(125))
    with pytest.raises(ValueError):
        decompose((400, 400), _p(100, tile_size=60))
    assert (decompose((100, 100), _p(10, boundary="valid")).out_h,) == (80,)


def test_no_cpu_fallback(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        filter_image(np.zeros((9, 9), np.uint8), _p())
