"""CPU oracle for the rank-order filter -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its CPU-baseline
leg and ``--impl reference`` arm) may import this package, and only as the
checker / the timed CPU reference; the product package
``paper_2505_22938_b200`` never imports it and has no CPU fallback.

``liboracle.so`` is a plain-C restatement of the reference ``isomedian``
algorithm (see isomedian_oracle.c for the file:line map):

* :func:`fast_filter`  -- the reference fast engine (``tiling.filter_image``):
  ordinal transform per tile, seed + horizontal/vertical pivot/count slides,
  64-rank segment refine, forwarding between tiles; multithreaded over tile
  columns like the reference's ThreadPoolExecutor (tiling.py:237-248).
* :func:`brute_filter` -- the reference brute oracle (``oracle.reference_filter``):
  gather every window and select rank t.
* :func:`ordinal_transform` -- ranks / positions / values of one tile.

Parity pinning: the restatement is checked against golden outputs of the real
reference (``tests/golden``, generated in the build container by
``tests/golden/make_golden.py``) before it is trusted as a checker.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _Kernel(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int), ("rad", ctypes.c_int), ("lim", ctypes.c_int64),
        ("nplanes", ctypes.c_int), ("planes", ctypes.c_void_p), ("area", ctypes.c_int),
        ("off_dx", ctypes.c_void_p), ("off_dy", ctypes.c_void_p),
        ("nrows", ctypes.c_int), ("row_dy", ctypes.c_void_p), ("row_xlo", ctypes.c_void_p),
        ("row_xhi", ctypes.c_void_p), ("ncols", ctypes.c_int), ("col_dx", ctypes.c_void_p),
        ("col_ytop", ctypes.c_void_p), ("col_ybot", ctypes.c_void_p),
    ]


def build() -> str:
    """Compile liboracle.so in place (make); returns its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "isomedian_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(path)
        p = ctypes.c_void_p
        lib.orc_filter_fast.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(_Kernel), ctypes.c_int64, p, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, p]
        lib.orc_filter_brute.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(_Kernel), ctypes.c_int64, p, ctypes.c_int, p]
        lib.orc_ordinal_transform.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              p, p, p, p]
        _LIB = lib
    return _LIB


_DT = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.float32): 2}


def to_keys(img: np.ndarray) -> np.ndarray:
    """u32 order keys: integers unchanged; f32 via the float order key
    (ordinal.py:109-123 / oracle.py:26-28)."""
    if img.dtype == np.float32:
        u = np.ascontiguousarray(img).view(np.uint32)
        return np.where(u >> 31, ~u, u | np.uint32(0x80000000)).astype(np.uint32)
    return np.ascontiguousarray(img, dtype=np.uint32)


def from_keys(keys: np.ndarray, dtype) -> np.ndarray:
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        u = np.where(keys >> 31, keys ^ np.uint32(0x80000000), ~keys).astype(np.uint32)
        return u.view(np.float32)
    return keys.astype(dtype)


def _kernel_struct(kernel):
    keep = [np.ascontiguousarray(a, dtype=np.int32) for a in
            (kernel.off_dx, kernel.off_dy, kernel.row_dy, kernel.row_xlo, kernel.row_xhi,
             kernel.col_dx, kernel.col_ytop, kernel.col_ybot)]
    planes = np.ascontiguousarray(kernel.planes, dtype=np.float64)
    keep.append(planes)
    ks = _Kernel(kernel.shape_code, kernel.radius, kernel.lim, planes.shape[0],
                 planes.ctypes.data, kernel.area, keep[0].ctypes.data, keep[1].ctypes.data,
                 len(kernel.row_dy), keep[2].ctypes.data, keep[3].ctypes.data, keep[4].ctypes.data,
                 len(kernel.col_dx), keep[5].ctypes.data, keep[6].ctypes.data, keep[7].ctypes.data)
    return ks, keep


def _targets(kernel, percentile, out_shape):
    from .kernel_geom import target_rank
    if np.isscalar(percentile) or np.ndim(percentile) == 0:
        return target_rank(kernel.area, float(percentile)), None
    pmap = np.asarray(percentile, dtype=np.float64)
    t = np.floor(pmap * (kernel.area - 1) + 0.5).astype(np.int64)
    return 0, np.ascontiguousarray(np.clip(t, 0, kernel.area - 1))


def _run(which, image, shape, percentile, boundary, threads, tile_size=None, forwarding=True):
    from .kernel_geom import kernel_of  # the oracle's own rasterization (kernels.py:127-182)
    image = np.asarray(image)
    if image.ndim == 3:
        return np.stack([_run(which, image[..., c], shape, percentile, boundary, threads,
                              tile_size, forwarding) for c in range(image.shape[2])], axis=-1)
    kernel = kernel_of(shape)
    r = shape.radius
    H, W = image.shape
    bnd = 1 if boundary == "valid" else 0
    out_h, out_w = (H - 2 * r, W - 2 * r) if bnd else (H, W)
    keys = to_keys(image)
    t, tmap = _targets(kernel, percentile, (out_h, out_w))
    out = np.empty((out_h, out_w), np.uint32)
    ks, keep = _kernel_struct(kernel)
    threads = threads or os.cpu_count() or 1
    lib = _lib()
    if which == "fast":
        st = lib.orc_filter_fast(keys.ctypes.data, H, W, _DT[image.dtype], bnd, ctypes.byref(ks),
                                 t, None if tmap is None else tmap.ctypes.data,
                                 tile_size or 0, 1 if forwarding else 0, threads, out.ctypes.data)
    else:
        st = lib.orc_filter_brute(keys.ctypes.data, H, W, bnd, ctypes.byref(ks), t,
                                  None if tmap is None else tmap.ctypes.data, threads,
                                  out.ctypes.data)
    if st != 0:
        raise RuntimeError(f"oracle {which} filter failed with status {st}")
    return from_keys(out, image.dtype)


def fast_filter(image, shape, percentile=0.5, boundary="replicate", threads=None,
                tile_size=None, forwarding=True):
    """Reference fast engine restated in C (tiling.py:213-249)."""
    return _run("fast", image, shape, percentile, boundary, threads, tile_size, forwarding)


def segment_stats(image, shape, percentile=0.5, boundary="replicate"):
    """Measured S-bar: mean 64-rank segments the reference
    refine scans per window, over one single-threaded fast-engine pass."""
    lib = _lib()
    lib.orc_segment_stats.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.orc_segment_stats(1, None, None)
    try:
        fast_filter(image, shape, percentile, boundary, threads=1)
    finally:
        segs, refines = ctypes.c_longlong(), ctypes.c_longlong()
        lib.orc_segment_stats(0, ctypes.byref(segs), ctypes.byref(refines))
    return segs.value / max(refines.value, 1)


def brute_filter(image, shape, percentile=0.5, boundary="replicate", threads=None):
    """Reference brute oracle restated in C (oracle.py:88-121)."""
    return _run("brute", image, shape, percentile, boundary, threads)


def ordinal_transform(tile: np.ndarray):
    """(ranks, pos_x, pos_y, values) of one tile (ordinal.py:126-172)."""
    tile = np.asarray(tile)
    h, w = tile.shape
    keys = to_keys(tile)
    ranks = np.empty((h, w), np.int32)
    px = np.empty(h * w, np.int32)
    py = np.empty(h * w, np.int32)
    vals = np.empty(h * w, np.uint32)
    st = _lib().orc_ordinal_transform(keys.ctypes.data, h, w, _DT[tile.dtype], ranks.ctypes.data,
                                      px.ctypes.data, py.ctypes.data, vals.ctypes.data)
    if st:
        raise ValueError(f"tile dimensions {h}x{w} out of range")
    return ranks, px, py, from_keys(vals, tile.dtype)
