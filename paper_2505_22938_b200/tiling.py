"""Drop-in entry point: ``filter_image(image, FilterParams)`` on the B200.

Mirrors the public surface of the reference ``isomedian.tiling``
(/root/reference/pkg/src/isomedian/tiling.py) -- same dataclass fields and
defaults, same validation order, same exception types and messages -- and
replaces everything below the host prologue (padding, tiling, the thread
pool, the per-tile ordinal transform and selection, tiling.py:228-249) with
one call into the CUDA extension (C ABI: include/isomedian_b200.h).

``forwarding``, ``workers`` and ``footprint_mask`` are accepted and
output-neutral, exactly as in the reference (test_tiling.py:71-85,113-116);
the GPU tiles independently.  ``tile_size`` keeps the reference validation
(tiling.py:110-117) and is passed to the kernels as the output-tile side.

Inputs may be numpy arrays or torch tensors (CPU or CUDA); the result has the
same kind (and device).  There is no CPU fallback: without the extension or a
GPU the call raises.
"""

from __future__ import annotations

import collections
import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import MAX_RADIUS, ShapeSpec, make_kernel, target_rank

MAX_TILE_SIDE = 256
DEFAULT_OUTPUT_TILE = 64


class ScanDefectError(RuntimeError):
    """A segment scan ran off the end of the rank array (core.py:31-36).

    Signals an internal invariant violation (never an input-data condition).
    """


@dataclass(frozen=True)
class FilterParams:
    """Filter-level parameters: kernel, percentile, boundary, and tiling.

    Same fields, defaults and validation as tiling.py:27-45.
    """

    shape: ShapeSpec
    percentile: float | np.ndarray = 0.5
    boundary: str = "replicate"
    forwarding: bool = True
    tile_size: int | None = None
    workers: int | None = None
    footprint_mask: bool = False

    def __post_init__(self):
        if self.boundary not in ("replicate", "valid"):
            raise ValueError(f"unknown boundary mode {self.boundary!r}")
        if np.isscalar(self.percentile) or np.ndim(self.percentile) == 0:
            p = float(self.percentile)
            if not 0.0 <= p <= 1.0:
                raise ValueError("percentile must be in [0, 1]")


@dataclass(frozen=True)
class Tile:
    """One tile of the reference schedule (tiling.py:46-78): an output
    rectangle and the padded-input rectangle it reads (one extra row above
    when seeded by the tile above).  The GPU picks its own tiles (output is
    tile-invariant); this is the reference-facing description."""

    out_x0: int
    out_y0: int
    out_w: int
    out_h: int
    seeded: bool
    radius: int

    @property
    def in_x0(self) -> int:
        return self.out_x0

    @property
    def in_y0(self) -> int:
        return self.out_y0 - int(self.seeded)

    @property
    def in_w(self) -> int:
        return self.out_w + 2 * self.radius

    @property
    def in_h(self) -> int:
        return self.out_h + 2 * self.radius + int(self.seeded)


@dataclass(frozen=True)
class TileGrid:
    """Reference tile grid (tiling.py:81-91): columns of tiles, top to bottom."""

    out_h: int
    out_w: int
    tile_size: int
    columns: list
    forwarding: bool

    @property
    def tiles(self) -> list:
        return [t for col in self.columns for t in col]


def decompose(image_shape: tuple[int, int], params: FilterParams) -> TileGrid:
    """The reference's tile grid with its validation (tiling.py:94-131)."""
    h, w, t = _grid_size(image_shape, params)
    r = params.shape.radius
    fw = params.forwarding
    columns = [[Tile(out_x0=x0, out_y0=y0, out_w=min(t, w - x0), out_h=min(t, h - y0),
                     seeded=fw and y0 > 0, radius=r) for y0 in range(0, h, t)]
               for x0 in range(0, w, t)]
    return TileGrid(out_h=h, out_w=w, tile_size=t, columns=columns, forwarding=fw)


def _grid_size(image_shape, params: FilterParams):
    """(out_h, out_w, tile) after the reference checks (tiling.py:94-131), in
    its order and with its messages; no Tile objects (host prologue)."""
    r = params.shape.radius
    if r > MAX_RADIUS:
        raise ValueError(
            f"radius {r} exceeds the maximum of {MAX_RADIUS} (input tiles "
            "are capped at 256 pixels per side)")
    h, w = image_shape
    if params.boundary == "valid":
        h, w = h - 2 * r, w - 2 * r
        if h <= 0 or w <= 0:
            raise ValueError("image smaller than the kernel in valid mode")
    if h <= 0 or w <= 0:
        raise ValueError("image is empty")
    seed_extra = 1 if params.forwarding else 0
    if params.tile_size is not None:
        t = params.tile_size
        if t < 1:
            raise ValueError("tile size must be positive")
        if t + 2 * r + seed_extra > MAX_TILE_SIDE:
            raise ValueError(
                f"tile size {t} with radius {r} exceeds the "
                f"{MAX_TILE_SIDE}-pixel input tile cap")
    else:
        t = min(DEFAULT_OUTPUT_TILE, MAX_TILE_SIDE - 2 * r - seed_extra)
    return h, w, t


def pad_image(image: np.ndarray, r: int, mode: str) -> np.ndarray:
    """Host padding helper kept for API parity (tiling.py:134-145).

    The GPU path never materializes the padded image: replicate padding is a
    coordinate clamp inside the tile load.
    """
    if mode == "replicate":
        if r == 0:
            return image
        pads = ((r, r), (r, r)) + ((0, 0),) * (image.ndim - 2)
        return np.pad(image, pads, mode="edge")
    if mode == "valid":
        if image.shape[0] < 2 * r + 1 or image.shape[1] < 2 * r + 1:
            raise ValueError("image smaller than the kernel in valid mode")
        return image
    raise ValueError(f"unknown boundary mode {mode!r}")


# ----------------------------------------------------------------- helpers

_DTYPES = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.float32): 2}


def _torch():
    import torch
    return torch


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _np_dtype_of(x) -> np.dtype:
    if _is_tensor(x):
        torch = _torch()
        m = {torch.uint8: np.uint8, torch.uint16: np.uint16, torch.float32: np.float32}
        if x.dtype not in m:
            return np.dtype(str(x.dtype).replace("torch.", ""))
        return np.dtype(m[x.dtype])
    return x.dtype


def _check_dtype(dt):
    if dt not in _DTYPES:
        raise ValueError(f"unsupported image dtype {dt}; use uint8, uint16, or float32")


def _target_spec(area: int, percentile, out_shape, device, host: bool = False):
    """(scalar target, target map or None, tmin, tmax) -- tiling.py:165-177.

    The map is an int32 CUDA tensor on `device`, or a contiguous int32 numpy
    array when `host` is set (for imf_filter_host)."""
    if np.isscalar(percentile) or np.ndim(percentile) == 0:
        t = target_rank(area, float(percentile))
        return t, None, t, t
    if _is_tensor(percentile):
        pmap = percentile.detach().cpu().numpy().astype(np.float64)
    else:
        pmap = np.asarray(percentile, dtype=np.float64)
    if pmap.shape != tuple(out_shape):
        raise ValueError(
            f"percentile map shape {pmap.shape} does not match the output "
            f"shape {tuple(out_shape)}")
    if pmap.min() < 0.0 or pmap.max() > 1.0:
        raise ValueError("percentile map values must lie in [0, 1]")
    targets = np.clip(np.floor(pmap * (area - 1) + 0.5).astype(np.int64), 0, area - 1)
    if host:
        return 0, np.ascontiguousarray(targets, dtype=np.int32), int(targets.min()), int(targets.max())
    torch = _torch()
    tmap = torch.from_numpy(targets.astype(np.int32)).to(device)
    return 0, tmap, int(targets.min()), int(targets.max())


class _Workspace:
    """Cached device workspace per (device, stream), grown on demand.

    The workspace holds the omega scratch and the status word of a call, so
    two calls in flight on different streams must not share one: the cache
    key includes the stream.  A buffer is allocated on (and only ever used
    by) its own stream, so the caching allocator's stream tracking is exact.
    """

    MAX_ENTRIES = 8  # least recently used (device, stream) workspaces beyond this are dropped

    def __init__(self):
        self.buf = collections.OrderedDict()
        self.lock = threading.Lock()

    def get(self, device, nbytes: int, stream=None):
        torch = _torch()
        idx = device.index if device.index is not None else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(idx)
        key = (idx, stream.cuda_stream)
        with self.lock:
            cur = self.buf.get(key)
            if cur is None or cur.numel() < nbytes:
                with torch.cuda.stream(stream):
                    cur = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=torch.device("cuda", idx))
                self.buf[key] = cur
            self.buf.move_to_end(key)
            # callers that make a stream per call must not pin a workspace per
            # stream: a dropped buffer was only ever used on its own stream, so
            # the caching allocator reuses it there in stream order
            while len(self.buf) > self.MAX_ENTRIES:
                self.buf.popitem(last=False)
            return cur


_WS = _Workspace()


def workspace_for(device, stream=None):
    """The cached device workspace of (device, stream) (holds the status word
    of the last call on that stream)."""
    return _WS.get(device, 1, stream)


_KSTRUCT = {}  # id(kernel) -> (kernel, imf_kernel, arrays it points into); kernels are immutable


def _kernel_struct(kernel):
    hit = _KSTRUCT.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit[1], hit[2]
    keep = [np.ascontiguousarray(a, dtype=np.int32) for a in
            (kernel.row_dy, kernel.row_xlo, kernel.row_xhi, kernel.col_dx,
             kernel.col_ytop, kernel.col_ybot)]
    ks = _lib.ImfKernel(kernel.shape_code, kernel.radius, kernel.area, len(kernel.row_dy),
                        keep[0].ctypes.data, keep[1].ctypes.data, keep[2].ctypes.data,
                        len(kernel.col_dx), keep[3].ctypes.data, keep[4].ctypes.data,
                        keep[5].ctypes.data)
    if len(_KSTRUCT) > 256:
        _KSTRUCT.clear()
    _KSTRUCT[id(kernel)] = (kernel, ks, keep)
    return ks, keep


def _image_struct(t, dt_code, batched: bool, has_c: bool):
    """imf_image for a CUDA tensor of shape ([B,] H, W[, C])."""
    shape = list(t.shape)
    strides = list(t.stride())
    if not has_c:
        shape.append(1)
        strides.append(0)
    if not batched:
        shape.insert(0, 1)
        strides.insert(0, 0)
    b, h, w, c = shape
    sb, sy, sx, sc = strides
    return _lib.ImfImage(t.data_ptr(), dt_code, b, h, w, c, sb, sy, sx, sc)


def run_device(src, params: FilterParams, out=None, *, batched: bool = False, stream=None,
               check: bool = True, kernel=None, profile: bool = False):
    """Filter a CUDA tensor ([B,] H, W[, C]) into a new (or given) CUDA tensor.

    Host prologue (validation, kernel, targets) is the caller's job except for
    the target map; this is the device half of :func:`filter_image`.
    """
    torch = _torch()
    with torch.cuda.device(src.device):  # streams, workspace and launches on src's device
        return _run_device(src, params, out, batched, stream, check, kernel, profile)


def _run_device(src, params, out, batched, stream, check, kernel, profile):
    torch = _torch()
    L = _lib.lib()
    dt = _np_dtype_of(src)
    dt_code = _DTYPES[dt]
    kernel = kernel or make_kernel(params.shape)
    r = params.shape.radius
    has_c = src.dim() == (4 if batched else 3)
    h, w = src.shape[1:3] if batched else src.shape[0:2]
    valid = params.boundary == "valid"
    out_h, out_w = (h - 2 * r, w - 2 * r) if valid else (h, w)
    hy = 1 if batched else 0
    oshape = list(src.shape)
    oshape[hy], oshape[hy + 1] = out_h, out_w
    if out is None:
        out = torch.empty(oshape, dtype=src.dtype, device=src.device)
    elif out.dtype != src.dtype or list(out.shape) != oshape or out.device != src.device:
        raise ValueError(f"out must be a {src.dtype} tensor of shape {tuple(oshape)} on {src.device}")
    cur = torch.cuda.current_stream(src.device)
    if stream is None:
        stream = cur
    target, tmap, tmin, tmax = _target_spec(kernel.area, params.percentile, (out_h, out_w),
                                            src.device)
    if stream.cuda_stream != cur.cuda_stream:
        # src / out / the target map were produced on the current stream: order
        # the launch after them, and keep their memory alive until `stream` is done
        stream.wait_stream(cur)
        for t in (src, out, tmap):
            if t is not None:
                t.record_stream(stream)
    ks, keep = _kernel_struct(kernel)
    simg = _image_struct(src, dt_code, batched, has_c)
    dimg = _image_struct(out, dt_code, batched, has_c)
    opt = _lib.ImfOptions(1 if valid else 0, int(params.tile_size or 0), 0, 0)
    if profile:
        opt.flags = _lib.IMF_FLAG_PROFILE  # per-kernel CUDA-event timing (synchronizes)
    need = L.imf_workspace_size(ctypes.byref(simg), ctypes.byref(ks), ctypes.byref(opt))
    if need == 0:
        raise ValueError("unsupported filter geometry for the CUDA engine")
    ws = _WS.get(src.device, need, stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    st = L.imf_filter(ctypes.byref(simg), ctypes.byref(dimg), ctypes.byref(ks), target,
                      None if tmap is None else tmap.data_ptr(), tmin, tmax, ctypes.byref(opt),
                      ws.data_ptr(), ws.numel(), sptr)
    if st != _lib.IMF_OK:
        raise RuntimeError(f"imf_filter failed: {_lib.strerror(st)}")
    if check:
        st = L.imf_workspace_status(ws.data_ptr(), sptr)
        if st == _lib.IMF_ERR_DEFECT:
            raise ScanDefectError("segment scan exhausted while solving tile; "
                                  "pivot/count state was inconsistent")
        if st != _lib.IMF_OK:
            raise RuntimeError(f"imf_filter failed: {_lib.strerror(st)}")
    del keep, tmap
    return out


def _validate_plane(shape2d, dt, has_nan, params: FilterParams):
    """tiling.py:222-233 checks for one 2D plane, in the reference order."""
    if len(shape2d) != 2 or shape2d[0] * shape2d[1] == 0:
        raise ValueError("image must be a non-empty 2D or 3D array")
    if dt == np.float32 and has_nan():
        raise ValueError("image contains NaN; NaN has no rank under the "
                         "total order used by this filter")
    kernel = make_kernel(params.shape)
    out_h, out_w, _ = _grid_size(tuple(shape2d), params)
    if params.boundary == "valid":
        pad_image_check(shape2d, params.shape.radius)
    if not (np.isscalar(params.percentile) or np.ndim(params.percentile) == 0):
        pshape = tuple(np.shape(params.percentile))
        if pshape != (out_h, out_w):
            raise ValueError(
                f"percentile map shape {pshape} does not match the output "
                f"shape {(out_h, out_w)}")
    return kernel, (out_h, out_w)


def pad_image_check(shape2d, r):
    if shape2d[0] < 2 * r + 1 or shape2d[1] < 2 * r + 1:
        raise ValueError("image smaller than the kernel in valid mode")


def filter_image(image, params: FilterParams):
    """Rank-order filter a full image on the GPU (drop-in for tiling.py:213)."""
    is_t = _is_tensor(image)
    if not is_t:
        image = np.asarray(image)
    dt = _np_dtype_of(image)
    _check_dtype(dt)
    ndim = image.dim() if is_t else image.ndim
    shape = tuple(image.shape)
    if is_t:
        has_nan = lambda: bool(_torch().isnan(image).any()) if dt == np.float32 else False
    else:
        has_nan = lambda: bool(np.isnan(image).any())
    if ndim == 3:
        if shape[2] == 0:
            raise ValueError("need at least one array to concatenate")
        kernel, _ = _validate_plane(shape[:2], dt, has_nan, params)
    else:
        kernel, _ = _validate_plane(shape, dt, has_nan, params)

    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 rank-order filter needs a CUDA device (no CPU fallback)")
    if is_t and image.is_cuda:
        return run_device(image, params, kernel=kernel)
    if is_t:
        return torch.from_numpy(run_host(image.numpy(), params, kernel=kernel))
    return run_host(image, params, kernel=kernel)


def _host_image_struct(a: np.ndarray, dt_code: int, batched: bool):
    """imf_image for a host array of shape ([B,] H, W[, C]) (strides in elements)."""
    it = a.itemsize
    shape, strides = list(a.shape), [st // it for st in a.strides]
    has_c = a.ndim == (4 if batched else 3)
    if not has_c:
        shape.append(1)
        strides.append(0)
    if not batched:
        shape.insert(0, 1)
        strides.insert(0, 0)
    b, h, w, c = shape
    sb, sy, sx, sc = strides
    return _lib.ImfImage(a.ctypes.data, dt_code, b, h, w, c, sb, sy, sx, sc)


def run_host(image, params: FilterParams, out=None, *, batched: bool = False, kernel=None,
             stream=None, rows=None) -> np.ndarray:
    """Filter a HOST array through the C-ABI host entry point (imf_filter_host).

    The extension uploads, filters and downloads in output-row stripes on
    three streams, so the copies of one stripe overlap the filter of another
    (include/isomedian_b200.h).  `image` may be a numpy array or a CPU torch
    tensor (pinned memory gives full copy bandwidth); the result is a numpy
    array (or `out`, a host array/tensor of the output shape, filled in place).
    `rows=(y0, y1)` filters output rows [y0, y1) only (the other rows of `out`
    are left as they are): one device's stripe of a multi-device job.
    """
    torch = _torch()
    L = _lib.lib()
    a = image.numpy() if _is_tensor(image) else image
    if a.dtype.byteorder not in ("=", "|") or any(st % a.itemsize for st in a.strides) or \
            any(st < 0 for st in a.strides):
        a = np.ascontiguousarray(a)
    dt_code = _DTYPES[a.dtype]
    kernel = kernel or make_kernel(params.shape)
    r = params.shape.radius
    valid = params.boundary == "valid"
    hy = 1 if batched else 0
    h, w = a.shape[hy], a.shape[hy + 1]
    out_h, out_w = (h - 2 * r, w - 2 * r) if valid else (h, w)
    oshape = list(a.shape)
    oshape[hy], oshape[hy + 1] = out_h, out_w
    stage = None
    if out is None:
        o = np.empty(oshape, dtype=a.dtype)
    else:
        o = out.numpy() if _is_tensor(out) else out
        if not isinstance(o, np.ndarray) or o.dtype != a.dtype or list(o.shape) != oshape:
            raise ValueError(f"out must be a {a.dtype} host array of shape {tuple(oshape)}")
        if not o.flags.c_contiguous:
            # the C ABI copies results back as whole row ranges (dense dst only):
            # filter into a dense buffer, then scatter into the caller's view
            stage, o = o, np.empty(oshape, dtype=a.dtype)
    target, tmap, tmin, tmax = _target_spec(kernel.area, params.percentile, (out_h, out_w), None,
                                            host=True)
    ks, keep = _kernel_struct(kernel)
    simg = _host_image_struct(a, dt_code, batched)
    dimg = _host_image_struct(o, dt_code, batched)
    opt = _lib.ImfOptions(1 if valid else 0, int(params.tile_size or 0), 0, 0)
    if rows is not None:
        y0, y1 = int(rows[0]), int(rows[1])
        if not 0 <= y0 < y1 <= out_h:
            raise ValueError(f"row range {rows} outside the {out_h} output rows")
        if stage is not None:  # rows outside the range must keep the caller's values
            np.copyto(o, stage)
        opt.row_begin, opt.row_end = y0, y1
    if stream is None:
        stream = torch.cuda.current_stream()
    st = L.imf_filter_host(ctypes.byref(simg), ctypes.byref(dimg), ctypes.byref(ks), target,
                           None if tmap is None else tmap.ctypes.data, tmin, tmax,
                           ctypes.byref(opt), ctypes.c_void_p(stream.cuda_stream))
    del keep
    if st == _lib.IMF_ERR_DEFECT:
        raise ScanDefectError("segment scan exhausted while solving tile; "
                              "pivot/count state was inconsistent")
    if st != _lib.IMF_OK:
        raise RuntimeError(f"imf_filter_host failed: {_lib.strerror(st)}")
    if stage is not None:
        np.copyto(stage, o)
    return out if out is not None else o


def filter_batch(images, params: FilterParams, out=None, *, check: bool = True, stream=None):
    """Filter a CUDA batch (B, H, W[, C]) in one launch sequence (images share params)."""
    if not images.is_cuda:
        raise ValueError("filter_batch expects a CUDA tensor")
    dt = _np_dtype_of(images)
    _check_dtype(dt)
    kernel, _ = _validate_plane(tuple(images.shape[1:3]), dt,
                                lambda: bool(_torch().isnan(images).any()) if dt == np.float32
                                else False, params)
    return run_device(images, params, out=out, batched=True, check=check, stream=stream,
                      kernel=kernel)


def filter_image_bracket(image, params: FilterParams, percentiles) -> list:
    """Rank-order "bracketing": one output per percentile, one ordinal transform.

    Image-level counterpart of the reference's tile-level
    ``bracket_filter(ot, kernel, percentiles, ...)`` (core.py:412-426, SPEC
    "[OP] bracket_filter"): every output equals
    ``filter_image(image, replace(params, percentile=p))`` for its p, but each
    tile is rank-transformed once (K1) and selected once per percentile (K2),
    through ``imf_filter_bracket``.  ``params.percentile`` is ignored.  Inputs
    and outputs follow :func:`filter_image` (numpy in -> numpy out, torch ->
    torch on the same device).
    """
    percentiles = list(percentiles)
    if not percentiles:
        raise ValueError("percentile list is empty")
    for p in percentiles:
        if not 0.0 <= float(p) <= 1.0:
            raise ValueError("percentile must be in [0, 1]")
    is_t = _is_tensor(image)
    if not is_t:
        image = np.asarray(image)
    dt = _np_dtype_of(image)
    _check_dtype(dt)
    ndim = image.dim() if is_t else image.ndim
    shape = tuple(image.shape)
    if is_t:
        has_nan = lambda: bool(_torch().isnan(image).any()) if dt == np.float32 else False
    else:
        has_nan = lambda: bool(np.isnan(image).any())
    if ndim == 3 and shape[2] == 0:
        raise ValueError("need at least one array to concatenate")
    kernel, grid = _validate_plane(shape[:2] if ndim == 3 else shape, dt, has_nan,
                                   FilterParams(shape=params.shape, boundary=params.boundary,
                                                tile_size=params.tile_size))
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 rank-order filter needs a CUDA device (no CPU fallback)")
    if is_t:
        src = image if image.is_cuda else image.to("cuda")
    else:
        src = torch.from_numpy(np.ascontiguousarray(image)).to("cuda")
    with torch.cuda.device(src.device):
        outs = _bracket_device(src, dt, kernel, grid, params, percentiles)
    if is_t:
        return outs if image.is_cuda else [o.cpu() for o in outs]
    return [o.cpu().numpy() for o in outs]


def _bracket_device(src, dt, kernel, out_hw, params, percentiles):
    torch = _torch()
    L = _lib.lib()
    dt_code = _DTYPES[dt]
    has_c = src.dim() == 3
    oshape = list(src.shape)
    oshape[0], oshape[1] = out_hw
    outs = [torch.empty(oshape, dtype=src.dtype, device=src.device) for _ in percentiles]
    targets = (ctypes.c_int32 * len(percentiles))(*[target_rank(kernel.area, float(p))
                                                   for p in percentiles])
    dimgs = (_lib.ImfImage * len(outs))(*[_image_struct(o, dt_code, False, has_c) for o in outs])
    ks, keep = _kernel_struct(kernel)
    simg = _image_struct(src, dt_code, False, has_c)
    opt = _lib.ImfOptions(1 if params.boundary == "valid" else 0, int(params.tile_size or 0), 0, 0)
    need = L.imf_workspace_size(ctypes.byref(simg), ctypes.byref(ks), ctypes.byref(opt))
    if need == 0:
        raise ValueError("unsupported filter geometry for the CUDA engine")
    stream = torch.cuda.current_stream(src.device)
    ws = _WS.get(src.device, need, stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    st = L.imf_filter_bracket(ctypes.byref(simg), dimgs, len(outs), targets, ctypes.byref(ks),
                              ctypes.byref(opt), ws.data_ptr(), ws.numel(), sptr)
    if st != _lib.IMF_OK:
        raise RuntimeError(f"imf_filter_bracket failed: {_lib.strerror(st)}")
    st = L.imf_workspace_status(ws.data_ptr(), sptr)
    if st == _lib.IMF_ERR_DEFECT:
        raise ScanDefectError("segment scan exhausted while solving tile; "
                              "pivot/count state was inconsistent")
    del keep
    return outs
