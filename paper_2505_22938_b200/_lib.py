"""ctypes binding of the C ABI declared in include/isomedian_b200.h.

The extension is loaded from the package directory (built in-tree by
``paper_2505_22938_b200.build``).  There is no fallback: if the shared library
is missing or CUDA is unavailable, :func:`lib` raises and the filter fails
loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IMF_LIB") or os.path.join(_HERE, "libisomedian_b200.so")

IMF_OK = 0
IMF_ERR_INVALID = 1
IMF_ERR_CUDA = 2
IMF_ERR_DEFECT = 3
IMF_ERR_WORKSPACE = 4
IMF_ERR_UNSUPPORTED = 5

EXPORTED = ("imf_workspace_size", "imf_filter", "imf_filter_bracket", "imf_workspace_status",
            "imf_filter_host",
            "imf_strerror", "imf_version", "imf_last_error", "imf_launch_count",
            "imf_profile_last", "imf_int_peak", "imf_last_features", "imf_tile_omega", "imf_plan_info")

_i32p = ctypes.POINTER(ctypes.c_int32)


class ImfKernel(ctypes.Structure):
    _fields_ = [("shape_code", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("area", ctypes.c_int32), ("nrows", ctypes.c_int32),
                ("row_dy", ctypes.c_void_p), ("row_xlo", ctypes.c_void_p),
                ("row_xhi", ctypes.c_void_p), ("ncols", ctypes.c_int32),
                ("col_dx", ctypes.c_void_p), ("col_ytop", ctypes.c_void_p),
                ("col_ybot", ctypes.c_void_p)]


class ImfImage(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("stride_b", ctypes.c_int64), ("stride_y", ctypes.c_int64),
                ("stride_x", ctypes.c_int64), ("stride_c", ctypes.c_int64)]


class ImfOptions(ctypes.Structure):
    _fields_ = [("boundary", ctypes.c_int32), ("tile_size", ctypes.c_int32),
                ("seed_rows", ctypes.c_int32), ("seeds_per_row", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("row_begin", ctypes.c_int32),
                ("row_end", ctypes.c_int32), ("reserved", ctypes.c_int32)]

IMF_FLAG_PROFILE = 1
IMF_FEATURE_K1_TMA = 1


_lock = threading.Lock()
_LIB = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare its signatures (no CUDA work)."""
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.imf_workspace_size.argtypes = [P(ImfImage), P(ImfKernel), P(ImfOptions)]
    lib.imf_workspace_size.restype = ctypes.c_size_t
    lib.imf_filter.argtypes = [P(ImfImage), P(ImfImage), P(ImfKernel), ctypes.c_int32,
                               ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, P(ImfOptions),
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.imf_filter.restype = ctypes.c_int
    lib.imf_filter_bracket.argtypes = [P(ImfImage), P(ImfImage), ctypes.c_int32, ctypes.c_void_p,
                                       P(ImfKernel), P(ImfOptions), ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p]
    lib.imf_filter_bracket.restype = ctypes.c_int
    lib.imf_workspace_status.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.imf_workspace_status.restype = ctypes.c_int
    lib.imf_filter_host.argtypes = [P(ImfImage), P(ImfImage), P(ImfKernel), ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                    P(ImfOptions), ctypes.c_void_p]
    lib.imf_filter_host.restype = ctypes.c_int
    lib.imf_strerror.argtypes = [ctypes.c_int]
    lib.imf_strerror.restype = ctypes.c_char_p
    lib.imf_version.argtypes = []
    lib.imf_version.restype = ctypes.c_int
    lib.imf_last_error.argtypes = []
    lib.imf_last_error.restype = ctypes.c_char_p
    lib.imf_launch_count.argtypes = []
    lib.imf_launch_count.restype = ctypes.c_uint64
    lib.imf_profile_last.argtypes = [P(ctypes.c_float), P(ctypes.c_float), P(ctypes.c_int32),
                                     P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_int32)]
    lib.imf_profile_last.restype = ctypes.c_int
    lib.imf_int_peak.argtypes = [P(ctypes.c_double), P(ctypes.c_double)]
    lib.imf_int_peak.restype = ctypes.c_int
    lib.imf_last_features.argtypes = []
    lib.imf_last_features.restype = ctypes.c_uint32
    lib.imf_tile_omega.argtypes = [P(ImfImage), P(ImfKernel), P(ImfOptions), ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_void_p]
    lib.imf_tile_omega.restype = ctypes.c_int
    lib.imf_plan_info.argtypes = [P(ImfImage), P(ImfKernel), P(ImfOptions), ctypes.c_void_p]
    lib.imf_plan_info.restype = ctypes.c_int
    return lib


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        with _lock:
            if _LIB is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"CUDA extension {LIB_PATH} is not built; run "
                        "`python -m paper_2505_22938_b200.build` (there is no CPU fallback)")
                _LIB = load(LIB_PATH)
    return _LIB


def strerror(code: int) -> str:
    msg = lib().imf_strerror(code).decode()
    if code == IMF_ERR_CUDA:
        msg += " (" + lib().imf_last_error().decode() + ")"
    return msg
