"""B200-native rank-order (circular median / percentile) filter.

A from-scratch sm_100a implementation of the hot path of Weiss, *Fast
Isotropic Median Filtering* (arXiv 2505.22938), behind the public surface of
the reference ``isomedian`` package: ``filter_image(image, FilterParams)``
with ``ShapeSpec`` kernels (circle / square / regular polygon), u8 / u16 / f32
images, replicate / valid boundaries, scalar or per-pixel percentiles.

Host prologue (validation, kernel rasterization, target ranks) in Python;
everything else in one CUDA extension behind a C ABI
(``include/isomedian_b200.h``).  No CPU fallback.
"""

from .kernels import (MAX_POLYGON_SIDES, MAX_RADIUS, KernelShape, ShapeSpec, contains,
                      make_kernel, target_rank)
from .netpbm import read_image, write_image
from .shard import filter_batch_multi, filter_multi
from .tiling import (FilterParams, ScanDefectError, Tile, TileGrid, decompose, filter_batch,
                     filter_image, filter_image_bracket, pad_image)

__all__ = [
    "KernelShape", "ShapeSpec", "contains", "make_kernel", "target_rank",
    "MAX_RADIUS", "MAX_POLYGON_SIDES",
    "FilterParams", "ScanDefectError", "Tile", "TileGrid", "decompose", "filter_image",
    "filter_batch", "filter_image_bracket", "pad_image", "float_order_key",
    "read_image", "write_image", "filter_multi", "filter_batch_multi",
]

__version__ = "0.1.0"


def float_order_key(values):
    """u32 keys that sort float32 values in IEEE total order (ordinal.py:109-123)."""
    import numpy as np

    arr = np.asarray(values, dtype="<f4")
    if np.isnan(arr).any():
        raise ValueError("float_order_key is undefined for NaN")
    u = arr.view(np.uint32)
    key = np.where(u >> 31, ~u, u | np.uint32(0x80000000))
    if np.isscalar(values) or arr.ndim == 0:
        return np.uint32(key)
    return key.astype(np.uint32)
