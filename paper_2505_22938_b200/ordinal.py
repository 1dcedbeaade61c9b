"""Device-side ordinal transform of one tile (K1), for inspection and tests.

The reference computes, per tile, the ordinal transform (``ordinal.py:126-172``):
ranks of every pixel, the omnigram (rank -> position) and the sorted values.
The B200 engine computes the same thing inside K1 and never materializes it
on the host; :func:`tile_ordinal` runs K1 on ONE tile of a filter call through
``imf_tile_omega`` and returns the reference's ``OrdinalTile`` fields, so the
reference's invariants (``tests/test_ordinal.py:33-63``: permutation, mutual
inverse, sorted reverse map consistent with the source) can be checked on the
device's own output.

Differences from the reference, both output-neutral for the filter: ties are
ranked in arbitrary order (the reference breaks them row-major; only its
tile-to-tile forwarding needs that, ``oracle.py:8-13``), and only the tile's
footprint is ranked when the planner uses one (the reference's optional
``footprint_mask``, ``tiling.py:148-162``) -- unranked pixels get rank -1, as
masked pixels do in the reference (``test_ordinal.py:76-82``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import make_kernel


@dataclass
class DeviceOrdinalTile:
    """Reference ``OrdinalTile`` fields (ordinal.py:37-59) of one device tile."""

    ranks: np.ndarray      # (Sh, Sw) int32, -1 where unranked
    pos_x: np.ndarray      # (N,) int32
    pos_y: np.ndarray      # (N,) int32
    values: np.ndarray     # (N,) ascending, the image dtype
    count: int
    x0: int                # image column of input-tile column 0 (before clamping)
    y0: int                # image row of input-tile row 0 (before clamping)
    channel: int
    image: int
    footprint: bool

    @property
    def packed_positions(self) -> np.ndarray:
        """Omega packed x | y << 8 (ordinal.py:56-59)."""
        return (self.pos_x | (self.pos_y << 8)).astype(np.uint16)

    def tile_values(self, img2d: np.ndarray) -> np.ndarray:
        """The (Sh, Sw) input tile this transform ranked, read from one plane of
        the image with the replicate clamp (tiling.py:134-140)."""
        h, w = self.ranks.shape
        ys = np.clip(self.y0 + np.arange(h), 0, img2d.shape[0] - 1)
        xs = np.clip(self.x0 + np.arange(w), 0, img2d.shape[1] - 1)
        return img2d[np.ix_(ys, xs)]


def tile_ordinal(image, params, tile: int, *, batched: bool = False) -> DeviceOrdinalTile:
    """Run the filter call's K1 on tile `tile` (channel fastest, then tile
    column, tile row, image) of a CUDA tensor and return its ordinal transform."""
    import torch

    from .tiling import _DTYPES, _WS, _image_struct, _kernel_struct, _np_dtype_of

    if not (isinstance(image, torch.Tensor) and image.is_cuda):
        raise ValueError("tile_ordinal expects a CUDA tensor")
    L = _lib.lib()
    dt = _np_dtype_of(image)
    kernel = make_kernel(params.shape)
    ks, keep = _kernel_struct(kernel)
    has_c = image.dim() == (4 if batched else 3)
    simg = _image_struct(image, _DTYPES[dt], batched, has_c)
    opt = _lib.ImfOptions(1 if params.boundary == "valid" else 0, int(params.tile_size or 0), 0, 0)
    with torch.cuda.device(image.device):
        stream = torch.cuda.current_stream(image.device)
        need = L.imf_workspace_size(ctypes.byref(simg), ctypes.byref(ks), ctypes.byref(opt))
        if need == 0:
            raise ValueError("unsupported filter geometry for the CUDA engine")
        ws = _WS.get(image.device, need, stream)
        om = np.empty(65536, np.uint16)
        info = np.zeros(8, np.int32)
        st = L.imf_tile_omega(ctypes.byref(simg), ctypes.byref(ks), ctypes.byref(opt), int(tile),
                              om.ctypes.data, om.size, info.ctypes.data, ws.data_ptr(), ws.numel(),
                              ctypes.c_void_p(stream.cuda_stream))
    del keep
    if st != _lib.IMF_OK:
        raise RuntimeError(f"imf_tile_omega failed: {_lib.strerror(st)}")
    n, x0, y0, sw, sh, c, b, fp = (int(v) for v in info)
    om = om[:n]
    px = (om & 0xff).astype(np.int32)
    py = (om >> 8).astype(np.int32)
    ranks = np.full((sh, sw), -1, np.int32)
    ranks[py, px] = np.arange(n, dtype=np.int32)
    host = image.detach().cpu().numpy()
    plane = host[b] if batched else host
    plane = plane[..., c] if has_c else plane
    ys = np.clip(y0 + py, 0, plane.shape[0] - 1)
    xs = np.clip(x0 + px, 0, plane.shape[1] - 1)
    return DeviceOrdinalTile(ranks=ranks, pos_x=px, pos_y=py, values=plane[ys, xs], count=n,
                             x0=x0, y0=y0, channel=c, image=b, footprint=bool(fp))
