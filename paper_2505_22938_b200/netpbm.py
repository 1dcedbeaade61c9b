"""Netpbm image files either side of the filter: P5/P6 (8/16-bit) and Pf/PF.

Same formats and conventions as the reference's reader/writer
(/root/reference/pkg/src/isomedian/netpbm.py:1-86):

* P5 (gray) / P6 (RGB) with maxval 255 (uint8) or 65535 (uint16, big-endian
  samples on disk);
* Pf (gray) / PF (RGB) float32, rows stored bottom-to-top, the sign of the
  scale field giving the byte order (negative = little-endian); written as
  little-endian with scale -1.0;
* header tokens separated by whitespace, ``#`` comments skipped;
* errors are ``ValueError`` naming the problem ("magic", "maxval", "dtype",
  "truncated").

``read_image(path, pinned=True)`` reads the samples straight into page-locked
host memory (a pinned torch tensor's storage), so the C-ABI host entry
(``imf_filter_host``) can stream them to the GPU at full copy bandwidth.
"""

from __future__ import annotations

import os

import numpy as np

_WS = b" \t\n\r\v\f"


def _header(f, ntok: int) -> list[bytes]:
    """Read `ntok` header tokens after the magic, skipping comments; the file is
    left positioned at the first sample byte (one whitespace byte after the
    last token, as the format requires)."""
    toks: list[bytes] = []
    cur = bytearray()
    while True:
        ch = f.read(1)
        if not ch:
            raise ValueError("truncated image header")
        if ch == b"#" and not cur:
            while ch not in (b"\n", b"\r", b""):
                ch = f.read(1)
            continue
        if ch in _WS:
            if cur:
                toks.append(bytes(cur))
                cur = bytearray()
                if len(toks) == ntok:
                    return toks
            continue
        cur += ch


def _alloc(shape, dtype, pinned: bool):
    if pinned:
        import torch
        pinned = torch.cuda.is_available()
    if not pinned:
        return np.empty(shape, dtype=dtype)
    import torch
    tdt = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.uint16,
           np.dtype(np.float32): torch.float32}[np.dtype(dtype)]
    return torch.empty(shape, dtype=tdt).pin_memory().numpy()


def read_image(path, pinned: bool = False) -> np.ndarray:
    """Read a PGM/PPM/PFM file into an (H, W) or (H, W, 3) native-endian array."""
    with open(path, "rb") as f:
        magic = f.read(2)
        if magic in (b"P5", b"P6"):
            w, h, maxval = (int(t) for t in _header(f, 3))
            if maxval not in (255, 65535):
                raise ValueError(f"unsupported maxval {maxval} (want 255 or 65535)")
            c = 3 if magic == b"P6" else 1
            dt = np.uint16 if maxval == 65535 else np.uint8
            shape = (h, w, c) if c == 3 else (h, w)
            img = _alloc(shape, dt, pinned)
            buf = memoryview(img.reshape(-1).view(np.uint8))
            if f.readinto(buf) != buf.nbytes:
                raise ValueError("truncated image data")
            if dt == np.uint16:
                img.byteswap(inplace=True)  # big-endian on disk
            return img
        if magic in (b"Pf", b"PF"):
            w, h = (int(t) for t in _header(f, 2))
            scale = float(_header(f, 1)[0])
            c = 3 if magic == b"PF" else 1
            shape = (h, w, c) if c == 3 else (h, w)
            raw = np.empty(shape, dtype=np.float32)
            buf = memoryview(raw.reshape(-1).view(np.uint8))
            if f.readinto(buf) != buf.nbytes:
                raise ValueError("truncated image data")
            if scale > 0:  # big-endian samples
                raw.byteswap(inplace=True)
            img = _alloc(shape, np.float32, pinned)
            img[...] = raw[::-1]  # rows bottom-to-top on disk
            return img
        raise ValueError(f"unsupported image magic {magic!r} (want P5, P6, Pf, or PF)")


def write_image(path, image) -> None:
    """Write PGM (integer gray), PPM (integer RGB) or PFM (float32)."""
    if hasattr(image, "detach"):
        image = image.detach().cpu().numpy()
    a = np.asarray(image)
    if a.ndim == 3 and a.shape[2] == 1:
        a = a[:, :, 0]
    if a.ndim not in (2, 3) or (a.ndim == 3 and a.shape[2] != 3):
        raise ValueError("image must be (H, W) or (H, W, 3)")
    h, w = a.shape[:2]
    rgb = a.ndim == 3
    if a.dtype == np.float32:
        head = (b"PF" if rgb else b"Pf") + f"\n{w} {h}\n-1.0\n".encode()
        body = np.ascontiguousarray(a[::-1], dtype="<f4")
    elif a.dtype == np.uint8:
        head = (b"P6" if rgb else b"P5") + f"\n{w} {h}\n255\n".encode()
        body = np.ascontiguousarray(a)
    elif a.dtype == np.uint16:
        head = (b"P6" if rgb else b"P5") + f"\n{w} {h}\n65535\n".encode()
        body = np.ascontiguousarray(a, dtype=">u2")
    else:
        raise ValueError(f"unsupported image dtype {a.dtype}")
    with open(os.fspath(path), "wb") as f:
        f.write(head)
        f.write(memoryview(body.reshape(-1).view(np.uint8)))
