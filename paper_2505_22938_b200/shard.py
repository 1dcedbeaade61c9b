"""Multi-GPU partitioning of the filter: no collective on the data path.

Output pixels depend only on input within the kernel radius, so work shards
by independent units:

* a batch of images: whole images per rank (round-robin), zero halo overhead;
* one image: contiguous output-row stripes; each rank reads its input rows
  plus an r-row halo on each side from the host (clamped at the image edges,
  where the clamp *is* the reference's replicate padding, tiling.py:134-140).

Every rank filters its own unit with :func:`paper_2505_22938_b200.filter_image`
(one process per GPU, launched by torchrun); results are written into
disjoint slices of the host output.  Collectives (when a caller wants the
stripes on one rank) are plumbing outside the filter -- the bench never uses
one on the hot path.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Stripe:
    """Output rows [y0, y1) of one rank and the input rows [in_y0, in_y1) it reads."""

    rank: int
    y0: int
    y1: int
    in_y0: int
    in_y1: int

    @property
    def rows(self) -> int:
        return self.y1 - self.y0


def stripe_plan(height: int, radius: int, boundary: str, world: int) -> list[Stripe]:
    """Split the output rows of an image of `height` rows into `world` stripes.

    Stripe sizes differ by at most one row; ranks beyond the row count get
    empty stripes.  Input extents include the r-row halos (replicate mode) or
    the 2r extra rows of the valid window (valid mode).
    """
    if world < 1:
        raise ValueError("world size must be >= 1")
    out_h = height - 2 * radius if boundary == "valid" else height
    if out_h < 1:
        raise ValueError("image smaller than the kernel in valid mode")
    base, extra = divmod(out_h, world)
    plan, y = [], 0
    for rk in range(world):
        n = base + (1 if rk < extra else 0)
        y0, y1 = y, y + n
        y = y1
        if boundary == "valid":
            in_y0, in_y1 = y0, (y1 + 2 * radius) if n else y0
        else:
            in_y0, in_y1 = max(0, y0 - radius), min(height, y1 + radius) if n else y0
        plan.append(Stripe(rk, y0, y1, in_y0, in_y1))
    return plan


def image_shard(n_images: int, world: int, rank: int) -> list[int]:
    """Round-robin image indices of `rank` (whole images per GPU)."""
    return list(range(rank, n_images, world))


def filter_stripe(image: np.ndarray, params, stripe: Stripe, filter_fn=None) -> np.ndarray:
    """Filter one rank's stripe: returns its output rows [y0, y1).

    `filter_fn(image, params)` defaults to the GPU :func:`filter_image`; the
    stripe input is the image rows [in_y0, in_y1) filtered with the caller's
    boundary mode, cropped to the stripe's own rows.
    """
    if filter_fn is None:
        from .tiling import filter_image as filter_fn
    if stripe.rows == 0:
        shp = list(image.shape)
        shp[0] = 0
        if params.boundary == "valid":
            shp[1] -= 2 * params.shape.radius
        return np.empty(shp, image.dtype)
    sub = image[stripe.in_y0:stripe.in_y1]
    pct = params.percentile
    if not (np.isscalar(pct) or np.ndim(pct) == 0):
        # a per-pixel map covers the full output: give the stripe its own rows
        # (replicate: the sub-image's output rows are input rows in_y0..in_y1;
        # valid: exactly the stripe's rows)
        lo, hi = (stripe.y0, stripe.y1) if params.boundary == "valid" else (stripe.in_y0, stripe.in_y1)
        params = replace(params, percentile=np.asarray(pct)[lo:hi])
    out = filter_fn(sub, params)
    if params.boundary == "valid":
        return out
    off = stripe.y0 - stripe.in_y0
    return out[off:off + stripe.rows]


def assemble(stripes: list[Stripe], parts: list[np.ndarray]) -> np.ndarray:
    """Concatenate per-rank stripe outputs in row order."""
    order = sorted(range(len(stripes)), key=lambda i: stripes[i].y0)
    return np.concatenate([parts[i] for i in order], axis=0)


def filter_multi(images, params, devices=None, *, batched: bool = False, out=None):
    """Filter host images on several GPUs from ONE process (no collective).

    `images`: a host array (H, W[, C]), or (B, H, W[, C]) with `batched`.
    Work is split as SURVEY.md 8(e) plans it: whole images per device when the
    batch has at least as many images as devices (contiguous blocks, zero halo
    overhead), else output-row stripes of each image, each device uploading
    only the input rows its stripe reads (imf_filter_host with a row range).
    One host thread per device drives that device's streams through the C-ABI
    host entry (the GIL is released inside the call); results land in
    disjoint parts of one host output.  `devices` defaults to every visible
    GPU; a device may be listed twice (two pipelines on one GPU).
    """
    import torch

    from .tiling import _check_dtype, _validate_plane, run_host

    a = images.numpy() if isinstance(images, torch.Tensor) else np.asarray(images)
    a = np.ascontiguousarray(a)
    _check_dtype(a.dtype)
    plane = a.shape[1:3] if batched else a.shape[:2]
    kernel, (out_h, out_w) = _validate_plane(tuple(plane), a.dtype,
                                             lambda: bool(np.isnan(a).any()), params)
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = list(devices)
    if not devices:
        raise RuntimeError("filter_multi needs at least one CUDA device (no CPU fallback)")
    oshape = list(a.shape)
    hy = 1 if batched else 0
    oshape[hy], oshape[hy + 1] = out_h, out_w
    o = np.empty(oshape, dtype=a.dtype) if out is None else out
    jobs = [[] for _ in devices]  # per worker (= entry of `devices`): run_host kwargs
    nb = a.shape[0] if batched else 1
    if batched and nb >= len(devices):
        cuts = [nb * i // len(devices) for i in range(len(devices) + 1)]
        for w, (b0, b1) in enumerate(zip(cuts[:-1], cuts[1:])):
            jobs[w].append(dict(image=a[b0:b1], out=o[b0:b1], batched=True))
    else:
        for w, st in enumerate(stripe_plan(a.shape[hy], params.shape.radius, params.boundary,
                                           len(devices))):
            for b in range(nb if st.rows else 0):
                src, dst = (a[b], o[b]) if batched else (a, o)
                jobs[w].append(dict(image=src, out=dst, rows=(st.y0, st.y1)))
    errors = []

    def worker(dev, lst):
        try:
            with torch.cuda.device(dev):
                for kws in lst:
                    run_host(kws.pop("image"), params, kernel=kernel, **kws)
                torch.cuda.synchronize()
        except BaseException as e:  # re-raised in the caller
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(d, lst)) for d, lst in zip(devices, jobs) if lst]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return o


def filter_batch_multi(images, params, devices=None, *, out=None):
    """Filter a CUDA batch (B, H, W[, C]) that lives on ONE GPU using several
    GPUs (a device-resident batch is scattered to its peers over
    NVLink / NVSwitch by peer copies -- no NCCL -- filtered in place there, and
    gathered back).  Whole images per device, contiguous blocks; each device
    works on its own stream, so the copies of one device overlap the kernels of
    another.  `devices` defaults to every visible GPU; the batch's own device
    keeps the first block without copies."""
    import torch

    from .tiling import filter_batch

    if not (isinstance(images, torch.Tensor) and images.is_cuda and images.dim() >= 3):
        raise ValueError("filter_batch_multi expects a CUDA batch (B, H, W[, C])")
    home = images.device
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not devices:
        raise RuntimeError("filter_batch_multi needs at least one CUDA device")
    nb = images.shape[0]
    cuts = [nb * i // len(devices) for i in range(len(devices) + 1)]
    parts = []
    for d, b0, b1 in zip(devices, cuts[:-1], cuts[1:]):
        if b1 <= b0:
            continue
        stream = torch.cuda.Stream(device=d)
        stream.wait_stream(torch.cuda.current_stream(home))  # the batch is ready
        with torch.cuda.device(d), torch.cuda.stream(stream):
            src = images[b0:b1].to(d, non_blocking=True)   # peer copy (NVLink) when d != home
            res = filter_batch(src, params, check=True, stream=stream)
            parts.append((b0, b1, res, stream, src))
    if out is None:
        out = torch.empty_like(images) if params.boundary != "valid" else None
    chunks = []
    for b0, b1, res, stream, src in parts:
        stream.synchronize()
        chunks.append((b0, b1, res))
    if out is None:
        return torch.cat([res.to(home) for _, _, res in sorted(chunks, key=lambda c: c[0])])
    for b0, b1, res in chunks:
        out[b0:b1].copy_(res.to(home))
    return out
