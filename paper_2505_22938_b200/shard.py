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

from dataclasses import dataclass

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
    out = filter_fn(sub, params)
    if params.boundary == "valid":
        return out
    off = stripe.y0 - stripe.in_y0
    return out[off:off + stripe.rows]


def assemble(stripes: list[Stripe], parts: list[np.ndarray]) -> np.ndarray:
    """Concatenate per-rank stripe outputs in row order."""
    order = sorted(range(len(stripes)), key=lambda i: stripes[i].y0)
    return np.concatenate([parts[i] for i in order], axis=0)
