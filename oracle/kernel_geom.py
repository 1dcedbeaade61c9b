"""Oracle-side kernel rasterization and target ranks (TEST INFRASTRUCTURE).

An independent restatement of the reference's kernel geometry, so the C
oracle does not borrow the product's ``make_kernel``:

* ``ShapeSpec`` semantics and the membership test ``contains``
  (/root/reference/pkg/src/isomedian/kernels.py:27-42, :67-78): circle
  ``4(dx^2+dy^2) <= (2r+1)^2``, square ``|dx|, |dy| <= r``, regular polygon
  ``a*dx + b*dy <= c`` for every edge half-plane;
* the polygon half-planes (kernels.py:45-64): vertices at radius ``r + 0.5``
  and angles ``radians(rotation) + 2*pi*k/n``, edge normals pointing away from
  the origin -- the same float64 operations in the same order, so the rasterized
  boundary pixels round identically;
* ``make_kernel`` (kernels.py:127-182): offsets in row-major order, per-row
  half-open spans ``[xlo, xhi)``, per-column inclusive extents;
* ``target_rank`` (kernels.py:185-192): ``floor(p * (area - 1) + 0.5)``.

Pinned by tests/test_oracle.py against the 375 span-table digests the real
reference produced (tests/golden/golden.json).  Only tests, ``smoke()`` and
bench.py's CPU legs reach this module (through ``oracle``).
"""

from __future__ import annotations

import math
from functools import lru_cache
from types import SimpleNamespace

import numpy as np

SHAPE_CODES = {"circle": 0, "square": 1, "regular_polygon": 2}  # kernels.py shape order


def polygon_planes(radius: int, sides: int, rotation_deg: float) -> np.ndarray:
    """(k, 3) half-planes (a, b, c), inside iff a*dx + b*dy <= c (kernels.py:45-64)."""
    rc = radius + 0.5
    ang = np.radians(rotation_deg) + 2.0 * np.pi * np.arange(sides + 1) / sides
    vx, vy = rc * np.cos(ang), rc * np.sin(ang)
    out = np.empty((sides, 3), dtype=np.float64)
    for i in range(sides):
        ex, ey = vx[i + 1] - vx[i], vy[i + 1] - vy[i]
        a, b = ey, -ex
        c = a * vx[i] + b * vy[i]
        if c < 0.0:
            a, b, c = -a, -b, -c
        out[i] = (a, b, c)
    return out


def _row_inside(kind: str, radius: int, planes: np.ndarray, dy: int, dx: np.ndarray) -> np.ndarray:
    """contains() (kernels.py:67-78) for one kernel row, vectorized over dx."""
    if kind == "circle":
        return 4 * (dx * dx + dy * dy) <= (2 * radius + 1) ** 2
    if kind == "square":
        return np.ones(dx.shape, dtype=bool)
    fdx, fdy = dx.astype(np.float64), float(dy)
    ok = np.ones(dx.shape, dtype=bool)
    for a, b, c in planes:
        ok &= ~((a * fdx + b * fdy) > c)  # two rounded products, one rounded add
    return ok


@lru_cache(maxsize=512)
def make_kernel(kind: str, radius: int, sides: int = 0, rotation_deg: float = 0.0) -> SimpleNamespace:
    """Rasterized kernel with the fields the C oracle reads (kernels.py:127-182)."""
    r = radius
    planes = (polygon_planes(r, sides, rotation_deg) if kind == "regular_polygon"
              else np.empty((0, 3), dtype=np.float64))
    d = np.arange(-r, r + 1, dtype=np.int64)
    grid = np.stack([_row_inside(kind, r, planes, int(dy), d) for dy in d])  # [dy + r, dx + r]
    off_dy, off_dx = np.nonzero(grid)                                       # row-major
    rows = [(int(dy), np.flatnonzero(grid[dy + r])) for dy in d]
    cols = [(int(dx), np.flatnonzero(grid[:, dx + r])) for dx in d]
    i32 = lambda a: np.asarray(a, dtype=np.int32)
    return SimpleNamespace(
        shape_code=SHAPE_CODES[kind], radius=r, lim=(2 * r + 1) ** 2, planes=planes,
        area=int(off_dx.size), off_dx=i32(off_dx - r), off_dy=i32(off_dy - r),
        row_dy=i32([dy for dy, xs in rows if xs.size]),
        row_xlo=i32([xs[0] - r for _, xs in rows if xs.size]),
        row_xhi=i32([xs[-1] - r + 1 for _, xs in rows if xs.size]),
        col_dx=i32([dx for dx, ys in cols if ys.size]),
        col_ytop=i32([ys[0] - r for _, ys in cols if ys.size]),
        col_ybot=i32([ys[-1] - r for _, ys in cols if ys.size]))


def kernel_of(shape) -> SimpleNamespace:
    """make_kernel for a ShapeSpec-like object (kind, radius, sides, rotation_deg)."""
    return make_kernel(shape.kind, int(shape.radius), int(getattr(shape, "sides", 0) or 0),
                       float(getattr(shape, "rotation_deg", 0.0) or 0.0))


def target_rank(area: int, percentile: float) -> int:
    """0-indexed selection rank (kernels.py:185-192)."""
    return min(max(math.floor(percentile * (area - 1) + 0.5), 0), area - 1)
