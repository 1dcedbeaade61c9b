"""Deterministic parity cases shared by make_golden.py and the tests.

Every input is regenerated from a numpy ``default_rng`` seed (same numpy
build in the build container and on the GPU box), so golden files only store
reference *outputs*: full arrays for small cases (golden_small.npz) and
SHA-256 digests for the BASELINE configurations (golden.json).

Input recipes follow SURVEY.md section 8(d) (c1..c5) and the reference's
acceptance suite (test_acceptance.py:37-59 exactness images).
"""

from __future__ import annotations

import hashlib

import numpy as np

# --------------------------------------------------------------- generators


def baseline_input(name: str, index: int = 0) -> np.ndarray:
    """BASELINE.json configs c1..c5."""
    if name == "c1":
        return np.random.default_rng(1).integers(0, 256, (512, 512), dtype=np.uint8)
    if name == "c2":
        return np.random.default_rng(2).integers(0, 65536, (2160, 3840, 3), dtype=np.uint16)
    if name == "c3":
        return np.random.default_rng(3).standard_normal((2048, 2048)).astype(np.float32)
    if name == "c4":
        return np.random.default_rng(4).integers(0, 256, (2160, 3840, 3), dtype=np.uint8)
    if name == "c5":
        return np.random.default_rng(1000 + index).integers(0, 65536, (4320, 7680),
                                                            dtype=np.uint16)
    raise KeyError(name)


C4_SHAPES = [("square", 32, 0, 0.0), ("regular_polygon", 32, 6, 0.0),
             ("regular_polygon", 32, 12, 0.0)]
C3_RADII = list(range(2, 101))


def _checkerboard_gray_border(side, border=24):
    yy, xx = np.indices((side, side))
    img = np.where((yy + xx) & 1, 255, 0).astype(np.int64)
    img[:border, :] = img[-border:, :] = 128
    img[:, :border] = img[:, -border:] = 128
    return img


def acceptance_images(side=256):
    """The 13 base images of acceptance criterion 1 (test_acceptance.py:46-51),
    drawn from the suite's fixture rng (conftest.py:21-23)."""
    rng = np.random.default_rng(0xC0FFEE)
    images = [rng.integers(0, 256, (side, side)) for _ in range(10)]
    images.append(rng.integers(0, 2, (side, side)) * 255)
    images.append(np.full((side, side), 137, dtype=np.int64))
    images.append(_checkerboard_gray_border(side))
    return images


def as_dtype(img, dtype):
    """test_acceptance.py:54-59: u16 = u8*257, f32 = (u8-128)/37."""
    dtype = np.dtype(dtype)
    if dtype == np.uint8:
        return img.astype(np.uint8)
    if dtype == np.uint16:
        return img.astype(np.uint16) * 257
    return (img.astype(np.float32) - 128.0) / 37.0


ACC_RADII = [0, 1, 2, 3, 5, 8, 16, 32, 48]
ACC_PERCENTILES = [0.0, 0.10, 0.50, 0.90, 1.0]
ACC_DTYPES = ["uint8", "uint16", "float32"]


def smooth_image(shape, dtype, seed):
    """Refine-stress distribution: smooth field + N(0, 0.03)."""
    rng = np.random.default_rng(seed)
    h, w = shape[:2]
    yy, xx = np.indices((h, w), dtype=np.float64)
    f = 0.25 * (np.sin(xx / 23.0) + np.cos(yy / 31.0)) + 0.5
    f = f + rng.normal(0.0, 0.03, (h, w))
    f = np.clip(f, 0.0, 1.0)
    if len(shape) == 3:
        f = np.stack([np.roll(f, 7 * c, axis=1) for c in range(shape[2])], axis=-1)
    dtype = np.dtype(dtype)
    if dtype == np.uint8:
        return np.round(f * 255).astype(np.uint8)
    if dtype == np.uint16:
        return np.round(f * 65535).astype(np.uint16)
    return f.astype(np.float32)


def special_floats(shape, seed):
    """f32 noise with planted -0.0/+0.0, +-inf, denormals and extremes."""
    rng = np.random.default_rng(seed)
    img = (rng.standard_normal(shape) * np.exp(rng.uniform(-8, 8, shape))).astype(np.float32)
    flat = img.reshape(-1)
    specials = np.array([-0.0, 0.0, np.inf, -np.inf, 1e-45, -1e-45, 1e-40, -3.4e38, 3.4e38],
                        dtype=np.float32)
    idx = rng.choice(flat.size, size=flat.size // 4, replace=False)
    flat[idx] = specials[rng.integers(0, specials.size, idx.size)]
    return img


def small_input(kind, shape, dtype, seed):
    dtype = np.dtype(dtype)
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        if dtype == np.float32:
            return rng.standard_normal(shape).astype(np.float32)
        hi = 256 if dtype == np.uint8 else 65536
        return rng.integers(0, hi, shape).astype(dtype)
    if kind == "lowent":  # heavy ties
        vals = rng.integers(0, 4, shape)
        return as_dtype(vals * 60, dtype)
    if kind == "smooth":
        return smooth_image(shape, dtype, seed)
    if kind == "special":
        return special_floats(shape, seed)
    if kind == "constant":
        return as_dtype(np.full(shape, 137), dtype)
    if kind == "binary":
        return as_dtype(rng.integers(0, 2, shape) * 255, dtype)
    if kind == "checker":
        side = shape[0]
        return as_dtype(_checkerboard_gray_border(side, border=max(1, side // 10)), dtype)
    raise KeyError(kind)


def _spec(kind, r, sides=0, rot=0.0):
    return (kind, r, sides, rot)


def small_cases():
    """(name, input-recipe, params) for the full-array golden fixtures."""
    cases = []
    sizes = [(67, 93), (130, 77)]
    for dt in ACC_DTYPES:
        for kind in ("uniform", "lowent", "smooth"):
            for r in (1, 4, 9, 20):
                for bnd in ("replicate", "valid"):
                    shape = sizes[(r + len(kind)) % 2]
                    cases.append((f"{dt}_{kind}_r{r}_{bnd}", (kind, shape, dt, 11 + r),
                                  dict(shape=_spec("circle", r), percentile=0.5, boundary=bnd)))
        cases.append((f"{dt}_p10_r7", ("uniform", (64, 64), dt, 3),
                      dict(shape=_spec("circle", 7), percentile=0.1, boundary="replicate")))
        cases.append((f"{dt}_p90_r7", ("uniform", (64, 64), dt, 4),
                      dict(shape=_spec("circle", 7), percentile=0.9, boundary="replicate")))
        cases.append((f"{dt}_rgb_r5", ("uniform", (48, 40, 3), dt, 5),
                      dict(shape=_spec("circle", 5), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_c1ch_r3", ("uniform", (33, 29, 1), dt, 6),
                      dict(shape=_spec("circle", 3), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_c4ch_r2", ("uniform", (21, 26, 4), dt, 7),
                      dict(shape=_spec("circle", 2), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_tiny_r6", ("uniform", (3, 5), dt, 8),
                      dict(shape=_spec("circle", 6), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_1x1_r4", ("uniform", (1, 1), dt, 9),
                      dict(shape=_spec("circle", 4), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_valid_min", ("uniform", (13, 13), dt, 10),
                      dict(shape=_spec("circle", 6), percentile=0.5, boundary="valid")))
        cases.append((f"{dt}_r0", ("uniform", (40, 50), dt, 12),
                      dict(shape=_spec("circle", 0), percentile=0.5, boundary="replicate")))
        for shp in [_spec("square", 6), _spec("regular_polygon", 9, 6, 0.0),
                    _spec("regular_polygon", 9, 12, 0.0), _spec("regular_polygon", 11, 3, 90.0),
                    _spec("regular_polygon", 12, 12, 7.5), _spec("regular_polygon", 6, 5, 10.0)]:
            cases.append((f"{dt}_{shp[0]}{shp[2]}_r{shp[1]}", ("uniform", (70, 66), dt, 13),
                          dict(shape=shp, percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_checker_r9", ("checker", (100, 100), dt, 0),
                      dict(shape=_spec("circle", 9), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_binary_r6", ("binary", (90, 70), dt, 14),
                      dict(shape=_spec("circle", 6), percentile=0.3, boundary="replicate")))
        cases.append((f"{dt}_const_r12", ("constant", (80, 60), dt, 0),
                      dict(shape=_spec("circle", 12), percentile=0.5, boundary="replicate")))
        cases.append((f"{dt}_pmap_r7", ("uniform", (70, 90), dt, 15),
                      dict(shape=_spec("circle", 7), percentile=("pmap", 16), boundary="replicate")))
        cases.append((f"{dt}_pmap_valid_r5", ("uniform", (50, 61), dt, 17),
                      dict(shape=_spec("circle", 5), percentile=("pmap", 18), boundary="valid")))
    cases.append(("float32_special_r4", ("special", (60, 70), "float32", 21),
                  dict(shape=_spec("circle", 4), percentile=0.5, boundary="replicate")))
    cases.append(("float32_special_r13_p0", ("special", (60, 70), "float32", 22),
                  dict(shape=_spec("circle", 13), percentile=0.0, boundary="replicate")))
    cases.append(("float32_special_r13_p1", ("special", (60, 70), "float32", 23),
                  dict(shape=_spec("circle", 13), percentile=1.0, boundary="replicate")))
    # large radii on small images (tile geometry edge: T = 256 - 2r)
    for r, dt in ((100, "float32"), (124, "uint16"), (90, "uint8"), (70, "float32")):
        cases.append((f"{dt}_big_r{r}", ("uniform", (150, 170), dt, 30 + r),
                      dict(shape=_spec("circle", r), percentile=0.5, boundary="replicate")))
    return cases


def make_input(recipe):
    kind, shape, dt, seed = recipe
    return small_input(kind, tuple(shape), dt, seed)


def resolve_percentile(p, out_shape):
    if isinstance(p, tuple) and p[0] == "pmap":
        return np.random.default_rng(p[1]).uniform(0.0, 1.0, out_shape)
    return p


def out_shape_of(img_shape, r, boundary):
    h, w = img_shape[:2]
    return (h - 2 * r, w - 2 * r) if boundary == "valid" else (h, w)


def digest(arr: np.ndarray) -> str:
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(f"{arr.dtype.str}{arr.shape}".encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def kernel_digest(k) -> str:
    h = hashlib.sha256()
    for f in ("off_dx", "off_dy", "row_dy", "row_xlo", "row_xhi", "col_dx", "col_ytop", "col_ybot"):
        h.update(np.ascontiguousarray(getattr(k, f), dtype=np.int32).tobytes())
        h.update(b"|")
    h.update(str(int(k.area)).encode())
    return h.hexdigest()


def kernel_specs():
    specs = [_spec("circle", r) for r in range(0, 125)]
    specs += [_spec("square", r) for r in (0, 1, 2, 4, 6, 17, 32, 64, 124)]
    for n in (3, 5, 6, 8, 12, 64):
        for r in (0, 1, 2, 6, 9, 11, 12, 16, 32, 48):
            for rot in (0.0, 7.5, 10.0, 90.0):
                specs.append(_spec("regular_polygon", r, n, rot))
    specs += [_spec("regular_polygon", 100, 12, 0.0)]
    return specs
