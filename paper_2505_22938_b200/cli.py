"""Command-line front end of the B200 filter: ``filter`` and ``bench``.

Mirrors the reference CLI (/root/reference/pkg/src/isomedian/cli.py:1-152):
same subcommand names, options, percent-scale percentiles, shape syntax
(``circle``, ``square``, ``poly:SIDES[:ROTATION]``), CSV bench output
(experiments.py:83-125) and exit codes (0 ok, 1 processing error, 2 usage).
The engine is the CUDA path (``--engine cuda``; ``fast`` is accepted as an
alias so reference invocations run unchanged).  The reference's ``oracle``
engine and the ``compare`` rotation study are not part of this package
(DESIGN.md section 7).

    python -m paper_2505_22938_b200.cli filter in.pgm out.pgm --radius 48
    python -m paper_2505_22938_b200.cli bench in.pgm --radii 8,16,32,48
"""

from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

from .kernels import ShapeSpec
from .netpbm import read_image, write_image
from .tiling import FilterParams

BENCH_CSV_HEADER = "radius,engine,dtype,mp,ms,mps"


def parse_shape(text: str, radius: int) -> ShapeSpec:
    """``circle`` | ``square`` | ``poly:SIDES[:ROTATION_DEG]`` (cli.py:18-31)."""
    if text in ("circle", "square"):
        return ShapeSpec(text, radius)
    if text.startswith("poly:"):
        fields = text.split(":")[1:]
        if len(fields) not in (1, 2):
            raise ValueError(f"bad shape {text!r}; want poly:SIDES[:ROTATION]")
        rot = float(fields[1]) if len(fields) == 2 else 0.0
        return ShapeSpec("regular_polygon", radius, sides=int(fields[0]), rotation_deg=rot)
    raise ValueError(f"bad shape {text!r}; want circle, square, or poly:K[:ROT]")


def _percentile(args, image):
    if args.percentile_map is None:
        if not 0.0 <= args.percentile <= 100.0:
            raise ValueError("percentile must be in [0, 100]")
        return args.percentile / 100.0
    pmap = read_image(args.percentile_map)
    if pmap.ndim != 2:
        raise ValueError("percentile map must be grayscale")
    if pmap.shape != image.shape[:2]:
        raise ValueError("percentile map dimensions must match the input")
    p = np.clip(pmap.astype(np.float64), 0.0, 100.0) / 100.0
    if args.boundary == "valid":
        r = args.radius
        p = p[r:p.shape[0] - r, r:p.shape[1] - r]
    return p


def cmd_filter(args) -> int:
    # samples land in pinned memory; imf_filter_host streams row stripes
    image = read_image(args.input, pinned=True)
    params = FilterParams(shape=parse_shape(args.shape, args.radius),
                          percentile=_percentile(args, image), boundary=args.boundary,
                          forwarding=not args.no_forwarding, tile_size=args.tile,
                          workers=args.threads)
    from .tiling import filter_image
    write_image(args.output, filter_image(image, params))
    return 0


def cmd_bench(args) -> int:
    """Best-of-N wall time per radius (experiments.py:101-125), CSV to stdout."""
    image = read_image(args.input, pinned=True)
    if image.ndim == 3:
        image = np.ascontiguousarray(image[:, :, 0])
    radii = [int(r) for r in args.radii.split(",")]
    mp = image.shape[0] * image.shape[1] / 1e6
    print(BENCH_CSV_HEADER)
    for r in radii:
        params = FilterParams(shape=ShapeSpec("circle", r), workers=args.threads)
        from .tiling import filter_image
        filter_image(image, params)  # warm-up (kernel-table caches, pools)
        best = math.inf
        for _ in range(max(1, args.repeats)):
            t0 = time.perf_counter()
            filter_image(image, params)
            best = min(best, time.perf_counter() - t0)
        print(f"{r},{args.engine},{image.dtype},{mp:.3f},{best * 1e3:.2f},{mp / best:.3f}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="isomedian-b200",
                                 description="Exact median/percentile filtering on the B200")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("filter", help="filter an image")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--radius", type=int, required=True)
    p.add_argument("--percentile", type=float, default=50.0,
                   help="selection percentile, 0..100 (default 50)")
    p.add_argument("--percentile-map", default=None,
                   help="grayscale image of per-pixel percentiles, 0..100")
    p.add_argument("--shape", default="circle", help="circle, square, or poly:SIDES[:ROTATION]")
    p.add_argument("--boundary", choices=["replicate", "valid"], default="replicate")
    p.add_argument("--tile", type=int, default=None, help="output tile size override")
    p.add_argument("--no-forwarding", action="store_true")
    p.add_argument("--engine", choices=["cuda", "fast"], default="cuda")
    p.add_argument("--threads", type=int, default=None)
    p.set_defaults(func=cmd_filter)
    p = sub.add_parser("bench", help="wall-time the CUDA engine over a radius sweep")
    p.add_argument("input")
    p.add_argument("--radii", default="2,4,8,16,32,48,64,96")
    p.add_argument("--engine", choices=["cuda", "fast"], default="cuda")
    p.add_argument("--repeats", type=int, default=3)
    p.add_argument("--threads", type=int, default=None)
    p.set_defaults(func=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (OSError, ValueError, RuntimeError) as exc:
        print(f"isomedian-b200: error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
