"""Generate golden parity fixtures by running the REAL reference package.

Run in the build container (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--c5 N]

It imports ``isomedian`` from /root/reference/pkg/src (read-only) and writes

* golden_small.npz  -- full reference outputs of the small cases in cases.py,
                       each cross-checked fast engine == brute oracle;
* golden.json       -- SHA-256 digests: kernel span tables (make_kernel),
                       acceptance-criterion-1 matrix (3 dtypes x 13 images x
                       9 radii x 5 percentiles at 256^2), BASELINE configs
                       c1, c2, c3 (r=2..100), c4 (square/hexagon/12-gon);
* golden_c5.json    -- digests of c5 images 0..N-1 (8K u16, r=64).

Inputs are regenerated from seeds (cases.py), so only outputs are stored.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import isomedian as R  # noqa: E402
from isomedian.oracle import reference_filter  # noqa: E402

import cases as C  # noqa: E402


def ref_params(p, out_shape=None):
    kind, r, sides, rot = p["shape"]
    perc = C.resolve_percentile(p["percentile"], out_shape)
    return R.FilterParams(shape=R.ShapeSpec(kind, r, sides, rot), percentile=perc,
                          boundary=p["boundary"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5", type=int, default=0, help="number of c5 images to digest")
    ap.add_argument("--skip-main", action="store_true")
    args = ap.parse_args()
    gold = {}
    if not args.skip_main:
        t0 = time.time()
        gold["kernels"] = {}
        for spec in C.kernel_specs():
            k = R.make_kernel(R.ShapeSpec(*spec))
            gold["kernels"][json.dumps(spec)] = C.kernel_digest(k)
        print(f"kernels {len(gold['kernels'])} in {time.time() - t0:.1f}s", flush=True)

        small = {}
        for name, recipe, p in C.small_cases():
            img = C.make_input(recipe)
            out_shape = C.out_shape_of(img.shape, p["shape"][1], p["boundary"])
            params = ref_params(p, out_shape)
            fast = R.filter_image(img, params)
            brute = reference_filter(img, params)
            assert fast.tobytes() == brute.tobytes(), name
            small[name] = fast
        np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
        print(f"small {len(small)} in {time.time() - t0:.1f}s", flush=True)

        acc = {}
        for dt in C.ACC_DTYPES:
            for idx, base in enumerate(C.acceptance_images()):
                img = C.as_dtype(base, dt)
                for r in C.ACC_RADII:
                    for p in C.ACC_PERCENTILES:
                        out = R.filter_image(img, R.FilterParams(shape=R.ShapeSpec("circle", r),
                                                                 percentile=p))
                        acc[f"{dt}/{idx}/{r}/{p}"] = C.digest(out)
        gold["acceptance"] = acc
        print(f"acceptance {len(acc)} in {time.time() - t0:.1f}s", flush=True)

        base = {}
        img = C.baseline_input("c1")
        prm = R.FilterParams(shape=R.ShapeSpec("circle", 8))
        out = R.filter_image(img, prm)
        assert out.tobytes() == reference_filter(img, prm).tobytes()
        base["c1"] = C.digest(out)
        img = C.baseline_input("c2")
        base["c2"] = C.digest(R.filter_image(img, R.FilterParams(shape=R.ShapeSpec("circle", 48))))
        print(f"c1,c2 in {time.time() - t0:.1f}s", flush=True)
        img = C.baseline_input("c3")
        for r in C.C3_RADII:
            base[f"c3/r{r}"] = C.digest(R.filter_image(img, R.FilterParams(
                shape=R.ShapeSpec("circle", r))))
        print(f"c3 in {time.time() - t0:.1f}s", flush=True)
        img = C.baseline_input("c4")
        for spec in C.C4_SHAPES:
            base[f"c4/{json.dumps(list(spec))}"] = C.digest(R.filter_image(
                img, R.FilterParams(shape=R.ShapeSpec(*spec))))
        print(f"c4 in {time.time() - t0:.1f}s", flush=True)
        gold["baseline"] = base
        gold["_meta"] = {"numpy": np.__version__, "reference": "isomedian " + R.__version__,
                         "generator": "tests/golden/make_golden.py"}
        with open(os.path.join(HERE, "golden.json"), "w") as f:
            json.dump(gold, f, indent=1, sort_keys=True)
    if args.c5:
        c5 = {}
        t0 = time.time()
        for i in range(args.c5):
            img = C.baseline_input("c5", i)
            c5[str(i)] = C.digest(R.filter_image(img, R.FilterParams(
                shape=R.ShapeSpec("circle", 64))))
            with open(os.path.join(HERE, "golden_c5.json"), "w") as f:
                json.dump(c5, f, indent=1)
            print(f"c5 image {i} at {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
