"""Build the in-tree CUDA extension libisomedian_b200.so for sm_100a.

    python -m paper_2505_22938_b200.build [-v] [--force]

Plain nvcc (no torch JIT cache): every kernel source is compiled to its own
object in parallel (only host launch stubs cross translation units, so no
-rdc), objects are rebuilt when their source or a header changed, and the
shared library lands next to this file so it travels with the repository
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libisomedian_b200.so")
SOURCES = ["imf_sort.cu", "imf_count.cu", "imf_pair.cu", "imf_select.cu", "imf_direct.cu", "imf_api.cu", "imf_peak.cu"]
HEADERS = ["imf_common.cuh", "imf_kernels.cuh", "imf_k1.cuh", os.path.join("..", "..", "include", "isomedian_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    # template kernels are instantiated in their own TU and launched from imf_api.cu
    "-static-global-template-stub=false",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJ, src.replace(".cu", ".o"))


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _stale_obj(src: str, hdr_t: float) -> bool:
    o = _obj(src)
    return not os.path.exists(o) or max(_mtime(os.path.join(CSRC, src)), hdr_t) > _mtime(o)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    hdr_t = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    t = _mtime(LIB)
    return any(_stale_obj(s, hdr_t) or _mtime(os.path.join(CSRC, s)) > t for s in SOURCES)


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    todo = [s for s in SOURCES if force or _stale_obj(s, hdr_t)]

    def compile_one(src: str) -> None:
        cmd = [nvcc(), *NVCC_FLAGS, "-c", os.path.join(CSRC, src), "-o", _obj(src) + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(_obj(src) + ".tmp", _obj(src))

    with ThreadPoolExecutor(max_workers=len(todo) or 1) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", "-o", LIB + ".tmp", *[_obj(s) for s in SOURCES], "-lcudart"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="--force" in sys.argv)
    print(LIB)
