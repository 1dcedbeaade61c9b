"""The boundary from plain C (no Python, no torch): examples/c_abi_demo.c is
compiled against include/isomedian_b200.h and the in-tree library.  On the
host it plans a call (imf_workspace_size / imf_plan_info, no CUDA work); on a
GPU it filters through imf_filter_host (host buffers) and through imf_filter
(device buffers, caller-owned workspace, a stream) and checks every pixel
against a brute-force median written in the same C file."""
import os
import shutil
import subprocess

import pytest

from paper_2505_22938_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


CUDA = "/usr/local/cuda"


def _build(tmp_path, cudart=False):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = str(tmp_path / ("c_abi_demo_rt" if cudart else "c_abi_demo"))
    extra = ["-DWITH_CUDART", "-I", f"{CUDA}/include", "-L", f"{CUDA}/lib64", "-lcudart",
             f"-Wl,-rpath,{CUDA}/lib64"] if cudart else []
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", libdir, "-lisomedian_b200",
                    f"-Wl,-rpath,{libdir}", *extra, "-lm", "-o", exe], check=True)
    return exe


def test_c_caller_links_and_plans(tmp_path):
    out = subprocess.run([_build(tmp_path), "--plan"], capture_output=True, text=True, check=True).stdout
    assert "plan: status 0" in out


@pytest.mark.gpu
def test_c_caller_filters_bit_exact(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, check=True).stdout
    assert " 0 mismatches vs brute force" in out


@pytest.mark.gpu
def test_c_caller_device_entry_bit_exact(tmp_path):
    if not os.path.exists(f"{CUDA}/include/cuda_runtime.h"):
        pytest.skip("no CUDA headers")
    out = subprocess.run([_build(tmp_path, cudart=True), "--device"], capture_output=True, text=True,
                         check=True).stdout
    assert " 0 mismatches vs brute force" in out
