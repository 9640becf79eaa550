"""Build libgeer_b200.so in-tree with nvcc for sm_100a (no JIT, no torch C++ ABI).

    python -m paper_2505_24053_b200.build [--force]

Each translation unit is compiled separately so the fp64 geometry kernels can
use -fmad=false (no fp64 contraction: association decisions round exactly like
the reference's numpy expressions) while the raster keeps FMA contraction
explicit through intrinsics.  The shared object links cudart statically and is
loaded with ctypes by ``paper_2505_24053_b200._lib``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libgeer_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr",
          "-I", INCLUDE, "-I", CSRC, "-Xptxas", "-warn-spills"]
UNITS = {
    "geer_geometry.cu": ["-fmad=false"],
    "geer_raster.cu": [],
    "geer_sort.cu": [],
    "geer_api.cu": [],
    "geer_train.cu": [],
    "geer_loss.cu": [],
    "geer_camera.cu": ["-fmad=false"],
    "geer_check.cu": ["-fmad=false"],
    "geer_bin.cu": [],
    "geer_host.cu": [],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (set NVCC)")


def _deps_mtime() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "geer.h"), __file__]
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, extra: list[str], verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    defs = os.environ.get("GEER_NVCC_DEFS", "").split()  # tuning experiments, e.g. -DFWD_MIN_BLOCKS=2
    cmd = [nvcc(), *ARCH, *COMMON, *defs, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    if res.stderr.strip() and verbose:
        print(res.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA unit for sm_100a and link libgeer_b200.so; returns its path."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as pool:
        objs = list(pool.map(lambda kv: _compile(kv[0], kv[1], verbose), UNITS.items()))
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose=True)
    print(path)
