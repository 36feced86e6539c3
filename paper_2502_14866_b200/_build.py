"""Build the in-tree C-ABI library ``libsparsekv_b200.so`` for sm_100a.

Each ``csrc/*.cu`` is compiled with nvcc in parallel (only when it or a
header changed), then linked with ``nvcc -shared`` (static cudart, so the
library does not depend on torch's CUDA runtime build).  The resulting .so
lives next to this file; it is git-ignored but travels to the GPU box with
the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", os.environ.get("SK_OBJ_DIR", "obj"))
LIB = os.environ.get("SK_LIB_OUT") or os.path.join(PKG, "libsparsekv_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + os.environ.get("SK_NVCC_EXTRA", "").split()


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; the sparsekv-b200 library needs the CUDA 12.9 toolkit")
    return path


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _deps_mtime()):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{res.stderr[-4000:]}")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile every kernel for sm_100a and link the shared library."""
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    # A/B experiments: SK_SRC_OVERRIDE="prefill.cu=/path/alt.cu,..." swaps sources
    for pair in filter(None, os.environ.get("SK_SRC_OVERRIDE", "").split(",")):
        name, alt = pair.split("=")
        sources = [alt if os.path.basename(x) == name else x for x in sources]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), sources))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + ".tmp"
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
        os.replace(tmp, LIB)
    if verbose:
        print(f"[sparsekv-b200] built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force=bool(os.environ.get("SK_FORCE_BUILD")))
