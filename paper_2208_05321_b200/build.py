"""Build libfreqcache_b200.so in-tree for sm_100a (B200).

    python -m paper_2208_05321_b200.build        # or __graft_entry__.build()

Plain nvcc, no torch extension machinery: the library is a C ABI
(include/freqcache_b200.h) that the Python host package loads with ctypes.
The CUDA runtime is linked statically so the .so only needs libcuda at run time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libfreqcache_b200.so")
SOURCES = ["fc_api.cu", "fc_index.cu", "fc_rows.cu", "fc_sort.cu", "fc_backward.cu", "fc_engine.cu", "fc_reorder.cu"]
HEADERS = [os.path.join(CSRC, "fc_internal.cuh"), os.path.join(CSRC, "fc_rowutil.cuh"),
           os.path.join(CSRC, "fc_tma.cuh"),
           os.path.join(ROOT, "include", "freqcache_b200.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build freqcache_b200")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    if _stale(o, [s] + HEADERS):
        cmd = [nvcc(), *ARCH, *FLAGS, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        log = os.path.join(OBJ, src.replace(".cu", ".ptxas.txt"))
        with open(log, "w") as fh:
            fh.write(r.stderr)
        if verbose:
            print(f"[build] compiled {src}")
    return o


def build(verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
