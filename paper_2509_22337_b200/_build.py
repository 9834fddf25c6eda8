"""In-tree build of the native library (``_lib/libhbp.so``) for sm_100a.

Plain nvcc, no build system: the library is a handful of translation units.
The fp64 translation unit is compiled with ``-fmad=false`` (bitwise contract,
see csrc/lbp_kernels.cuh) and ``-lineinfo`` so ncu's source page maps back.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libhbp.so")

SOURCES = ["engine.cu", "sweep.cu", "layout_dev.cu", "layout.cpp", "compiler.cpp", "capi.cpp"]
HEADERS = ["internal.h", "device.h", "lbp_kernels.cuh", "lbp_node.inc", os.path.join("..", "..", "include", "hornbp_gpu.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for name in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, name)) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libhbp.so")
    if verbose:
        sys.stderr.write(proc.stderr)
    with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as fh:
        fh.write(proc.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
