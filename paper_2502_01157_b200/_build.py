"""In-tree build of librfb.so (sm_100a) and the CPU oracle.

``build_extension()`` compiles ``csrc/rfb.cu`` with nvcc for
``-gencode arch=compute_100a,code=sm_100a``.  The walk's bit-exactness needs
``-fmad=false`` (no FMA contraction, like numba's fastmath=False); the one
place that needs FMA (camera rays, to reproduce numpy's matmul) uses
explicit ``__fma_rn``.
"""

from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librfb.so")
CU_FILES = [os.path.join(CSRC, f) for f in ("rfb.cu", "rfb_adjacency.cu", "rfb_segments.cu")]
SOURCES = CU_FILES + [os.path.join(CSRC, "rfb_device.cuh")] + [
    os.path.join(REPO, "include", "rfb.h")
]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_extension(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(LIB, SOURCES):
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *CU_FILES]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_oracle(force: bool = False) -> str:
    odir = os.path.join(REPO, "oracle")
    target = os.path.join(odir, "liboracle.so")
    if force or _stale(target, [os.path.join(odir, "rfoam_oracle.c"), os.path.join(odir, "Makefile")]):
        subprocess.run(["make", "-C", odir, "-B" if force else "liboracle.so"], check=True)
    return target
