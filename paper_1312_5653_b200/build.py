"""Builds the sm_100a shared library ``_lib/libfetigpu.so`` in-tree with nvcc.

The library is the C-ABI of include/fetigpu.h: C++ host core + hand-written CUDA
kernels, compiled for ``-gencode arch=compute_100a,code=sm_100a`` only.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libfetigpu.so")
SOURCES = ["host_core.cpp", "host3d.cpp", "comm.cu", "fetigpu.cu", "fetigpu3d.cu"]
HEADERS = ["host_core.hpp", "comm.hpp", "common.cuh", "band.cuh", "blockthomas.cuh", "kernels.cuh", "fullspace.hpp", "host3d.hpp",
           "kernels3d.cuh"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def nccl_dirs():
    """NCCL of the torch install (nvidia-nccl wheel) when present, else the system one.

    The library must link the SAME libnccl.so.2 torch loads: both use the soname libnccl.so.2,
    so whichever is loaded first serves the other, and torch needs its own (newer) version.
    """
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")) and os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "fetigpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    nccl_inc, nccl_lib = nccl_dirs()
    cmd = [
        nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-shared", "-Xptxas", "-v" if verbose else "-O3",
        "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + nccl_inc,
        *os.environ.get("FETIGPU_NVCC_DEFINES", "").split(),  # experiment switches (-DNAME)
        *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp",
        "-L" + nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl_lib,
    ]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
