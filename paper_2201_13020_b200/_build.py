"""Build libszx_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The numerics contract: no --use_fast_math, -ftz=false,
-prec-div/-prec-sqrt true, no FMA contraction of the float ops that decide stream bytes
(every such op is an explicit __f*_rn / __d*_rn intrinsic anyway).
"""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libszx_b200.so")
SOURCES = ["abi.cu", "compress.cu", "compress_v3.cu", "compress_v4.cu", "compress_v5.cu", "encode128.cu", "compress_generic.cu", "decompress.cu",
           "decompress_generic.cu", "range_validate.cu", "analysis.cu"]
HEADERS = ["szx_device.cuh", "szx_kernels.h", "k1_common.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-cudart", "static",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


STAMP = os.path.join(LIBDIR, "build.sha256")


def source_digest() -> str:
    """sha256 over every input of the library build (sources, headers, flags).  Content,
    not mtimes: a snapshot copied to another machine is not rebuilt for nothing, and an
    edited kernel is never silently ignored."""
    import hashlib

    h = hashlib.sha256()
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "szx_b200.h"))
    for d in deps:
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVCC_FLAGS + os.environ.get("SZX_NVCC_FLAGS", "").split()).encode())
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_digest()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + ".tmp"
    extra = os.environ.get("SZX_NVCC_FLAGS", "").split()  # e.g. -DSZX_STATS (profiling builds)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(source_digest() + "\n")
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write(res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
