"""Build libzinc.so in-tree with nvcc for sm_100a (static cudart, -lineinfo).

Each translation unit compiles to an object in parallel; the objects link into
one shared library.  Rebuilds only when a source or header is newer than the
library."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("ZINC_BUILD_OUT", os.path.join(HERE, "libzinc.so"))
OBJDIR = os.environ.get("ZINC_BUILD_DIR", os.path.join(HERE, "build"))
SOURCES = ["api.cu", "k_stream.cu", "k_vanilla.cu", "k_ntt.cu", "k_fft.cu", "k_split.cu", "k_small.cu"]
HEADERS = ["common.cuh", "ntt.cuh", "fft.cuh", "kernels.h", "kcommon.cuh", "zinc_coeff.cuh", "encode_real.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O2", *os.environ.get("ZINC_DEFS", "").split()]
LFLAGS = [*ARCH, "-shared", "-cudart", "static"]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, d) for d in SOURCES + HEADERS] + [os.path.join(HERE, "..", "include", "zinc.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, src.replace(".cu", ".o"))
    cmd = [NVCC, *CFLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        print(" ".join(cmd), file=sys.stderr, flush=True)
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    os.makedirs(OBJDIR, exist_ok=True)
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC, *LFLAGS, *objs, "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr, flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
