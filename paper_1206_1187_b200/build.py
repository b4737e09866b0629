"""Build the sm_100a shared library in-tree (nvcc cross-compiles without a GPU).

Produces ``paper_1206_1187_b200/libbcnrand_b200.so`` from ``csrc/*.cu``:

    nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -shared ...

The library statically links the CUDA runtime so it has no loader dependency
beyond libcuda (the driver). It is git-ignored but travels to the GPU box with
the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbcnrand_b200.so")
SOURCES = ["bcn_kernels.cu", "bcn_deint_tma.cu", "bcn_quality.cu", "bcn_capi.cu"]
HEADERS = ["bcn_math.cuh", "bcn_kernels.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _inputs() -> list[str]:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "bcnrand_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libbcnrand_b200.so if any input changed; return its path.

    Serialised by a file lock: several ranks of one job (torchrun) may call
    this at once; the first rebuilds, the others find the library fresh."""
    if not force and not stale():
        return LIB
    import fcntl

    with open(LIB + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not stale():
            return LIB
        tmp = f"{LIB}.tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-O3", "-shared", "-cudart", "static",
               "-I", os.path.join(ROOT, "include"),
               "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
