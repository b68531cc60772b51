"""Build libsem.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2104_08416_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsem.so")
SOURCES = ["api.cu", "reorder.cu", "step.cu", "heun.cu", "chunks_gpu.cu", "partition_gpu.cu", "chunks.cpp", "partition.cpp", "refelem.cpp"]
HEADERS = ["kernels.h", "sem_internal.h", "dev_common.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off",
    "-shared",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sem.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile the library (out/defines: experiment variants, e.g. out=libsem_alt.so)."""
    if not force and out == LIB and not stale():
        return LIB
    cmd = [_nvcc(), *NVCC_FLAGS, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, f) for f in SOURCES], "-o", out + ".tmp", "-lgomp", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(CSRC, "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed (see %s)" % os.path.join(CSRC, "build.log"))
    os.replace(out + ".tmp", out)
    if verbose:
        sys.stdout.write(log)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
