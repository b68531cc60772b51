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
    """Compile the library (out/defines: experiment variants, e.g. out=libsem_alt.so).

    Each source compiles to its own object in parallel (build/<variant>/), then one link."""
    if not force and out == LIB and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    tag = os.path.splitext(os.path.basename(out))[0]
    odir = os.path.join(ROOT, "build", tag)
    os.makedirs(odir, exist_ok=True)
    base = [_nvcc(), *[f for f in NVCC_FLAGS if f != "-shared"], *["-D" + d for d in defines],
            "-I", os.path.join(ROOT, "include"), "-I", CSRC]

    def compile_one(src):
        obj = os.path.join(odir, src + ".o")
        cmd = [*base, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r.returncode, " ".join(cmd) + "\n" + r.stdout + r.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(r[3] for r in results)
    ok = all(r[2] == 0 for r in results)
    if ok:
        link = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC,-fopenmp",
                *[r[1] for r in results], "-o", out + ".tmp", "-lgomp", "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        log += " ".join(link) + "\n" + r.stdout + r.stderr
        ok = r.returncode == 0
    with open(os.path.join(CSRC, "build.log"), "w") as f:
        f.write(log)
    if not ok:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed (see %s)" % os.path.join(CSRC, "build.log"))
    os.replace(out + ".tmp", out)
    if verbose:
        sys.stdout.write(log)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
