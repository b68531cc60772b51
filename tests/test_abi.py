"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/sem.h declares; without a GPU it fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2104_08416_b200 import build, sem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sem.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sem_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return sem.load()


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ("sem_mesh_reorder", "sem_build_operators", "sem_step_n", "sem_read_field"):
        assert n in names


def test_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sem_[a-z_]+)\b", out))
    missing = [n for n in declared_symbols() if n not in exported]
    assert not missing, missing
    assert set(sem.EXPORTED) <= exported
    # no POSIX-semaphore names are interposed by this library
    for posix in ("sem_destroy", "sem_init", "sem_open", "sem_close", "sem_post", "sem_wait"):
        assert posix not in exported


def test_sm100a_cubin_only():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version(lib):
    assert "sm_100a" in sem.version()


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="only meaningful without a GPU")
def test_no_gpu_fails_loudly(lib):
    with pytest.raises(sem.SemError) as e:
        sem.SemContext(0)
    assert e.value.status == sem.SEM_E_CUDA


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_library_reference_tables_equal_oracle(P):
    # host-only: the library derives its tables independently (80-bit / binary128
    # Gauss-Jordan in refelem.cpp); they round to the oracle's fp64 values
    # (sympy exact / 60-digit mpmath) bit for bit
    from oracle import refelem
    g = sem.sem_debug_ref_tables(P)
    o = refelem.tables(P)
    for k in ("nodes", "wK", "wM", "Dr", "Ds"):
        assert np.array_equal(g[k], o[k]), k


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_library_stiffness_tables_equal_oracle(P):
    # P = 4, 6 (reading R21b): exact integrals, bitwise; nodal orders: D^T W D
    # formed here from the oracle's own tables (rounding-level agreement)
    from oracle import refelem
    g = sem.sem_debug_ref_stiffness(P)
    o = refelem.tables(P)
    if o.get("consistent"):
        for k in ("Srr", "Sss", "Srs"):
            assert np.array_equal(g[k], o[k]), k
    else:
        W = np.diag(o["wK"])
        ref = {"Srr": o["Dr"].T @ W @ o["Dr"], "Sss": o["Ds"].T @ W @ o["Ds"],
               "Srs": o["Dr"].T @ W @ o["Ds"] + o["Ds"].T @ W @ o["Dr"]}
        for k in ref:
            assert np.abs(g[k] - ref[k]).max() <= 1e-13 * np.abs(ref[k]).max(), k


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_stiffness_tables_reflection_symmetry(P):
    # K7's one-thread element products (P3-P5, step.cu mirror_products) read one set of
    # (Srr, Sss, Srs) per mirror pair: the reflection r <-> s of the reference triangle,
    # lattice node (i, j) -> (j, i), maps Srr onto Sss and Srs onto itself.  The identity is
    # exact in the library's P4-P7 tables and holds to a few ulp at P2/P3 (DESIGN.md v12).
    g = sem.sem_debug_ref_stiffness(P)
    lat = [(i, j) for j in range(P + 1) for i in range(P + 1 - j)]
    idx = {n: k for k, n in enumerate(lat)}
    pi = np.array([idx[(j, i)] for (i, j) in lat])
    A = np.ix_(pi, pi)
    scale = max(np.abs(g[k]).max() for k in ("Srr", "Sss", "Srs"))
    tol = 0.0 if P >= 4 else 4 * np.finfo(float).eps * scale
    assert np.abs(g["Sss"] - g["Srr"][A]).max() <= tol
    assert np.abs(g["Srs"] - g["Srs"][A]).max() <= tol
    # the rotation (i, j) -> (P - i - j, i) maps K^e(G) onto K^e(T(G)) with
    # T(G) = (gss, grr + 2 grs + gss, -(grs + gss)) (the six-symmetry form of section 6)
    rho = np.array([idx[(P - i - j, i)] for (i, j) in lat])
    grr, gss, grs = 1.3, 0.7, -0.2
    K = grr * g["Srr"] + gss * g["Sss"] + grs * g["Srs"]
    KT = gss * g["Srr"] + (grr + 2 * grs + gss) * g["Sss"] - (grs + gss) * g["Srs"]
    assert np.abs(K[np.ix_(rho, rho)] - KT).max() <= 64 * np.finfo(float).eps * np.abs(K).max()


@pytest.mark.parametrize("P", [1, 8])
def test_library_rejects_unsupported_degrees(P):
    with pytest.raises(sem.SemError) as e:
        sem.sem_debug_ref_tables(P)
    assert e.value.status == sem.SEM_E_UNSUPPORTED


def _run_isolated(code):
    env = dict(os.environ)
    env.pop("SEM_NCCL_LIB", None)
    return subprocess.run(["python", "-c", code], capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)


def test_nccl_before_torch_does_not_break_torch(lib):
    """Round-1 regression (VERDICT weak #1): loading NCCL through libsem before
    `import torch` must not map the system libnccl under torch's soname."""
    r = _run_isolated("from paper_2104_08416_b200 import sem\n"
                      "a = sem.nccl_unique_id()\n"
                      "assert len(a) == 128 and any(a)\n"
                      "import torch, torch.distributed\n"
                      "print('ok', torch.__version__)\n")
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_nccl_resolves_torch_wheel_copy(lib):
    """The binding points libsem at the nvidia-nccl wheel's library (the file torch loads)."""
    r = _run_isolated("import os\n"
                      "from paper_2104_08416_b200 import sem\n"
                      "sem.nccl_unique_id()\n"
                      "maps = open('/proc/self/maps').read()\n"
                      "libs = {l.split()[-1] for l in maps.splitlines() if 'libnccl' in l}\n"
                      "print(sorted(libs))\n"
                      "assert len(libs) == 1, libs\n"
                      "assert os.environ['SEM_NCCL_LIB'] in libs, (os.environ['SEM_NCCL_LIB'], libs)\n")
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
