"""Thin ctypes binding of libsem.so (include/sem.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.  There is no CPU
fallback -- if libsem.so is missing or no B200 is present, calls raise.

The names mirror the C ABI (sem_create, sem_mesh_reorder, sem_build_operators,
sem_step_n, sem_read_field, sem_write_state, ...); ``SemContext`` wraps them
for convenience.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEM_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("SEM_LIB") or os.path.join(_HERE, "libsem.so")

SEM_OK, SEM_E_ARG, SEM_E_STATE, SEM_E_MESH, SEM_E_UNSUPPORTED = 0, 1, 2, 3, 4
SEM_E_CUDA, SEM_E_NCCL, SEM_E_OOM, SEM_E_NONFINITE = 5, 6, 7, 8
STATUS_NAMES = {0: "SEM_OK", 1: "SEM_E_ARG", 2: "SEM_E_STATE", 3: "SEM_E_MESH", 4: "SEM_E_UNSUPPORTED",
                5: "SEM_E_CUDA", 6: "SEM_E_NCCL", 7: "SEM_E_OOM", 8: "SEM_E_NONFINITE"}
SEM_ORDER_INPUT, SEM_ORDER_HILBERT, SEM_ORDER_RANDOM, SEM_ORDER_CONN, SEM_ORDER_DIST = 0, 1, 2, 3, 4
SEM_NODES_FIRST_TOUCH, SEM_NODES_FIRST_TOUCH_DEGREE, SEM_NODES_CANONICAL, SEM_NODES_VISIT = 0, 1, 2, 3
SEM_NUMBERING_CANONICAL, SEM_NUMBERING_INTERNAL = 0, 1
SEM_INTEGRATOR_LEAPFROG, SEM_INTEGRATOR_HEUN = 0, 1
SEM_SCATTER_CHUNK, SEM_SCATTER_ATOMIC, SEM_SCATTER_COLOR = 0, 1, 2

EXPORTED = ["sem_create", "sem_free", "sem_last_error", "sem_mesh_reorder", "sem_build_operators",
            "sem_step_n", "sem_read_field", "sem_write_state", "sem_set_step", "sem_sync",
            "sem_get_info", "sem_set_kernel_timing", "sem_kernel_times", "sem_version",
            "sem_debug_chunk_stats", "sem_debug_partition", "sem_nccl_unique_id",
            "sem_group_build_operators", "sem_group_step_n", "sem_set_integrator", "sem_read_velocity",
            "sem_write_velocity", "sem_set_scatter", "sem_debug_ref_tables", "sem_debug_ref_stiffness"]


class SemError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status
        self.msg = msg


class sem_info(C.Structure):
    _fields_ = [("n_elements", C.c_int64), ("n_nodes", C.c_int64), ("n_nodes_global", C.c_int64),
                ("degree", C.c_int32), ("nodes_per_elem", C.c_int32), ("n_chunks", C.c_int64),
                ("chunk_elems", C.c_int32), ("max_chunk_nodes", C.c_int32),
                ("n_interior_nodes", C.c_int64), ("n_shared_nodes", C.c_int64),
                ("n_partial_slots", C.c_int64), ("max_colors", C.c_int32),
                ("launches_per_step", C.c_int32), ("step", C.c_int64),
                ("bytes_alg_per_step", C.c_double), ("prep_reorder_ms", C.c_double),
                ("prep_build_ms", C.c_double), ("n_interface_nodes", C.c_int64),
                ("n_neighbors", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("n_elements_global", C.c_int64), ("first_element", C.c_int64),
                ("integrator", C.c_int32), ("scatter", C.c_int32), ("n_global_colors", C.c_int32),
                ("reserved0", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class sem_allocator(C.Structure):
    """The device-memory hook of include/sem.h."""
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("user", C.c_void_p)]


def torch_allocator(device: int = 0) -> sem_allocator:
    """A sem_allocator that takes the library's device memory from PyTorch's caching
    allocator (stream-ordered on the context's stream).  Keep the returned object alive
    as long as the context (SemContext does)."""
    import torch

    def _alloc(nbytes, stream, user):
        try:
            with torch.cuda.device(device):
                return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
        except Exception:  # out of memory etc.: libsem reports SEM_E_CUDA
            return None

    def _free(ptr, stream, user):
        with torch.cuda.device(device):
            torch.cuda.caching_allocator_delete(int(ptr))

    return sem_allocator(_ALLOC_FN(_alloc), _FREE_FN(_free), None)


_lib = None
_lock = threading.Lock()


def _torch_nccl_path():
    """The libnccl.so.2 of the nvidia-nccl wheel (the file torch loads), found without
    importing torch; None if the wheel is absent."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        f = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(f):
            return f
    return None


def load(path: str = LIB_PATH):
    """Load libsem.so (raises if it has not been built: no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError("libsem.so not built (%s); run `python -m paper_2104_08416_b200.build`" % path)
        # libsem dlopens NCCL lazily; point it at torch's copy so that loading NCCL before
        # `import torch` cannot map the older system library under the same soname
        # (csrc/api.cu: nccl()).  An explicit SEM_NCCL_LIB wins.
        if not os.environ.get("SEM_NCCL_LIB"):
            f = _torch_nccl_path()
            if f:
                os.environ["SEM_NCCL_LIB"] = f
        L = C.CDLL(path)
        P, i64, i32, u64, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        L.sem_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, P, P, C.POINTER(sem_allocator)]
        L.sem_free.argtypes = [P]
        L.sem_free.restype = None
        L.sem_last_error.argtypes = [P]
        L.sem_last_error.restype = C.c_char_p
        L.sem_mesh_reorder.argtypes = [P, P, i64, P, i64, C.c_int, C.c_int, C.c_int, u64, P, P, P,
                                       C.POINTER(i64), P]
        L.sem_build_operators.argtypes = [P, P, i64, dbl, dbl, dbl, dbl]
        L.sem_step_n.argtypes = [P, i64]
        L.sem_read_field.argtypes = [P, P, C.c_int, C.POINTER(i64)]
        L.sem_write_state.argtypes = [P, P, P, C.c_int]
        L.sem_set_step.argtypes = [P, i64]
        L.sem_sync.argtypes = [P]
        L.sem_get_info.argtypes = [P, C.POINTER(sem_info)]
        L.sem_set_kernel_timing.argtypes = [P, C.c_int]
        L.sem_kernel_times.argtypes = [P, C.POINTER(dbl), C.POINTER(i64), C.POINTER(dbl), C.POINTER(i64)]
        L.sem_debug_chunk_stats.argtypes = [P, i64, C.c_int, i64, C.c_int, P, P, P, P]
        L.sem_debug_partition.argtypes = [P, i64, C.c_int, i64, C.c_int, C.c_int, P, P, P, P, P, P, P, P]
        L.sem_nccl_unique_id.argtypes = [P]
        L.sem_group_build_operators.argtypes = [P, C.c_int, P, i64, dbl, dbl, dbl, dbl]
        L.sem_group_step_n.argtypes = [P, C.c_int, i64]
        L.sem_set_integrator.argtypes = [P, C.c_int]
        L.sem_set_scatter.argtypes = [P, C.c_int]
        L.sem_debug_ref_tables.argtypes = [C.c_int, P, P, P, P, P, P]
        L.sem_debug_ref_stiffness.argtypes = [C.c_int, P, P, P]
        L.sem_read_velocity.argtypes = [P, P, C.POINTER(i64)]
        L.sem_write_velocity.argtypes = [P, P]
        L.sem_version.argtypes = []
        L.sem_version.restype = C.c_char_p
        for n in EXPORTED:
            if n not in ("sem_free", "sem_last_error", "sem_version"):
                getattr(L, n).restype = C.c_int
        _lib = L
        return L


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


class SemContext:
    """One libsem context (one GPU / rank)."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None,
                 stream: int | None = None, allocator: sem_allocator | str | None = None):
        """allocator: None (the library's stream-ordered pool), "torch" (PyTorch's caching
        allocator) or a sem_allocator."""
        self.L = load()
        h = C.c_void_p()
        idbuf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        if allocator == "torch":
            allocator = torch_allocator(device)
        self._allocator = allocator  # the callbacks must outlive the context
        st = self.L.sem_create(C.byref(h), device, rank, world_size, idbuf,
                               None if stream is None else C.c_void_p(stream),
                               None if allocator is None else C.byref(allocator))
        self.h = h
        if st != SEM_OK:
            msg = self.L.sem_last_error(h).decode() if h.value else ""
            if h.value:
                self.L.sem_free(h)
                self.h = C.c_void_p()
            raise SemError(st, msg or "sem_create failed")
        self.N = None
        self.E = None

    # -- helpers --
    def _check(self, st):
        if st != SEM_OK:
            raise SemError(st, self.L.sem_last_error(self.h).decode())

    def close(self):
        if self.h and self.h.value:
            self.L.sem_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- API --
    def sem_mesh_reorder(self, vxy, tri, degree: int, elem_order=SEM_ORDER_HILBERT,
                         node_order=SEM_NODES_FIRST_TOUCH, seed: int = 0, out=None):
        """Returns dict(keys, elem_perm, node_perm, n_nodes, grid).

        `out`: optional dict of caller-owned host arrays (e.g. pinned) with keys
        "keys" (uint32 [E]), "elem_perm" (int32 [E]), "node_perm" (int32, at least
        V + 3E(P-1) + E*nI entries); a key mapped to None skips that output."""
        vxy = np.ascontiguousarray(vxy, np.float64)
        tri = np.ascontiguousarray(tri, np.int32)
        E, nv = tri.shape[0], vxy.shape[0]
        nI = (degree - 1) * (degree - 2) // 2 if degree >= 1 else 0
        nmax = nv + 3 * E * max(degree - 1, 0) + E * nI
        want = {"keys": (np.uint32, E), "elem_perm": (np.int32, E), "node_perm": (np.int32, max(nmax, 1))}
        bufs = {}
        for k, (dt, n) in want.items():
            if out is not None and k in out:
                a = out[k]
                if a is not None and (a.dtype != dt or a.size < n or not a.flags.c_contiguous):
                    raise ValueError("out[%r] must be a contiguous %s array of at least %d entries" % (k, dt.__name__, n))
                bufs[k] = a
            else:
                bufs[k] = np.empty(n, dt)
        nn = C.c_int64(0)
        grid = np.zeros(2, np.int32)
        self._check(self.L.sem_mesh_reorder(self.h, _ptr(vxy), nv, _ptr(tri), E, degree, elem_order,
                                            node_order, seed, _ptr(bufs["keys"]), _ptr(bufs["elem_perm"]),
                                            _ptr(bufs["node_perm"]), C.byref(nn), _ptr(grid)))
        self.N = nn.value
        self.E = E
        keys, eperm, nperm = bufs["keys"], bufs["elem_perm"], bufs["node_perm"]
        return {"keys": None if keys is None else keys[:E], "elem_perm": None if eperm is None else eperm[:E],
                "node_perm": None if nperm is None else nperm[: nn.value],
                "n_nodes": nn.value, "grid": (int(grid[0]), int(grid[1]))}

    def sem_build_operators(self, c_elem, src_vertex: int, f0: float, t0: float, amplitude: float, dt: float):
        c_elem = np.ascontiguousarray(c_elem, np.float64)
        self._check(self.L.sem_build_operators(self.h, _ptr(c_elem), int(src_vertex), float(f0), float(t0),
                                               float(amplitude), float(dt)))

    def sem_step_n(self, n: int):
        self._check(self.L.sem_step_n(self.h, int(n)))

    def sem_read_field(self, numbering=SEM_NUMBERING_CANONICAL, out=None):
        """U^n as a global array [N]; with several ranks only this rank's owned
        entries are written into `out` (merge ranks by passing the same array)."""
        out = np.full(self.N, np.nan) if out is None else out
        step = C.c_int64(0)
        self._check(self.L.sem_read_field(self.h, _ptr(out), numbering, C.byref(step)))
        return out, step.value

    def sem_write_state(self, u_curr, u_prev, numbering=SEM_NUMBERING_CANONICAL):
        a = None if u_curr is None else np.ascontiguousarray(u_curr, np.float64)
        b = None if u_prev is None else np.ascontiguousarray(u_prev, np.float64)
        self._check(self.L.sem_write_state(self.h, _ptr(a), _ptr(b), numbering))

    def sem_set_scatter(self, mode: int):
        self._check(self.L.sem_set_scatter(self.h, int(mode)))

    def sem_set_integrator(self, integrator: int):
        self._check(self.L.sem_set_integrator(self.h, int(integrator)))

    def sem_read_velocity(self, out=None):
        """Heun: V^n as [E, Np, 2] in input element order; with several ranks
        only this rank's elements are written into `out` (merge ranks by passing
        the same array)."""
        info = self.sem_get_info()
        out = np.full((self.E, info["nodes_per_elem"], 2), np.nan) if out is None else out
        step = C.c_int64(0)
        self._check(self.L.sem_read_velocity(self.h, _ptr(out), C.byref(step)))
        return out, step.value

    def sem_write_velocity(self, V):
        v = None if V is None else np.ascontiguousarray(V, np.float64)
        self._check(self.L.sem_write_velocity(self.h, _ptr(v)))

    def sem_set_step(self, step: int):
        self._check(self.L.sem_set_step(self.h, int(step)))

    def sem_sync(self):
        self._check(self.L.sem_sync(self.h))

    def sem_get_info(self) -> dict:
        info = sem_info()
        self._check(self.L.sem_get_info(self.h, C.byref(info)))
        return info.as_dict()

    def sem_set_kernel_timing(self, enable: bool):
        self._check(self.L.sem_set_kernel_timing(self.h, int(bool(enable))))

    def sem_kernel_times(self):
        a, b = C.c_double(), C.c_double()
        na, nb = C.c_int64(), C.c_int64()
        self._check(self.L.sem_kernel_times(self.h, C.byref(a), C.byref(na), C.byref(b), C.byref(nb)))
        return {"k7_ms": a.value, "k7_launches": na.value, "k8_ms": b.value, "k8_launches": nb.value}


def version() -> str:
    return load().sem_version().decode()


CHUNK_STAT_KEYS = ["nchunks", "N_int", "N_sh", "n_slots", "max_local", "max_win", "max_count",
                   "max_colors", "sum_nint", "sum_nsh", "max_nsh"]


def sem_debug_chunk_stats(mu, N: int, B: int = 256, want_maps: bool = False):
    """Host-only chunk-builder diagnostics (see include/sem.h)."""
    L = load()
    mu = np.ascontiguousarray(mu, np.int32)
    E, Np = mu.shape
    st = np.zeros(16, np.int64)
    int_of = np.empty(N, np.int32) if want_maps else None
    nch = (E + B - 1) // B
    cmeta = np.empty(nch * 8, np.int32) if want_maps else None
    own0 = np.empty(nch + 1, np.int32) if want_maps else None
    rc = L.sem_debug_chunk_stats(_ptr(mu), E, Np, N, B, _ptr(st), _ptr(int_of), _ptr(cmeta), _ptr(own0))
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_chunk_stats failed")
    d = {k: int(v) for k, v in zip(CHUNK_STAT_KEYS, st)}
    if want_maps:
        d["int_of"] = int_of
        d["cmeta"] = cmeta.reshape(nch, 8)
        d["own0"] = own0
    return d


def sem_debug_ref_tables(degree: int) -> dict:
    """Host-only: the library's reference tables (see include/sem.h)."""
    L = load()
    n = np.zeros(1, np.int32)
    rc = L.sem_debug_ref_tables(degree, _ptr(n), None, None, None, None, None)
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_ref_tables(%d)" % degree)
    Np = int(n[0])
    out = {"Np": Np, "nodes": np.empty((Np, 2)), "wK": np.empty(Np), "wM": np.empty(Np),
           "Dr": np.empty((Np, Np)), "Ds": np.empty((Np, Np))}
    rc = L.sem_debug_ref_tables(degree, _ptr(n), _ptr(out["nodes"]), _ptr(out["wK"]), _ptr(out["wM"]),
                                _ptr(out["Dr"]), _ptr(out["Ds"]))
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_ref_tables(%d)" % degree)
    return out


def sem_debug_ref_stiffness(degree: int) -> dict:
    """Host-only: the library's Srr, Sss, Srs (see include/sem.h)."""
    Np = sem_debug_ref_tables(degree)["Np"]
    out = {k: np.empty((Np, Np)) for k in ("Srr", "Sss", "Srs")}
    rc = load().sem_debug_ref_stiffness(degree, _ptr(out["Srr"]), _ptr(out["Sss"]), _ptr(out["Srs"]))
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_ref_stiffness(%d)" % degree)
    return out


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast the bytes)."""
    L = load()
    buf = C.create_string_buffer(128)
    rc = L.sem_nccl_unique_id(buf)
    if rc != SEM_OK:
        raise SemError(rc, "sem_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


class LoopbackGroup:
    """G in-process partitions (loopback exchange, SURVEY §8e test transport)."""

    def __init__(self, world: int, device: int = 0, allocator=None):
        if allocator == "torch":
            allocator = torch_allocator(device)
        self._allocator = allocator
        self.ctxs = [SemContext(device, r, world, allocator=allocator) for r in range(world)]
        self.world = world
        self._arr = (C.c_void_p * world)(*[c.h.value for c in self.ctxs])

    def sem_mesh_reorder(self, *a, **k):
        return [c.sem_mesh_reorder(*a, **k) for c in self.ctxs][0]

    def sem_build_operators(self, c_elem, src_vertex, f0, t0, amplitude, dt):
        c_elem = np.ascontiguousarray(c_elem, np.float64)
        rc = load().sem_group_build_operators(self._arr, self.world, _ptr(c_elem), int(src_vertex), float(f0),
                                              float(t0), float(amplitude), float(dt))
        self._check(rc)

    def sem_step_n(self, n):
        self._check(load().sem_group_step_n(self._arr, self.world, int(n)))

    def _check(self, rc):
        if rc != SEM_OK:
            msgs = "; ".join(c.L.sem_last_error(c.h).decode() for c in self.ctxs)
            raise SemError(rc, msgs)

    def sem_write_state(self, u, up, numbering=SEM_NUMBERING_CANONICAL):
        for c in self.ctxs:
            c.sem_write_state(u, up, numbering)

    def sem_set_step(self, n):
        for c in self.ctxs:
            c.sem_set_step(n)

    def sem_set_integrator(self, integrator):
        for c in self.ctxs:
            c.sem_set_integrator(integrator)

    def sem_write_velocity(self, V):
        for c in self.ctxs:
            c.sem_write_velocity(V)

    def sem_read_velocity(self):
        out, step = None, None
        for c in self.ctxs:
            out, step = c.sem_read_velocity(out=out)
        return out, step

    def sem_read_field(self, numbering=SEM_NUMBERING_CANONICAL):
        out = np.full(self.ctxs[0].N, np.nan)
        step = None
        for c in self.ctxs:
            _, step = c.sem_read_field(numbering, out=out)
        return out, step

    def close(self):
        for c in self.ctxs:
            c.close()


def sem_debug_partition(mu, N: int, rank: int, world: int) -> dict:
    """Host-only partition diagnostics (see include/sem.h)."""
    L = load()
    mu = np.ascontiguousarray(mu, np.int32)
    E, Np = mu.shape
    sz = np.zeros(8, np.int64)
    rc = L.sem_debug_partition(_ptr(mu), E, Np, N, rank, world, _ptr(sz), None, None, None, None, None, None, None)
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_partition failed")
    e0, e1, nl, nn, ns, nif, nsum, nown = (int(x) for x in sz)
    out = {"e0": e0, "e1": e1, "loc2glob": np.empty(nl, np.int32), "nbr": np.empty(nn, np.int32),
           "nbr_off": np.empty(nn + 1, np.int32), "send_glob": np.empty(ns, np.int32),
           "if_glob": np.empty(nif, np.int32), "sum_start": np.empty(nif + 1, np.int32),
           "sum_src": np.empty(nsum, np.int32), "n_owned": nown}
    rc = L.sem_debug_partition(_ptr(mu), E, Np, N, rank, world, _ptr(sz), _ptr(out["loc2glob"]), _ptr(out["nbr"]),
                               _ptr(out["nbr_off"]), _ptr(out["send_glob"]), _ptr(out["if_glob"]),
                               _ptr(out["sum_start"]), _ptr(out["sum_src"]))
    if rc != SEM_OK:
        raise SemError(rc, "sem_debug_partition failed")
    return out
