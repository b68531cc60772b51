"""ctypes wrapper + pipeline for the C oracle (TEST INFRASTRUCTURE ONLY).

See oracle/__init__.py for who may import this.  Functions map 1:1 onto
``sem_oracle.c`` and onto the paper passages cited there.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

from . import refelem

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GCC_CMD = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
           "-shared", "-o", _LIB, _SRC, "-lm"]


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(GCC_CMD, check=True)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle()
            L = C.CDLL(_LIB)
            P = C.c_void_p
            i64, i32, u64, dbl = C.c_int64, C.c_int32, C.c_uint64, C.c_double
            L.orc_splitmix64_value.argtypes = [C.c_uint64]
            L.orc_splitmix64_value.restype = C.c_uint64
            L.orc_gilbert_path.argtypes = [i32, i32, P, P]
            L.orc_gilbert_path.restype = i64
            L.orc_orient.argtypes = [P, P, i64, P, P]
            L.orc_orient.restype = C.c_int
            L.orc_hilbert_order.argtypes = [P, i64, P, i64, P, P, P]
            L.orc_hilbert_order.restype = C.c_int
            L.orc_random_order.argtypes = [i64, u64, P]
            L.orc_random_order.restype = C.c_int
            L.orc_canonical_nodes.argtypes = [P, i64, i64, C.c_int, P]
            L.orc_canonical_nodes.restype = i64
            L.orc_first_touch.argtypes = [P, i64, C.c_int, i64, P, P]
            L.orc_first_touch.restype = C.c_int
            L.orc_geometry.argtypes = [P, P, i64, P, P, P]
            L.orc_geometry.restype = None
            L.orc_lumped_mass.argtypes = [P, i64, C.c_int, i64, P, P, P]
            L.orc_lumped_mass.restype = None
            L.orc_apply_R.argtypes = [P, i64, C.c_int, i64, P, P, P, P, P, P, P, P, P]
            L.orc_apply_R.restype = None
            L.orc_ricker.argtypes = [dbl, dbl, dbl]
            L.orc_ricker.restype = dbl
            L.orc_leapfrog.argtypes = [P, i64, C.c_int, i64, P, P, P, P, P, P, P, P, P, P,
                                       i64, dbl, dbl, dbl, dbl, i64, i64, P, P]
            L.orc_apply_R_tables.argtypes = [P, i64, C.c_int, i64, P, P, P, P, P, P, P, P, P]
            L.orc_apply_R_tables.restype = None
            L.orc_leapfrog.restype = C.c_int
            L.orc_vdot.argtypes = [P, i64, C.c_int, P, P, P, P, P, P]
            L.orc_vdot.restype = None
            L.orc_rv.argtypes = [P, i64, C.c_int, i64, P, P, P, P, P, P, P, P]
            L.orc_rv.restype = None
            L.orc_heun.argtypes = [P, i64, C.c_int, i64, P, P, P, P, P, P, P,
                                   i64, dbl, dbl, dbl, dbl, i64, i64, P, P]
            L.orc_heun.restype = C.c_int
            L.orc_node_degree.argtypes = [P, i64, C.c_int, i64, P]
            L.orc_node_degree.restype = C.c_int
            L.orc_first_touch_degree.argtypes = [P, i64, C.c_int, i64, P, P]
            L.orc_first_touch_degree.restype = C.c_int
            L.orc_strategy_order.argtypes = [P, i64, C.c_int, i64, P, P, P]
            L.orc_strategy_order.restype = C.c_int
            L.orc_node_coords.argtypes = [P, P, P, i64, C.c_int, P, P]
            L.orc_node_coords.restype = None
            L.orc_set_num_threads.argtypes = [C.c_int]
            L.orc_set_num_threads.restype = None
            L.orc_num_threads.argtypes = []
            L.orc_num_threads.restype = C.c_int
            _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# SFC pieces
# --------------------------------------------------------------------------

def gilbert_path(W: int, H: int) -> np.ndarray:
    """[W*H, 2] int32 cells of the generalized Hilbert path (docs/hilbert.md)."""
    px = np.empty(W * H, np.int32)
    py = np.empty(W * H, np.int32)
    n = lib().orc_gilbert_path(W, H, _p(px), _p(py))
    if n != W * H:
        raise OracleError("gilbert_path failed")
    return np.stack([px, py], axis=1)


def hilbert_order(vxy: np.ndarray, tri: np.ndarray):
    """PAPER.md:296-305 -> (key[E] uint32 input order, perm[E] new->input, (w_b, h_b))."""
    vxy = np.ascontiguousarray(vxy, np.float64)
    tri = np.ascontiguousarray(tri, np.int32)
    ne = tri.shape[0]
    key = np.empty(ne, np.uint32)
    perm = np.empty(ne, np.int32)
    grid = np.zeros(2, np.int32)
    rc = lib().orc_hilbert_order(_p(vxy), vxy.shape[0], _p(tri), ne, _p(key), _p(perm), _p(grid))
    if rc != 0:
        raise OracleError("hilbert_order rc=%d" % rc)
    return key, perm, (int(grid[0]), int(grid[1]))


def splitmix64(x: int) -> int:
    """The oracle's key mixer of reading R16 (sem_oracle.c orc_splitmix64)."""
    return int(lib().orc_splitmix64_value(x & (2**64 - 1)))


def random_order(ne: int, seed: int) -> np.ndarray:
    perm = np.empty(ne, np.int32)
    lib().orc_random_order(ne, seed, _p(perm))
    return perm


def orient(vxy: np.ndarray, tri: np.ndarray) -> np.ndarray:
    vxy = np.ascontiguousarray(vxy, np.float64)
    tri = np.ascontiguousarray(tri, np.int32)
    out = np.empty_like(tri)
    bad = np.full(1, -1, np.int64)
    rc = lib().orc_orient(_p(vxy), _p(tri), tri.shape[0], _p(out), _p(bad))
    if rc != 0:
        raise OracleError("element %d has zero area" % int(bad[0]))
    return out


def canonical_nodes(tri_oriented: np.ndarray, nv: int, P: int):
    """R13 canonical SEM node numbering -> (mu [E,Np] int32, N)."""
    tri_oriented = np.ascontiguousarray(tri_oriented, np.int32)
    ne = tri_oriented.shape[0]
    Np = refelem.n_nodes(P)
    mu = np.empty((ne, Np), np.int32)
    N = lib().orc_canonical_nodes(_p(tri_oriented), nv, ne, P, _p(mu))
    if N < 0:
        raise OracleError("canonical_nodes rc=%d" % N)
    return mu, int(N)


def first_touch(mu: np.ndarray, N: int):
    """PAPER.md:316 first-touch labels -> (node_perm [N] new->old, mu_new)."""
    mu = np.ascontiguousarray(mu, np.int32)
    ne, Np = mu.shape
    perm = np.empty(N, np.int32)
    out = np.empty_like(mu)
    rc = lib().orc_first_touch(_p(mu), ne, Np, N, _p(perm), _p(out))
    if rc != 0:
        raise OracleError("first_touch rc=%d" % rc)
    return perm, out


def node_degree(mu: np.ndarray, N: int) -> np.ndarray:
    """deg[g] = distinct nodes sharing an element with g."""
    mu = np.ascontiguousarray(mu, np.int32)
    deg = np.empty(N, np.int32)
    rc = lib().orc_node_degree(_p(mu), mu.shape[0], mu.shape[1], N, _p(deg))
    if rc != 0:
        raise OracleError("node_degree rc=%d" % rc)
    return deg


def first_touch_degree(mu: np.ndarray, N: int):
    """PAPER.md:312-321 steps 1 and 2 -> (node_perm [N] new->old, mu_new)."""
    mu = np.ascontiguousarray(mu, np.int32)
    perm = np.empty(N, np.int32)
    out = np.empty_like(mu)
    rc = lib().orc_first_touch_degree(_p(mu), mu.shape[0], mu.shape[1], N, _p(perm), _p(out))
    if rc != 0:
        raise OracleError("first_touch_degree rc=%d" % rc)
    return perm, out


def strategy_order(mu_can: np.ndarray, N: int, key: np.ndarray):
    """Conn./Dist. strategies (reading R20) on the canonical
    connectivity (input element order) -> (elem_perm [E] new->input,
    node_perm [N] new->canonical)."""
    mu_can = np.ascontiguousarray(mu_can, np.int32)
    key = np.ascontiguousarray(key, np.float64)
    ep = np.empty(mu_can.shape[0], np.int32)
    npm = np.empty(N, np.int32)
    rc = lib().orc_strategy_order(_p(mu_can), mu_can.shape[0], mu_can.shape[1], N, _p(key), _p(ep), _p(npm))
    if rc != 0:
        raise OracleError("strategy_order rc=%d" % rc)
    return ep, npm


def node_coords(vxy: np.ndarray, tri_oriented: np.ndarray, mu_can: np.ndarray, P: int) -> np.ndarray:
    """Canonical SEM node coordinates [N, 2] (reading R20)."""
    vxy = np.ascontiguousarray(vxy, np.float64)
    tri_oriented = np.ascontiguousarray(tri_oriented, np.int32)
    mu_can = np.ascontiguousarray(mu_can, np.int32)
    nodes = refelem.tables(P)["nodes"]
    edge_t = np.ascontiguousarray([nodes[i, 0] for i in range(1, P)], np.float64)
    N = int(mu_can.max()) + 1
    xy = np.full((N, 2), np.nan)
    lib().orc_node_coords(_p(vxy), _p(tri_oriented), _p(mu_can), mu_can.shape[0], P, _p(edge_t), _p(xy))
    return xy


def conn_key(mu_can: np.ndarray, N: int) -> np.ndarray:
    """Node Connectivity key: the degree."""
    return node_degree(mu_can, N).astype(np.float64)


def dist_key(vxy: np.ndarray, tri_oriented: np.ndarray, mu_can: np.ndarray, P: int) -> np.ndarray:
    """Node Distance key: squared distance to the lower-left corner of the
    vertex bounding box (reading R20), dx*dx + dy*dy in fp64."""
    xy = node_coords(vxy, tri_oriented, mu_can, P)
    x0, y0 = vxy[:, 0].min(), vxy[:, 1].min()
    dx = xy[:, 0] - x0
    dy = xy[:, 1] - y0
    return dx * dx + dy * dy


def ricker(t: float, f0: float, t0: float) -> float:
    return lib().orc_ricker(t, f0, t0)


# --------------------------------------------------------------------------
# Mesh + operators + leapfrog
# --------------------------------------------------------------------------

class OracleSEM:
    """The whole method on the canonical (input-order) numbering, in fp64."""

    def __init__(self, vxy, tri, P: int, c_elem=None):
        self.vxy = np.ascontiguousarray(vxy, np.float64)
        self.tri_in = np.ascontiguousarray(tri, np.int32)
        self.P = P
        self.T = refelem.tables(P)
        self.Np = self.T["Np"]
        self.nv = self.vxy.shape[0]
        self.ne = self.tri_in.shape[0]
        self.tri = orient(self.vxy, self.tri_in)
        self.mu, self.N = canonical_nodes(self.tri, self.nv, P)
        self.J = np.empty((self.ne, 4))
        self.detJ = np.empty(self.ne)
        self.Jinv = np.empty((self.ne, 4))
        lib().orc_geometry(_p(self.vxy), _p(self.tri), self.ne, _p(self.J), _p(self.detJ), _p(self.Jinv))
        self.Dr = np.ascontiguousarray(self.T["Dr"])
        self.Ds = np.ascontiguousarray(self.T["Ds"])
        self.wK = np.ascontiguousarray(self.T["wK"])
        self.wM = np.ascontiguousarray(self.T["wM"])
        self.Mbar = np.empty(self.N)
        lib().orc_lumped_mass(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.wM), _p(self.Mbar))
        self.c = np.ones(self.ne) if c_elem is None else np.ascontiguousarray(c_elem, np.float64)
        self._ebuf = None
        # reading R21b (P = 4, 6): consistent stiffness from the exact S tables
        self.S = (tuple(np.ascontiguousarray(self.T[k]) for k in ("Srr", "Sss", "Srs"))
                  if self.T.get("consistent") else None)

    def set_c(self, c_elem):
        self.c = np.ascontiguousarray(c_elem, np.float64)

    def apply_R(self, U: np.ndarray) -> np.ndarray:
        """R = -K U (Algorithm 1 then Algorithm 2)."""
        U = np.ascontiguousarray(U, np.float64)
        R = np.empty(self.N)
        if self._ebuf is None:
            self._ebuf = np.empty(self.ne * self.Np)
        if self.S is not None:
            lib().orc_apply_R_tables(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.Jinv),
                                     _p(self.c), *(_p(x) for x in self.S), _p(U), _p(R), _p(self._ebuf))
        else:
            lib().orc_apply_R(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.Jinv), _p(self.c),
                              _p(self.Dr), _p(self.Ds), _p(self.wK), _p(U), _p(R), _p(self._ebuf))
        return R

    def apply_K(self, U):
        return -self.apply_R(U)

    def leapfrog(self, dt: float, n_steps: int, src: int = -1, A: float = 1.0, f0: float = 1.0,
                 t0: float = 0.0, U=None, Uprev=None, step0: int = 0):
        """n_steps of the leapfrog from (U^n, U^{n-1}) (zeros by default)."""
        U = np.zeros(self.N) if U is None else np.array(U, np.float64, copy=True)
        Up = np.zeros(self.N) if Uprev is None else np.array(Uprev, np.float64, copy=True)
        S = (None, None, None) if self.S is None else tuple(_p(x) for x in self.S)
        rc = lib().orc_leapfrog(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.Jinv),
                                _p(self.c), _p(self.Dr), _p(self.Ds), _p(self.wK), _p(self.Mbar), *S,
                                int(src), float(A), float(f0), float(t0), float(dt), int(step0),
                                int(n_steps), _p(U), _p(Up))
        if rc != 0:
            raise OracleError("leapfrog rc=%d" % rc)
        return U, Up

    # ---- the paper's Heun scheme on (U, V) (NEXT-1) ----
    def vdot(self, U):
        """Algorithm 1 (E = 0): Vdot [E, Np, 2]."""
        U = np.ascontiguousarray(U, np.float64)
        Vd = np.empty((self.ne, self.Np, 2))
        lib().orc_vdot(_p(self.mu), self.ne, self.Np, _p(self.Jinv), _p(self.c), _p(self.Dr), _p(self.Ds),
                       _p(U), _p(Vd))
        return Vd

    def rv(self, V):
        """Algorithm 2 first term (D = 0, B = -I) applied to V [E, Np, 2]."""
        V = np.ascontiguousarray(V, np.float64)
        R = np.empty(self.N)
        if self._ebuf is None:
            self._ebuf = np.empty(self.ne * self.Np)
        lib().orc_rv(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.Jinv), _p(self.Dr),
                     _p(self.Ds), _p(self.wK), _p(V), _p(R), _p(self._ebuf))
        return R

    def heun(self, h: float, n_steps: int, src: int = -1, A: float = 1.0, f0: float = 1.0, t0: float = 0.0,
             U=None, V=None, step0: int = 0):
        """n_steps Heun steps from (U^n, V^n) (zeros by default)."""
        U = np.zeros(self.N) if U is None else np.array(U, np.float64, copy=True)
        V = np.zeros((self.ne, self.Np, 2)) if V is None else np.array(V, np.float64, copy=True)
        rc = lib().orc_heun(_p(self.mu), self.ne, self.Np, self.N, _p(self.detJ), _p(self.Jinv), _p(self.c),
                            _p(self.Dr), _p(self.Ds), _p(self.wK), _p(self.Mbar), int(src), float(A), float(f0),
                            float(t0), float(h), int(step0), int(n_steps), _p(U), _p(V))
        if rc != 0:
            raise OracleError("heun rc=%d" % rc)
        return U, V

    def node_xy(self) -> np.ndarray:
        """Coordinates of every canonical node, x_mu(p,e) = F^(e)(x^_p)."""
        xy = np.full((self.N, 2), np.nan)
        nd = self.T["nodes"]
        v0 = self.vxy[self.tri[:, 0]]
        for p in range(self.Np):
            x = v0[:, 0] + self.J[:, 0] * nd[p, 0] + self.J[:, 1] * nd[p, 1]
            y = v0[:, 1] + self.J[:, 2] * nd[p, 0] + self.J[:, 3] * nd[p, 1]
            xy[self.mu[:, p], 0] = x
            xy[self.mu[:, p], 1] = y
        return xy


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))
