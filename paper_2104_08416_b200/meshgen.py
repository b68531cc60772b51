"""Seeded synthetic inputs (the ONLY module shared by the oracle tests and the
product path).  It holds none of the method's arithmetic: it makes linear
triangle meshes, per-element wave speeds, the source vertex and the time step
*as inputs*, the way the paper's Gmsh files and scenario scripts did
(PAPER.md:540, :572, :962-986, :1489-1516).

Recipe:
* grid nx x ny cells over [0,Lx] x [0,Ly]; vertex id = j*(nx+1) + i (row-major);
* each cell split on its v00-v11 diagonal into (v00,v10,v11) and (v00,v11,v01),
  both counter-clockwise, cell-major element order ("natural");
* optional grading per axis: spacing s(xi) = (rho+1)/2 + (rho-1)/2 sin(2 pi m xi + phi),
  vertex coordinate = L * S(xi_i) / S(1) with S the closed-form integral;
* jitter of interior vertices, each coordinate uniform in +-alpha * h_local where
  h_local is the smaller adjacent cell width on that axis;
* "random" order = seeded permutation of elements AND vertex ids;
* layered velocity by centroid depth (depth = y_max - y), half-open [lo, hi);
* source = mesh vertex nearest the domain centre (ties -> lowest vertex id);
* dt: C1 uses 0.2 h_min / c (BASELINE configs[0]); the others use
  dt = kappa_P * min_e(inradius_e / c_e) (reading R8).
Seeds: mesh s, element perm s+1, vertex perm s+2, layers s+3 (s = config index).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# Reading R8: CFL factors for dt = kappa * min(inradius / c). Chosen so that
# dt sits well below the element-Gershgorin-safe step on every config
# (tests/test_inputs.py checks it against the oracle's bound).
KAPPA = {2: 0.35, 3: 0.15, 4: 0.15, 5: 0.05, 6: 0.07, 7: 0.01}  # measured dt_crit / min(inradius/c): P4 0.40, P5 0.17, P6 0.19, P7 0.024 (R21, R21b)


@dataclasses.dataclass
class Mesh:
    vxy: np.ndarray          # [V, 2] float64
    tri: np.ndarray          # [E, 3] int32
    nx: int
    ny: int
    # permutations applied by `shuffle` (identity when natural):
    elem_perm: np.ndarray | None = None   # new element k came from natural element elem_perm[k]
    vert_perm: np.ndarray | None = None   # new vertex v came from natural vertex vert_perm[v]

    @property
    def nv(self) -> int:
        return self.vxy.shape[0]

    @property
    def ne(self) -> int:
        return self.tri.shape[0]


def _graded_coords(n: int, L: float, rho: float, m: int, phi: float) -> np.ndarray:
    xi = np.arange(n + 1, dtype=np.float64) / n
    a = (rho + 1.0) / 2.0
    b = (rho - 1.0) / 2.0
    k = 2.0 * math.pi * m
    S = a * xi - (b / k) * (np.cos(k * xi + phi) - math.cos(phi))
    S1 = a  # cos(k + phi) = cos(phi) for integer m
    x = L * S / S1
    x[0] = 0.0
    x[-1] = L
    return x


def grid_mesh(nx: int, ny: int, Lx: float, Ly: float, alpha: float = 0.0, seed: int = 0,
              grade: tuple | None = None) -> Mesh:
    """Jittered (optionally graded) 2-triangles-per-cell mesh in natural order."""
    rng = np.random.default_rng(seed)
    if grade is None:
        xs = np.linspace(0.0, Lx, nx + 1)
        ys = np.linspace(0.0, Ly, ny + 1)
    else:
        rho, mx, my = grade
        phx, phy = rng.uniform(0.0, 2.0 * math.pi, size=2)
        xs = _graded_coords(nx, Lx, rho, mx, phx)
        ys = _graded_coords(ny, Ly, rho, my, phy)
    X, Yg = np.meshgrid(xs, ys)  # [ny+1, nx+1]
    vxy = np.stack([X.ravel(), Yg.ravel()], axis=1).astype(np.float64)
    if alpha > 0.0:
        dx = np.diff(xs)
        dy = np.diff(ys)
        hx = np.minimum(dx[:-1], dx[1:])  # interior vertex i = 1..nx-1
        hy = np.minimum(dy[:-1], dy[1:])
        jx = rng.uniform(-alpha, alpha, size=(ny - 1, nx - 1)) * hx[None, :]
        jy = rng.uniform(-alpha, alpha, size=(ny - 1, nx - 1)) * hy[:, None]
        V = vxy.reshape(ny + 1, nx + 1, 2)
        V[1:-1, 1:-1, 0] += jx
        V[1:-1, 1:-1, 1] += jy
        vxy = V.reshape(-1, 2)
    i = np.arange(nx, dtype=np.int64)
    j = np.arange(ny, dtype=np.int64)
    I, J = np.meshgrid(i, j)
    v00 = (J * (nx + 1) + I).ravel()
    v10 = v00 + 1
    v01 = v00 + (nx + 1)
    v11 = v01 + 1
    tri = np.empty((2 * nx * ny, 3), np.int64)
    tri[0::2] = np.stack([v00, v10, v11], axis=1)
    tri[1::2] = np.stack([v00, v11, v01], axis=1)
    m = Mesh(vxy=np.ascontiguousarray(vxy), tri=tri.astype(np.int32), nx=nx, ny=ny)
    _assert_positive(m)
    return m


def fan_mesh(n=48, rings=3):
    """Test input: a vertex shared by n triangles (a high-valence fan) inside `rings` rings of
    vertices (the chunk builder's and node graph's limits, tests/)."""
    vxy = [(0.0, 0.0)]
    for r in range(1, rings + 1):
        for k in range(n):
            a = 2 * np.pi * (k + 0.5 * (r % 2)) / n
            vxy.append((r * np.cos(a), r * np.sin(a)))
    ring = lambda r, k: 1 + (r - 1) * n + (k % n)  # noqa: E731
    tri = [(0, ring(1, k), ring(1, k + 1)) for k in range(n)]
    for r in range(1, rings):
        for k in range(n):
            if r % 2:  # the outer ring is rotated by half a step
                tri.append((ring(r, k + 1), ring(r, k), ring(r + 1, k)))
                tri.append((ring(r, k + 1), ring(r + 1, k), ring(r + 1, k + 1)))
            else:
                tri.append((ring(r, k), ring(r + 1, k), ring(r, k + 1)))
                tri.append((ring(r, k + 1), ring(r + 1, k), ring(r + 1, k + 1)))
    vxy = np.array(vxy, np.float64)
    tri = np.array(tri, np.int32)
    p0, p1, p2 = vxy[tri[:, 0]], vxy[tri[:, 1]], vxy[tri[:, 2]]
    area2 = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
    tri[area2 < 0] = tri[area2 < 0][:, [0, 2, 1]]
    return Mesh(vxy=vxy, tri=tri, nx=0, ny=0)


def _signed_area2(vxy, tri):
    p0 = vxy[tri[:, 0]]
    p1 = vxy[tri[:, 1]]
    p2 = vxy[tri[:, 2]]
    return (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])


def _assert_positive(m: Mesh):
    a = _signed_area2(m.vxy, m.tri)
    if not (a > 0).all():
        bad = int(np.argmin(a))
        raise ValueError("generator produced a non-positive element %d (area2=%g)" % (bad, a[bad]))


def shuffle(m: Mesh, seed_elem: int, seed_vert: int) -> Mesh:
    """Permute element order and vertex ids (the paper's "None" on a shuffled file)."""
    ep = np.random.default_rng(seed_elem).permutation(m.ne).astype(np.int32)
    vp = np.random.default_rng(seed_vert).permutation(m.nv).astype(np.int32)
    inv_vp = np.empty_like(vp)
    inv_vp[vp] = np.arange(m.nv, dtype=np.int32)
    vxy = np.ascontiguousarray(m.vxy[vp])
    tri = np.ascontiguousarray(inv_vp[m.tri[ep]])
    return Mesh(vxy=vxy, tri=tri, nx=m.nx, ny=m.ny, elem_perm=ep, vert_perm=vp)


def centroids(m: Mesh) -> np.ndarray:
    return m.vxy[m.tri].mean(axis=1)


def layered_speed(m: Mesh, breaks, speeds) -> np.ndarray:
    """c_e from centroid depth below the top (half-open [lo, hi); a centroid on a
    break goes to the deeper layer)."""
    ymax = m.vxy[:, 1].max()
    depth = ymax - centroids(m)[:, 1]
    idx = np.searchsorted(np.asarray(breaks, np.float64), depth, side="right")
    return np.asarray(speeds, np.float64)[idx]


def source_vertex(m: Mesh) -> int:
    """Mesh vertex nearest the domain centre; ties -> lowest vertex id."""
    lo = m.vxy.min(axis=0)
    hi = m.vxy.max(axis=0)
    ctr = 0.5 * (lo + hi)
    d2 = ((m.vxy - ctr) ** 2).sum(axis=1)
    return int(np.flatnonzero(d2 == d2.min())[0])


def min_edge(m: Mesh) -> float:
    p = m.vxy[m.tri]
    e = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 1], p[:, 0] - p[:, 2]], axis=1)
    return float(np.sqrt((e ** 2).sum(axis=2)).min())


def inradius(m: Mesh) -> np.ndarray:
    p = m.vxy[m.tri]
    la = np.sqrt(((p[:, 1] - p[:, 0]) ** 2).sum(axis=1))
    lb = np.sqrt(((p[:, 2] - p[:, 1]) ** 2).sum(axis=1))
    lc = np.sqrt(((p[:, 0] - p[:, 2]) ** 2).sum(axis=1))
    area = 0.5 * np.abs(_signed_area2(m.vxy, m.tri))
    return 2.0 * area / (la + lb + lc)


def cfl_dt(m: Mesh, c: np.ndarray, P: int) -> float:
    return float(KAPPA[P] * (inradius(m) / c).min())


# --------------------------------------------------------------------------
# The BASELINE.json configurations
# --------------------------------------------------------------------------

@dataclasses.dataclass
class Problem:
    name: str
    mesh: Mesh
    P: int
    c: np.ndarray           # [E] per element, in mesh.tri order
    src_vertex: int
    f0: float
    t0: float
    amplitude: float
    dt: float
    n_steps: int
    natural: Mesh | None = None   # the unshuffled mesh (for the "natural" ordering)
    c_natural: np.ndarray | None = None

    @property
    def ne(self):
        return self.mesh.ne


def _finish(name, nat: Mesh, P, c_nat, f0, n_steps, s, dt=None, shuffled=True):
    if dt is None:
        dt = cfl_dt(nat, c_nat, P)
    if shuffled:
        sh = shuffle(nat, s + 1, s + 2)
        c = np.ascontiguousarray(c_nat[sh.elem_perm])
    else:
        sh, c = nat, c_nat
    return Problem(name=name, mesh=sh, P=P, c=c, src_vertex=source_vertex(sh), f0=f0, t0=1.2 / f0,
                   amplitude=1.0, dt=dt, n_steps=n_steps, natural=nat, c_natural=c_nat)


def config(name: str, scale: int = 1, gpus: int = 1, degree: int | None = None) -> Problem:
    """Build a BASELINE.json configuration.

    name: C1..C5; `scale` divides the cell counts (tests use reduced sizes of the
    same recipe); `gpus` sets the C4 weak-scaling global size.
    """
    if name == "C1":
        s = 0
        n = max(2, 32 // scale)
        nat = grid_mesh(n, n, 1.0, 1.0, alpha=0.2, seed=s)
        c = np.ones(nat.ne)
        dt = 0.2 * min_edge(nat) / 1.0
        return _finish("C1", nat, 2, c, 10.0, 200, s, dt=dt)
    if name == "C2":
        s = 1
        n = max(2, 512 // scale)
        nat = grid_mesh(n, n, 4000.0, 4000.0, alpha=0.25, seed=s)
        c = np.full(nat.ne, 2000.0)
        return _finish("C2", nat, 3, c, 15.0, 1000, s)
    if name == "C3":
        s = 2
        nx, ny = max(2, 2000 // scale), max(2, 1000 // scale)
        nat = grid_mesh(nx, ny, 8000.0, 4000.0, alpha=0.2, seed=s, grade=(10.0, 2, 1))
        c = layered_speed(nat, [1000.0, 2500.0], [1500.0, 2500.0, 3500.0])
        return _finish("C3", nat, 3, c, 10.0, 2000, s)
    if name == "C4":
        s = 3
        a, b = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}[gpus]
        n = max(2, 2048 // scale)
        h = 4000.0 / 512.0 * scale
        nx, ny = n * a, n * b
        nat = grid_mesh(nx, ny, nx * h, ny * h, alpha=0.25, seed=s)
        c = np.full(nat.ne, 2000.0)
        return _finish("C4", nat, 3, c, 15.0, 500, s)
    if name == "C5":
        s = 4
        nx, ny = max(2, 16384 // scale), max(2, 8192 // scale)
        nat = grid_mesh(nx, ny, 16000.0, 8000.0, alpha=0.2, seed=s, grade=(10.0, 2, 1))
        rng = np.random.default_rng(s + 3)
        breaks = np.sort(rng.uniform(0.0, 8000.0, size=9))
        speeds = rng.uniform(1500.0, 4500.0, size=10)
        c = layered_speed(nat, breaks, speeds)
        return _finish("C5", nat, 2, c, 10.0, 200, s)
    if name == "B1":
        # The paper's Benchmark 1: single-layered domain 2000 units
        # wide and 1000 deep, homogeneous element sizes, 250k / 500k / 1M elements,
        # orders 5-7.  Synthetic stand-in for its Gmsh mesh:
        # 1000 x 500 cells -> 1M triangles at scale 1; +-0.2h jitter; c = 2000;
        # Ricker 10 Hz at the centre.  Degree from `degree` (default 5).
        s = 5
        nx, ny = max(2, 1000 // scale), max(2, 500 // scale)
        nat = grid_mesh(nx, ny, 2000.0, 1000.0, alpha=0.2, seed=s)
        c = np.full(nat.ne, 2000.0)
        return _finish("B1", nat, degree or 5, c, 10.0, 200, s)
    raise KeyError(name)


# Reading R19: the Heun step amplifies a mode of frequency w
# by (1 + (w h)^4 / 4)^(1/2) per step; every recipe dt sits below half the
# leapfrog limit 2 / w_max (tests/test_inputs.py), so h = dt / 5 keeps
# w_max h < 0.2 (growth < 2e-4 per step for the stiffest mode).
HEUN_H_FRACTION = 0.2


def heun_h(pb: Problem) -> float:
    return pb.dt * HEUN_H_FRACTION
