"""Pins for the oracle's mesh, geometry, lumped mass and stiffness (Alg. 1 o Alg. 2).

Independent anchors:
* textbook P1 stiffness  K_ij = (b_i b_j + c_i c_j) / (4A)  on a non-symmetric
  triangle (pins the K^(e) index order, reading R5, and the sign of B = -I);
* exact P2 element stiffness by symbolic integration (the P2 nodal rule is
  exact for the degree-2 integrand, so the method must reproduce it exactly);
* a dense K assembled by a direct double loop over quadrature points (P-13);
* K 1 = 0, symmetry, PSD with a single zero mode, patch test on linear fields;
* sum of lumped masses = mesh area (shoelace), all positive;
* Rayleigh quotient of the standing mode cos(pi x) cos(pi y) -> 2 pi^2 with
  convergence (SURVEY P-8);
* canonical node counts and consistent node coordinates
  x_mu(p,e) = F^(e)(x^_p) across elements sharing a node.
"""
import numpy as np
import pytest
import sympy as sp

from oracle import core, refelem
from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg


def dense_K(o: OracleSEM) -> np.ndarray:
    K = np.empty((o.N, o.N))
    for j in range(o.N):
        e = np.zeros(o.N)
        e[j] = 1.0
        K[:, j] = o.apply_K(e)
    return K


def test_node_counts_and_two_triangles():
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    one = np.array([[0, 1, 2]], np.int32)
    two = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    assert OracleSEM(vxy[:3], one, 2).N == 6
    assert OracleSEM(vxy, two, 2).N == 9       # 6 + 6 - 3
    assert OracleSEM(vxy, two, 3).N == 16      # 10 + 10 - 4
    assert OracleSEM(vxy, two, 1).N == 4


@pytest.mark.parametrize("P", [2, 3, 5, 7])
def test_grid_node_count_and_coordinates(P):
    m = mg.shuffle(mg.grid_mesh(7, 5, 3.0, 2.0, alpha=0.2, seed=1), 2, 3)
    o = OracleSEM(m.vxy, m.tri, P)
    nx, ny = 7, 5
    nedges = nx * (ny + 1) + ny * (nx + 1) + nx * ny
    nI = (P - 1) * (P - 2) // 2
    assert o.N == (nx + 1) * (ny + 1) + nedges * (P - 1) + m.ne * nI
    # every write of x_mu(p,e) agrees (nodes shared across elements are the same point)
    nd = o.T["nodes"]
    v0 = o.vxy[o.tri[:, 0]]
    xy = o.node_xy()
    for p in range(o.Np):
        x = v0[:, 0] + o.J[:, 0] * nd[p, 0] + o.J[:, 1] * nd[p, 1]
        y = v0[:, 1] + o.J[:, 2] * nd[p, 0] + o.J[:, 3] * nd[p, 1]
        assert np.abs(xy[o.mu[:, p], 0] - x).max() < 1e-12
        assert np.abs(xy[o.mu[:, p], 1] - y).max() < 1e-12
    # distinct nodes are distinct points
    r = np.round(xy / 1e-9).astype(np.int64)
    assert len(np.unique(r, axis=0)) == o.N


def test_orientation_fix_and_degenerate():
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [2.0, 0.0]])
    cw = np.array([[0, 2, 1]], np.int32)
    assert core.orient(vxy, cw).tolist() == [[0, 1, 2]]
    with pytest.raises(core.OracleError, match="element 0"):
        core.orient(vxy, np.array([[0, 1, 3]], np.int32))


def test_geometry_pins():
    o = OracleSEM(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]), np.array([[0, 1, 2]], np.int32), 2)
    assert o.J[0].tolist() == [1, 0, 0, 1] and o.detJ[0] == 1.0
    o = OracleSEM(np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 2.0]]), np.array([[0, 1, 2]], np.int32), 2)
    assert o.detJ[0] == 4.0


def test_p1_textbook_stiffness_nonsymmetric_triangle():
    pts = np.array([[0.3, -0.2], [2.1, 0.4], [0.7, 1.9]])
    o = OracleSEM(pts, np.array([[0, 1, 2]], np.int32), 1, c_elem=np.array([1.7]))
    K = dense_K(o)
    x, y = pts[:, 0], pts[:, 1]
    A = 0.5 * ((x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]))
    b = np.array([y[1] - y[2], y[2] - y[0], y[0] - y[1]])
    c = np.array([x[2] - x[1], x[0] - x[2], x[1] - x[0]])
    Kt = 1.7 ** 2 * (np.outer(b, b) + np.outer(c, c)) / (4 * A)
    assert np.abs(K - Kt).max() < 1e-13 * np.abs(Kt).max()


def test_p2_exact_element_stiffness():
    # vertices with rational coordinates -> exact J; the P2 nodal rule with
    # w = int N is exact for grad N_p . grad N_q (degree 2).
    V = [(sp.Rational(1, 5), sp.Rational(-1, 3)), (sp.Rational(9, 4), sp.Rational(1, 2)),
         (sp.Rational(2, 3), sp.Rational(7, 3))]
    J = sp.Matrix([[V[1][0] - V[0][0], V[2][0] - V[0][0]], [V[1][1] - V[0][1], V[2][1] - V[0][1]]])
    Ji = J.inv()
    B = refelem.basis(2)
    X, Y = refelem.X, refelem.Y
    grads = [sp.Matrix([sp.diff(N, X), sp.diff(N, Y)]) for N in B]
    Kex = np.zeros((6, 6))
    for p in range(6):
        for q in range(6):
            gp = Ji.T * grads[p]   # physical gradient = J^-T grad^
            gq = Ji.T * grads[q]
            Kex[p, q] = float(refelem.integrate_ref((gp.T * gq)[0, 0]) * J.det())
    pts = np.array([[float(a), float(b)] for a, b in V])
    o = OracleSEM(pts, np.array([[0, 1, 2]], np.int32), 2)
    K = dense_K(o)
    # canonical numbering of a single element: vertices 0..2 then edges
    Kloc = K[np.ix_(o.mu[0], o.mu[0])]
    assert np.abs(Kloc - Kex).max() < 1e-13 * np.abs(Kex).max()


def brute_dense_K(m, P, c):
    """P-13: K_ij = sum_e sum_k w_k grad N_i(x_k) . grad N_j(x_k) c^2 detJ, directly."""
    T = refelem.tables(P)
    o = OracleSEM(m.vxy, m.tri, P)  # numbering only
    K = np.zeros((o.N, o.N))
    for e in range(m.ne):
        v = m.vxy[o.tri[e]]
        J = np.array([[v[1, 0] - v[0, 0], v[2, 0] - v[0, 0]], [v[1, 1] - v[0, 1], v[2, 1] - v[0, 1]]])
        Ji = np.linalg.inv(J)
        dJ = np.linalg.det(J)
        for k in range(T["Np"]):
            gref = np.stack([T["Dr"][k], T["Ds"][k]])       # [2, Np]
            g = Ji.T @ gref                                  # physical gradients
            Ke = T["wK"][k] * dJ * c[e] ** 2 * (g.T @ g)
            K[np.ix_(o.mu[e], o.mu[e])] += Ke
    return K


@pytest.mark.parametrize("P", [1, 2, 3, 5, 7])
def test_dense_K_matches_direct_quadrature(P):
    m = mg.shuffle(mg.grid_mesh(3, 2, 1.5, 1.0, alpha=0.2, seed=5), 1, 2)
    assert m.ne <= 12
    c = np.linspace(1.0, 2.0, m.ne)
    o = OracleSEM(m.vxy, m.tri, P, c)
    K = dense_K(o)
    Kb = brute_dense_K(m, P, c)
    assert np.abs(K - Kb).max() < 1e-12 * np.abs(Kb).max()


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_K_properties(P):
    m = mg.grid_mesh(4, 3, 1.3, 1.0, alpha=0.2, seed=2)
    o = OracleSEM(m.vxy, m.tri, P, np.linspace(0.5, 3.0, m.ne))
    K = dense_K(o)
    assert np.abs(K - K.T).max() < 1e-12 * np.abs(K).max()
    assert np.abs(K.sum(axis=1)).max() < 1e-12 * np.abs(K).max()   # K 1 = 0
    ev = np.linalg.eigvalsh(0.5 * (K + K.T))
    assert ev[0] > -1e-12 * ev[-1]
    assert ev[1] > 1e-8 * ev[-1]  # exactly one zero mode (connected mesh, natural BC)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6, 7])
def test_patch_test_linear_field(P):
    m = mg.shuffle(mg.grid_mesh(9, 7, 2.0, 1.5, alpha=0.2, seed=4), 5, 6)
    o = OracleSEM(m.vxy, m.tri, P, np.full(m.ne, 1.3))
    xy = o.node_xy()
    ell = 0.7 + 1.9 * xy[:, 0] - 2.3 * xy[:, 1]
    Kl = o.apply_K(ell)
    tol = 1e-9
    interior = (xy[:, 0] > tol) & (xy[:, 0] < 2.0 - tol) & (xy[:, 1] > tol) & (xy[:, 1] < 1.5 - tol)
    scale = np.abs(o.apply_K(np.where(interior, 1.0, 0.0))).max()
    assert np.abs(Kl[interior]).max() < 1e-12 * scale * np.abs(ell).max()
    assert np.abs(Kl[~interior]).max() > 1e-6  # the boundary flux is really there


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_lumped_mass_area_and_positivity(P):
    m = mg.shuffle(mg.grid_mesh(11, 6, 3.0, 1.0, alpha=0.25, seed=7, grade=(10.0, 2, 1)), 8, 9)
    o = OracleSEM(m.vxy, m.tri, P)
    p = m.vxy[o.tri]
    shoelace = 0.5 * ((p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1])
                      - (p[:, 2, 0] - p[:, 0, 0]) * (p[:, 1, 1] - p[:, 0, 1])).sum()
    assert abs(o.Mbar.sum() - shoelace) < 1e-12 * shoelace
    assert abs(shoelace - 3.0) < 1e-12
    assert (o.Mbar > 0).all()


def _rayleigh_err(P, n):
    m = mg.grid_mesh(n, n, 1.0, 1.0, alpha=0.2, seed=11)
    o = OracleSEM(m.vxy, m.tri, P)
    xy = o.node_xy()
    u = np.cos(np.pi * xy[:, 0]) * np.cos(np.pi * xy[:, 1])
    rq = (u @ o.apply_K(u)) / (u @ (o.Mbar * u))
    return abs(rq - 2 * np.pi ** 2) / (2 * np.pi ** 2)


@pytest.mark.parametrize("P,ratio", [(2, 3.0), (3, 6.0)])
def test_standing_mode_rayleigh_quotient_converges(P, ratio):
    errs = [_rayleigh_err(P, n) for n in (4, 8, 16)]
    assert errs[2] < 2e-3
    assert errs[0] / errs[1] > ratio and errs[1] / errs[2] > ratio


def test_standing_mode_higher_orders_more_accurate():
    # NEXT-2 (orders 5 and 7 of PAPER.md:746-776): on the same coarse mesh the
    # Rayleigh-quotient error drops with the order, and P5 converges fast
    e3, e4, e5, e7 = (_rayleigh_err(P, 4) for P in (3, 4, 5, 7))
    assert e5 < e3 / 20 and e7 < e5 / 20
    # R21b orders: consistent stiffness with HRZ-lumped mass; the lumping caps
    # the convergence rate (P6 ~ h^4), but both converge
    assert e4 < e3 / 10
    assert _rayleigh_err(4, 2) / e4 > 8 and _rayleigh_err(6, 4) / _rayleigh_err(6, 8) > 8
    assert _rayleigh_err(5, 2) / e5 > 30
