"""Pins for the oracle's reference-triangle tables (oracle/refelem.py).

Each check is fixed by the paper or by mathematics, not by re-typing the
oracle's own formulas:
* dual system N_p(x_q) = delta_pq (eq. dual_sys);
* quadrature exactness against the closed form int x^a y^b = a! b! / (a+b+2)!
  (eq. numerical_integ);
* order-5 element has 21 nodes;
* Gauss-Lobatto edge points are the roots of the derivative of the Legendre
  polynomial P_3 (textbook; reading R3);
* the P2 consistent-mass diagonal equals the textbook P2 triangle mass matrix
  diagonal A/180 * (6, 32) (reading R4, HRZ).
"""
import math

import numpy as np
import pytest
import sympy as sp

from oracle import refelem as R

X, Y = R.X, R.Y


def closed_form_monomial(a, b):
    return sp.Rational(math.factorial(a) * math.factorial(b), math.factorial(a + b + 2))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_dual_system_exact(P):
    nd = R.nodes(P)
    B = R.basis(P)
    for p, N in enumerate(B):
        for q, (x, y) in enumerate(nd):
            v = sp.simplify(N.subs({X: x, Y: y}))
            assert v == (1 if p == q else 0)


@pytest.mark.parametrize("P", [1, 2, 3])
def test_partition_of_unity(P):
    B = R.basis(P)
    assert sp.simplify(sum(B) - 1) == 0
    T = R.tables(P)
    assert np.abs(T["Dr"].sum(axis=1)).max() < 1e-13
    assert np.abs(T["Ds"].sum(axis=1)).max() < 1e-13


@pytest.mark.parametrize("P", [1, 2, 3])
def test_stiffness_weights_exact_to_degree_P(P):
    nd = R.nodes(P)
    w = R.weights_K(P)
    assert sp.simplify(sum(w) - sp.Rational(1, 2)) == 0
    for a in range(P + 1):
        for b in range(P + 1 - a):
            q = sum(wq * (x ** a) * (y ** b) for wq, (x, y) in zip(w, nd))
            assert sp.simplify(q - closed_form_monomial(a, b)) == 0, (a, b)


def test_p3_weights_fixed_by_exactness():
    # With the symmetric node set, exactness to degree 3 fixes the three weight
    # classes; these are the resulting closed forms.
    w = R.weights_K(3)
    assert w[0] == sp.Rational(1, 120) and w[3] == sp.Rational(1, 120) and w[9] == sp.Rational(1, 120)
    assert w[5] == sp.Rational(9, 40)
    for p in (1, 2, 4, 6, 7, 8):
        assert w[p] == sp.Rational(1, 24)


def test_p2_stiffness_weights_have_zero_vertices():
    # The literal reading makes P2 vertex weights exactly zero,
    # which is why the mass uses HRZ (R4).
    w = R.weights_K(2)
    assert [w[p] for p in (0, 2, 5)] == [0, 0, 0]
    assert [w[p] for p in (1, 3, 4)] == [sp.Rational(1, 6)] * 3


def test_p2_hrz_matches_textbook_mass_diagonal():
    # Textbook P2 triangle consistent mass matrix: A/180 * diag(6,6,6,32,32,32).
    A = sp.Rational(1, 2)
    B = R.basis(2)
    diag = [R.integrate_ref(N * N) for N in B]
    for p in (0, 2, 5):
        assert diag[p] == A * 6 / 180
    for p in (1, 3, 4):
        assert diag[p] == A * 32 / 180
    wM = R.weights_M(2)
    assert sp.simplify(sum(wM) - A) == 0
    assert all(v > 0 for v in wM)
    assert wM[0] == sp.Rational(1, 38) and wM[1] == sp.Rational(8, 57)
    # HRZ integrates degree <= 1 exactly (area + first moments by symmetry)
    nd = R.nodes(2)
    for a, b in [(0, 0), (1, 0), (0, 1)]:
        q = sum(wq * (x ** a) * (y ** b) for wq, (x, y) in zip(wM, nd))
        assert sp.simplify(q - closed_form_monomial(a, b)) == 0


@pytest.mark.parametrize("P", [1, 2, 3])
def test_derivative_tables_exact_on_monomials(P):
    T = R.tables(P)
    nd = T["nodes"]
    for a in range(P + 1):
        for b in range(P + 1 - a):
            f = nd[:, 0] ** a * nd[:, 1] ** b
            dfx = a * nd[:, 0] ** max(a - 1, 0) * nd[:, 1] ** b if a else np.zeros(len(nd))
            dfy = b * nd[:, 0] ** a * nd[:, 1] ** max(b - 1, 0) if b else np.zeros(len(nd))
            assert np.abs(T["Dr"] @ f - dfx).max() < 1e-12
            assert np.abs(T["Ds"] @ f - dfy).max() < 1e-12


def test_p3_edge_nodes_are_gauss_lobatto():
    xi = sp.symbols("xi")
    dP3 = sp.diff(sp.legendre(3, xi), xi)
    roots = sorted(sp.solve(dP3, xi), key=lambda r: float(r))
    pts = [(r + 1) / 2 for r in roots]  # map [-1,1] -> [0,1]
    nd = R.nodes(3)
    assert sp.simplify(nd[1][0] - pts[0]) == 0
    assert sp.simplify(nd[2][0] - pts[1]) == 0


def test_node_counts():
    assert R.n_nodes(5) == 21  # PAPER.md:572 "order of 5, resulting in 21 local nodes"
    assert [R.n_nodes(P) for P in (1, 2, 3)] == [3, 6, 10]
    assert [len(R.nodes(P)) for P in (1, 2, 3)] == [3, 6, 10]


@pytest.mark.parametrize("P", [2, 3])
def test_fp64_tables_rounded_once(P):
    T = R.tables(P)
    Dr, Ds = R.deriv_tables(P)
    for k in range(T["Np"]):
        for p in range(T["Np"]):
            assert T["Dr"][k, p] == float(sp.N(Dr[k][p], 40))
            assert T["Ds"][k, p] == float(sp.N(Ds[k][p], 40))


# ---- P >= 4 (NEXT-2, reading R21): the high-precision path ---------------------

@pytest.mark.parametrize("P", [2, 3])
def test_hp_path_reproduces_exact_tables_bitwise(P):
    # two independent computations (sympy exact vs 60-digit mpmath) round to
    # the same fp64 tables
    T, H = R.tables(P), R.tables_hp(P)
    for k in ("nodes", "wK", "Dr", "Ds"):
        assert np.array_equal(T[k], H[k]), k


@pytest.mark.parametrize("P", [4, 5, 6, 7])
def test_hp_lobatto_edges_are_legendre_derivative_roots(P):
    import mpmath as mp
    v = R.lobatto01_hp(P)
    assert v[0] == 0 and v[-1] == 1 and len(v) == P + 1
    for x in v[1:-1]:  # P_P'(2x - 1) = 0  (textbook Gauss-Lobatto)
        assert abs(mp.diff(lambda t: mp.legendre(P, t), 2 * x - 1)) < mp.mpf("1e-40")
    nd = R.tables(P)["nodes"]
    Np = (P + 1) * (P + 2) // 2
    assert nd.shape == (Np, 2)
    # edge v0-v1 carries the 1D points, in lattice order
    assert np.array_equal(nd[:P + 1, 0], np.array([float(x) for x in v]))
    assert (nd[:P + 1, 1] == 0).all()


@pytest.mark.parametrize("P", [5, 7])
def test_hp_dual_system_and_exactness(P):
    import mpmath as mp
    T = R.tables_hp(P)
    C, ex = T["C"], T["exps"]
    nd = R.nodes_hp(P)
    Np = len(nd)
    for q, (x, y) in enumerate(nd):  # N_p(x_q) = delta_pq
        for p in range(Np):
            val = mp.fsum(C[m, p] * x ** a * y ** b for m, (a, b) in enumerate(ex))
            assert abs(val - (1 if p == q else 0)) < mp.mpf("1e-40")
    w = T["wK"]
    assert abs(w.sum() - 0.5) < 1e-15
    xy = T["nodes"]
    for a in range(P + 1):  # nodal quadrature exact to degree P
        for b in range(P + 1 - a):
            q = float(np.sum(w * xy[:, 0] ** a * xy[:, 1] ** b))
            assert abs(q - float(closed_form_monomial(a, b))) < 1e-14, (a, b)
    for a in range(P + 1):  # D exact on monomials of degree <= P
        for b in range(P + 1 - a):
            f = xy[:, 0] ** a * xy[:, 1] ** b
            dfx = a * xy[:, 0] ** max(a - 1, 0) * xy[:, 1] ** b if a else 0 * f
            dfy = b * xy[:, 0] ** a * xy[:, 1] ** max(b - 1, 0) if b else 0 * f
            assert np.abs(T["Dr"] @ f - dfx).max() < 1e-10
            assert np.abs(T["Ds"] @ f - dfy).max() < 1e-10


def test_order_5_has_21_nodes_and_positive_weights_odd_orders_only():
    # order 5 -> 21 local nodes.  The paper's orders 5-7: int N_p
    # is positive for P = 5 and 7 but negative at the vertices for P = 4 and 6,
    # where the lumped mass would not be positive (why R21 keeps P in {5, 7}).
    assert R.tables(5)["Np"] == 21 and R.tables(7)["Np"] == 36
    for P in (5, 7):
        assert (R.tables(P)["wK"] > 0).all()
    for P in (4, 6):
        w = R.tables(P)["wK"]
        verts = [0, P, (P + 1) * (P + 2) // 2 - 1]
        assert (w[verts] < 0).all() and (np.delete(w, verts) > 0).all()


@pytest.mark.parametrize("P", [4, 6])
def test_consistent_tables_even_orders(P):
    """Reading R21b: exact S tables against an independent quadrature (Gauss-
    Legendre on the collapsed square, x = u (1 - v), y = v, Jacobian 1 - v,
    exact for the degree-2P-2 integrands) and the HRZ mass."""
    import mpmath as mp
    T = R.tables_hp(P)
    C, ex = T["C"], T["exps"]
    Np = T["Np"]
    n = P + 2
    gx, gw = np.polynomial.legendre.leggauss(n)
    u = 0.5 * (gx + 1.0)
    wq = 0.5 * gw
    X, Yq = np.meshgrid(u, u, indexing="ij")
    W = np.outer(wq, wq) * (1.0 - Yq)
    xx, yy = X * (1.0 - Yq), Yq
    Cf = np.array([[float(C[m, p]) for p in range(Np)] for m in range(Np)])
    dr = sum(Cf[m][:, None, None] * (a * xx ** max(a - 1, 0) * yy ** b if a else 0 * xx)
             for m, (a, b) in enumerate(ex))
    ds = sum(Cf[m][:, None, None] * (b * xx ** a * yy ** max(b - 1, 0) if b else 0 * xx)
             for m, (a, b) in enumerate(ex))
    val = sum(Cf[m][:, None, None] * xx ** a * yy ** b for m, (a, b) in enumerate(ex))
    Srr = np.einsum("pij,qij,ij->pq", dr, dr, W)
    Sss = np.einsum("pij,qij,ij->pq", ds, ds, W)
    Srs = np.einsum("pij,qij,ij->pq", dr, ds, W)
    Srs = Srs + Srs.T
    for k, S in (("Srr", Srr), ("Sss", Sss), ("Srs", Srs)):
        assert np.abs(T[k] - S).max() < 1e-9 * np.abs(S).max(), k
        assert np.abs(T[k] - T[k].T).max() == 0.0 or np.abs(T[k] - T[k].T).max() < 1e-14 * np.abs(S).max()
        assert np.abs(T[k].sum(axis=1)).max() < 1e-12 * np.abs(S).max()  # derivatives of sum N = 1 vanish
    M2 = np.einsum("pij,pij,ij->p", val, val, W)
    assert np.abs(T["wM"] - M2 * 0.5 / M2.sum()).max() < 1e-12
    assert (T["wM"] > 0).all() and abs(T["wM"].sum() - 0.5) < 1e-15
