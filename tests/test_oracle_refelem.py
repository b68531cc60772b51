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
