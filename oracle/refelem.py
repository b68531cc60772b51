"""Exact reference-triangle tables for the oracle (TEST INFRASTRUCTURE ONLY).

Everything here is computed symbolically with sympy (rationals and sqrt(5))
and rounded to fp64 exactly once, at the very end (``tables()``).

Paper passages followed
-----------------------
* PAPER.md:163-171 (eq. x = x^(e) + J x^): reference triangle (0,0),(1,0),(0,1).
* PAPER.md:173-177 (eq. dual_sys): nodal basis N_p(x_q) = delta_pq.
* "the local nodes ... are also quadrature points".
* PAPER.md:220-225 (eq. numerical_integ): int f ~= sum_q w_q f(x_q); with the
  nodal basis this forces w_q = int N_q (exactness for the basis itself).
* PAPER.md:195-206 (eq. deriv_u): derivatives of the nodal basis.

Readings:
* R3  node sets: P2 = vertices + edge midpoints; P3 = vertices + Gauss-Lobatto
      edge points (1 -/+ 1/sqrt5)/2 + centroid.  Local order = lattice order
      (row j = 0..P outer, i = 0..P-j inner).          -- parity unpinned (R3)
* R4  stiffness weights w^K = int N (paper); mass weights w^M = w^K for P3 and
      the HRZ-lumped diagonal for P2 (w^K has zero vertex weights for P2, which
      makes M-bar singular).                            -- HRZ parity unpinned
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np
import sympy as sp

X, Y = sp.symbols("x y", real=True)


def _lobatto_a():
    # Interior Gauss-Lobatto point of the 4-point rule on [0, 1].
    return (1 - 1 / sp.sqrt(5)) / 2


@lru_cache(maxsize=None)
def nodes(P: int):
    """Local nodes x^_p in lattice order (reading R3)."""
    if P == 1:
        return ((sp.Integer(0), sp.Integer(0)), (sp.Integer(1), sp.Integer(0)),
                (sp.Integer(0), sp.Integer(1)))
    if P == 2:
        h = sp.Rational(1, 2)
        return ((0, 0), (h, 0), (1, 0), (0, h), (h, h), (0, 1))
    if P == 3:
        a = _lobatto_a()
        t = sp.Rational(1, 3)
        return ((0, 0), (a, 0), (1 - a, 0), (1, 0),
                (0, a), (t, t), (1 - a, a),
                (0, 1 - a), (a, 1 - a),
                (0, 1))
    raise ValueError("exact node set only for P <= 3; P >= 4 uses tables_hp (reading R21)")


def monomials(P: int):
    return [X**a * Y**b for a in range(P + 1) for b in range(P + 1 - a)]


@lru_cache(maxsize=None)
def basis(P: int):
    """Nodal basis N_p (sympy expressions) solving the dual system (eq. dual_sys)."""
    nd = nodes(P)
    mons = monomials(P)
    V = sp.Matrix([[m.subs({X: x, Y: y}) for m in mons] for (x, y) in nd])
    C = V.inv()  # column p = coefficients of N_p
    return tuple(sp.expand(sp.simplify(sum(C[m, p] * mons[m] for m in range(len(mons)))))
                 for p in range(len(nd)))


def integrate_ref(f):
    """Exact integral over the reference triangle."""
    return sp.nsimplify(sp.integrate(sp.integrate(f, (Y, 0, 1 - X)), (X, 0, 1)))


@lru_cache(maxsize=None)
def weights_K(P: int):
    """w_q = int N_q  (nodes double as quadrature points, eq. numerical_integ)."""
    return tuple(sp.simplify(integrate_ref(N)) for N in basis(P))


@lru_cache(maxsize=None)
def weights_M(P: int):
    """Mass (lumping) weights: w^K for P1/P3, HRZ for P2 (reading R4)."""
    if P != 2:
        return weights_K(P)
    diag = [sp.simplify(integrate_ref(N * N)) for N in basis(P)]
    total = sum(diag)
    return tuple(sp.simplify(d * sp.Rational(1, 2) / total) for d in diag)


@lru_cache(maxsize=None)
def deriv_tables(P: int):
    """Dr[k][p] = dN_p/dx^_0 at node k;  Ds[k][p] = dN_p/dx^_1 at node k."""
    nd = nodes(P)
    B = basis(P)
    Dr = [[sp.simplify(sp.diff(B[p], X).subs({X: x, Y: y})) for p in range(len(nd))] for (x, y) in nd]
    Ds = [[sp.simplify(sp.diff(B[p], Y).subs({X: x, Y: y})) for p in range(len(nd))] for (x, y) in nd]
    return Dr, Ds


def _f64(e) -> float:
    return float(sp.N(e, 50))


@lru_cache(maxsize=None)
def tables(P: int):
    """fp64 tables (rounded once from exact values; P >= 4: tables_hp).

    Returns dict with numpy arrays:
      nodes [Np,2], wK [Np], wM [Np], Dr [Np,Np], Ds [Np,Np]  (Dr[k,p] = dN_p/dr at x_k)
    """
    if P >= 4:
        return tables_hp(P)
    nd = nodes(P)
    Dr, Ds = deriv_tables(P)
    out = {
        "P": P,
        "Np": len(nd),
        "nodes": np.array([[_f64(x), _f64(y)] for (x, y) in nd], dtype=np.float64),
        "wK": np.array([_f64(w) for w in weights_K(P)], dtype=np.float64),
        "wM": np.array([_f64(w) for w in weights_M(P)], dtype=np.float64),
        "Dr": np.array([[_f64(v) for v in row] for row in Dr], dtype=np.float64),
        "Ds": np.array([[_f64(v) for v in row] for row in Ds], dtype=np.float64),
    }
    for k in ("nodes", "wK", "wM", "Dr", "Ds"):
        out[k].setflags(write=False)
    return out


# --------------------------------------------------------------------------
# P >= 4 (NEXT-2, reading R21): Blyth-Pozrikidis Lobatto grid, computed in
# 60-digit arithmetic (mpmath) and rounded to fp64 once.  The 1D master nodes
# v_0..v_P are the Gauss-Lobatto points on [0, 1] (0, 1 and the roots of
# P_P'(2v - 1)); the triangle node of lattice indices (i, j), k = P - i - j, is
#   x = (1 + 2 v_i - v_j - v_k) / 3,   y = (1 + 2 v_j - v_i - v_k) / 3
# (Blyth & Pozrikidis 2006; for P = 2, 3 it gives the R3 node sets above).
# The paper cites these locations without printing them:
# parity unpinned beyond the invariants of tests/test_oracle_refelem.py.
# Reading R21b: for P = 4, 6 the nodal weights int N_p are negative at the
# vertices, so the nodes cannot serve as the quadrature (lumped mass not
# positive); these orders use the consistent stiffness S_ab = int dN/da dN/db
# (exact, monomial integrals) and the HRZ-lumped mass, like P2's mass (R4).
# --------------------------------------------------------------------------
HP_DPS = 60


def lobatto01_hp(P: int):
    """Gauss-Lobatto points on [0, 1] (mpmath, HP_DPS digits), ascending."""
    import mpmath as mp
    mp.mp.dps = HP_DPS
    leg = sp.legendre_poly(P, X)
    dpoly = sp.Poly(sp.diff(leg, X), X)
    roots = sorted(sp.Float(r, HP_DPS) for r in dpoly.nroots(n=HP_DPS, maxsteps=200))
    v = [mp.mpf(0)] + [(mp.mpf(str(r)) + 1) / 2 for r in roots] + [mp.mpf(1)]
    for i in range(P // 2 + 1):  # exact symmetry v_{P-i} = 1 - v_i (roots come in +- pairs)
        v[P - i] = 1 - v[i]
    if P % 2 == 0:
        v[P // 2] = mp.mpf(1) / 2
    return v


def nodes_hp(P: int):
    import mpmath as mp
    v = lobatto01_hp(P)
    out = []
    for j in range(P + 1):
        for i in range(P + 1 - j):
            k = P - i - j
            x = mp.mpf(0) if i == 0 else (1 + 2 * v[i] - v[j] - v[k]) / 3  # edges x = 0, y = 0 exact
            y = mp.mpf(0) if j == 0 else (1 + 2 * v[j] - v[i] - v[k]) / 3
            out.append((x, y))
    return out


@lru_cache(maxsize=None)
def tables_hp(P: int):
    """fp64 tables for any P (same keys as ``tables``) from the HP_DPS-digit
    dual-system solve: N_p = sum_m C[m, p] x^a y^b with V C = I; w_p = int N_p
    (closed-form monomial integrals a! b! / (a+b+2)!); Dr[k, p] = dN_p/dx (x_k)."""
    import mpmath as mp
    from math import factorial
    mp.mp.dps = HP_DPS
    nd = nodes_hp(P)
    Np = len(nd)
    ex = [(a, b) for a in range(P + 1) for b in range(P + 1 - a)]
    V = mp.matrix([[x ** a * y ** b for (a, b) in ex] for (x, y) in nd])
    C = mp.inverse(V)  # C[m, p]
    mint = [mp.mpf(factorial(a) * factorial(b)) / factorial(a + b + 2) for (a, b) in ex]
    w = [mp.fsum(C[m, p] * mint[m] for m in range(Np)) for p in range(Np)]

    def dN(p, x, y, d):
        acc = []
        for m, (a, b) in enumerate(ex):
            if d == 0 and a > 0:
                acc.append(C[m, p] * a * x ** (a - 1) * y ** b)
            if d == 1 and b > 0:
                acc.append(C[m, p] * b * x ** a * y ** (b - 1))
        return mp.fsum(acc)

    Dr = [[dN(p, x, y, 0) for p in range(Np)] for (x, y) in nd]
    Ds = [[dN(p, x, y, 1) for p in range(Np)] for (x, y) in nd]

    consistent = any(q <= 0 for q in w)  # P = 4, 6: reading R21b
    if consistent:
        # exact element matrices of the nodal basis: int N_p N_q (HRZ mass) and
        # int dN_p/da dN_q/db (consistent stiffness), monomial by monomial
        def mono(a, b):
            return mp.mpf(factorial(a) * factorial(b)) / factorial(a + b + 2)

        def grad_terms(p, d):  # derivative of N_p along d as (coef, a, b) terms
            out = []
            for m, (a, b) in enumerate(ex):
                if d == 0 and a > 0:
                    out.append((C[m, p] * a, a - 1, b))
                if d == 1 and b > 0:
                    out.append((C[m, p] * b, a, b - 1))
            return out

        def integ(t1, t2):
            return mp.fsum(c1 * c2 * mono(a1 + a2, b1 + b2) for (c1, a1, b1) in t1 for (c2, a2, b2) in t2)

        gr = [grad_terms(p, 0) for p in range(Np)]
        gs = [grad_terms(p, 1) for p in range(Np)]
        vals = [[(C[m, p], a, b) for m, (a, b) in enumerate(ex)] for p in range(Np)]
        M2 = [integ(vals[p], vals[p]) for p in range(Np)]
        tot = mp.fsum(M2)
        wM = [q / (2 * tot) for q in M2]  # HRZ: the consistent diagonal rescaled to area 1/2
        Srr = [[integ(gr[p], gr[q]) for q in range(Np)] for p in range(Np)]
        Sss = [[integ(gs[p], gs[q]) for q in range(Np)] for p in range(Np)]
        Srs = [[integ(gr[p], gs[q]) + integ(gs[p], gr[q]) for q in range(Np)] for p in range(Np)]
    def f(q):  # round once; |q| < 1e-40 is the 60-digit residue of an exact zero
        return 0.0 if abs(q) < mp.mpf("1e-40") else float(q)

    out = {
        "P": P,
        "Np": Np,
        "nodes": np.array([[f(x), f(y)] for (x, y) in nd], dtype=np.float64),
        "wK": np.array([f(q) for q in w], dtype=np.float64),
        "wM": np.array([f(q) for q in (wM if consistent else w)], dtype=np.float64),
        "Dr": np.array([[f(q) for q in row] for row in Dr], dtype=np.float64),
        "Ds": np.array([[f(q) for q in row] for row in Ds], dtype=np.float64),
        "C": C, "exps": ex,  # high-precision basis (pins only)
        "consistent": consistent,
    }
    keys = ["nodes", "wK", "wM", "Dr", "Ds"]
    if consistent:
        for k, M in (("Srr", Srr), ("Sss", Sss), ("Srs", Srs)):
            out[k] = np.array([[f(q) for q in row] for row in M], dtype=np.float64)
            keys.append(k)
    for k in keys:
        out[k].setflags(write=False)
    return out


def n_nodes(P: int) -> int:
    return (P + 1) * (P + 2) // 2
