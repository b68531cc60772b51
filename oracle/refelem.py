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
    raise ValueError("unsupported order %r (oracle supports P = 1, 2, 3)" % P)


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
    """fp64 tables (rounded once from exact values).

    Returns dict with numpy arrays:
      nodes [Np,2], wK [Np], wM [Np], Dr [Np,Np], Ds [Np,Np]  (Dr[k,p] = dN_p/dr at x_k)
    """
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


def n_nodes(P: int) -> int:
    return (P + 1) * (P + 2) // 2
