"""Pins for the oracle's Heun scheme on (U, V) -- the paper's own integrator
(PAPER.md:269-291 with Algorithms 1-3).

Independent anchors:
* Algorithm 1 reproduces c^2 grad(u) exactly for a linear u on a non-symmetric
  Jacobian (reading R5);
* Algorithm 2 of a constant V: zero at interior nodes (div of a constant) and
  zero total (partition of unity);
* Algorithm 2 o Algorithm 1 = -K with K the direct-quadrature stiffness of the
  leapfrog pins (north_star reading R1);
* one Heun step from zero has a closed form; zero source stays zero;
* second order in time (error ratio ~4 when h halves) and agreement
  with the leapfrog to O(h^2);
* the semi-discrete energy 1/2 U'MU + 1/2 sum detJ w |V|^2 / c^2 is conserved
  by the ODE; Heun's drift shrinks >= 3x when h halves.
"""
import math

import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg


def ricker(t, f0, t0):
    a = (math.pi * f0 * (t - t0)) ** 2
    return (1 - 2 * a) * math.exp(-a)


@pytest.mark.parametrize("P", [2, 3])
def test_vdot_exact_gradient_linear_field(P):
    m = mg.shuffle(mg.grid_mesh(5, 4, 1.7, 1.0, alpha=0.2, seed=9), 1, 2)
    c = np.linspace(0.7, 2.1, m.ne)
    o = OracleSEM(m.vxy, m.tri, P, c)
    xy = o.node_xy()
    U = 0.3 - 1.1 * xy[:, 0] + 2.4 * xy[:, 1]
    Vd = o.vdot(U)
    expect = np.stack([np.broadcast_to((c ** 2)[:, None] * -1.1, (m.ne, o.Np)),
                       np.broadcast_to((c ** 2)[:, None] * 2.4, (m.ne, o.Np))], axis=2)
    assert np.abs(Vd - expect).max() < 1e-12 * np.abs(expect).max()


@pytest.mark.parametrize("P", [2, 3])
def test_rv_constant_field(P):
    m = mg.grid_mesh(6, 5, 1.2, 1.0, alpha=0.2, seed=3)
    o = OracleSEM(m.vxy, m.tri, P)
    V = np.zeros((m.ne, o.Np, 2))
    V[..., 0] = 0.7
    V[..., 1] = -1.3
    R = o.rv(V)
    xy = o.node_xy()
    tol = 1e-9
    interior = (xy[:, 0] > tol) & (xy[:, 0] < 1.2 - tol) & (xy[:, 1] > tol) & (xy[:, 1] < 1.0 - tol)
    assert np.abs(R[interior]).max() < 1e-13
    assert abs(R.sum()) < 1e-13
    assert np.abs(R[~interior]).max() > 1e-3


@pytest.mark.parametrize("P", [2, 3])
def test_rv_of_vdot_is_minus_K(P):
    m = mg.shuffle(mg.grid_mesh(5, 5, 1.0, 1.0, alpha=0.2, seed=4), 5, 6)
    o = OracleSEM(m.vxy, m.tri, P, np.linspace(1.0, 3.0, m.ne))
    U = np.random.default_rng(0).standard_normal(o.N)
    a = o.rv(o.vdot(U))
    b = o.apply_R(U)
    assert np.abs(a - b).max() < 1e-12 * np.abs(b).max()


def test_one_heun_step_from_zero_closed_form():
    pb = mg.config("C1", scale=4)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    h, s = pb.dt, pb.src_vertex
    U, V = o.heun(h, 1, src=s, A=2.0, f0=pb.f0, t0=0.05)
    y0, y1 = 2.0 * ricker(0.0, pb.f0, 0.05), 2.0 * ricker(h, pb.f0, 0.05)
    expect = np.zeros(o.N)
    expect[s] = h / 2.0 * (y0 + y1) / o.Mbar[s]
    assert np.abs(U - expect).max() <= 1e-15 * abs(expect[s])
    e = np.zeros(o.N)
    e[s] = 1.0
    Vexp = h * h / 2.0 * (y0 / o.Mbar[s]) * o.vdot(e)
    assert np.abs(V - Vexp).max() <= 1e-13 * np.abs(Vexp).max()
    U0, V0 = o.heun(h, 30, src=s, A=0.0, f0=pb.f0, t0=0.05)
    assert (U0 == 0).all() and (V0 == 0).all()


def _mode_problem(P, n=8):
    m = mg.grid_mesh(n, n, 1.0, 1.0, alpha=0.2, seed=11)
    o = OracleSEM(m.vxy, m.tri, P)
    xy = o.node_xy()
    U0 = np.cos(np.pi * xy[:, 0]) * np.cos(np.pi * xy[:, 1])
    return o, U0


def _lam_max(o, iters=200):
    x = np.random.default_rng(0).standard_normal(o.N)
    for _ in range(iters):
        y = o.apply_K(x) / o.Mbar
        x = y / np.linalg.norm(y)
    return float(x @ o.apply_K(x) / (x @ (o.Mbar * x)))


def test_heun_second_order_in_time():
    o, U0 = _mode_problem(3)
    # Heun amplifies imaginary-axis modes by (1 + (w h)^4 / 4)^(1/2) per step
    # ("sufficiently small time steps"): keep w_max h <= 0.2
    h1 = 0.2 / math.sqrt(_lam_max(o))
    T = 40 * h1
    sol = {}
    for k in (40, 80, 160, 2560):
        U, _ = o.heun(T / k, k, U=U0)
        sol[k] = U
    e1 = np.linalg.norm(sol[40] - sol[2560])
    e2 = np.linalg.norm(sol[80] - sol[2560])
    e3 = np.linalg.norm(sol[160] - sol[2560])
    assert 3.0 < e1 / e2 < 5.0 and 3.0 < e2 / e3 < 5.0


def test_heun_agrees_with_leapfrog_to_second_order():
    o, U0 = _mode_problem(2)
    T = 60 * 0.2 / math.sqrt(_lam_max(o))
    d = []
    for k in (40, 80):
        Uh, _ = o.heun(T / k, k, U=U0)
        # leapfrog started consistently: U^{-1} from a Taylor step (V = 0 => U' = 0)
        h = T / k
        Um1 = U0 + 0.5 * h * h * (-o.apply_K(U0) / o.Mbar)  # U(-h) = U0 + h^2/2 U''(0)
        Ul, _ = o.leapfrog(h, k, U=U0, Uprev=Um1)
        d.append(np.linalg.norm(Uh - Ul) / np.linalg.norm(Ul))
    assert d[0] < 1e-3 and 3.0 < d[0] / d[1] < 5.5


def test_heun_energy_drift_shrinks():
    o, U0 = _mode_problem(3, n=6)

    def energy(U, V):
        eV = (o.detJ[:, None] * o.wK[None, :] * (V ** 2).sum(axis=2) / (o.c[:, None] ** 2)).sum()
        return 0.5 * (U @ (o.Mbar * U)) + 0.5 * eV

    E0 = energy(U0, np.zeros((o.ne, o.Np, 2)))
    h1 = 0.3 / math.sqrt(_lam_max(o))
    drifts = []
    for k in (100, 200):
        U, V = o.heun(100 * h1 / k, k, U=U0)
        drifts.append(abs(energy(U, V) - E0) / E0)
    assert drifts[0] < 1e-2 and drifts[0] / drifts[1] > 3.0
