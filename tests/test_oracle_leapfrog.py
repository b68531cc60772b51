"""Pins for the oracle's time stepping (north_star leapfrog; reading R1).

* discrete leapfrog energy  1/2 |(U^{n+1}-U^n)/dt|^2_M + 1/2 U^{n+1}' K U^n
  is conserved without a source (a property of the scheme, SURVEY P-9);
* one step from zero: U^1 = dt^2 A r(0) / Mbar_s e_s (closed form);
* output linear in the amplitude; zero source -> identically zero;
* relabelling invariance: the same physical mesh under a shuffled, natural or
  SFC+first-touch labelling gives the same field;
* Ricker closed-form values.
"""
import math

import numpy as np
import pytest

from oracle import core
from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg


def _ricker(t, f0, t0):
    a = (math.pi * f0 * (t - t0)) ** 2
    return (1 - 2 * a) * math.exp(-a)


def test_ricker_values():
    assert core.ricker(0.3, 10.0, 0.3) == 1.0
    assert abs(core.ricker(0.3 + 0.013, 10.0, 0.3) - core.ricker(0.3 - 0.013, 10.0, 0.3)) < 1e-15
    tau = 1.0 / (math.pi * 10.0)
    assert abs(core.ricker(0.3 + tau, 10.0, 0.3) - (-2.0 * math.exp(-1.0) + math.exp(-1.0))) < 1e-15


def _lam_max(o, iters=300):
    x = np.random.default_rng(0).standard_normal(o.N)
    for _ in range(iters):
        y = o.apply_K(x) / o.Mbar
        x = y / np.linalg.norm(y)
    return float(x @ o.apply_K(x) / (x @ (o.Mbar * x)))


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7])
def test_energy_conservation_no_source(P):
    m = mg.shuffle(mg.grid_mesh(6, 5, 1.2, 1.0, alpha=0.2, seed=3), 4, 5)
    o = OracleSEM(m.vxy, m.tri, P, np.linspace(1.0, 2.0, m.ne))
    dt = 0.9 * 2.0 / math.sqrt(_lam_max(o))
    rng = np.random.default_rng(1)
    U = rng.standard_normal(o.N)
    Up = U + 0.01 * rng.standard_normal(o.N)

    def energy(Un1, Un):
        v = (Un1 - Un) / dt
        return 0.5 * (v @ (o.Mbar * v)) + 0.5 * (Un1 @ o.apply_K(Un))

    E0 = energy(U, Up)
    for _ in range(4):
        U, Up = o.leapfrog(dt, 500, U=U, Uprev=Up)
        assert abs(energy(U, Up) - E0) < 1e-11 * abs(E0)


def test_energy_blows_up_above_cfl():
    # sanity of the stability bound used by the input recipe: 1.05 dt_crit diverges
    m = mg.grid_mesh(4, 4, 1.0, 1.0, alpha=0.2, seed=3)
    o = OracleSEM(m.vxy, m.tri, 2)
    dt = 1.05 * 2.0 / math.sqrt(_lam_max(o))
    U = np.random.default_rng(1).standard_normal(o.N)
    U, _ = o.leapfrog(dt, 2000, U=U, Uprev=U)
    assert not np.isfinite(U).all() or np.abs(U).max() > 1e6


def test_one_step_from_zero_closed_form():
    pb = mg.config("C1", scale=4)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    U, Up = o.leapfrog(pb.dt, 1, src=pb.src_vertex, A=2.5, f0=pb.f0, t0=pb.t0)
    expect = np.zeros(o.N)
    expect[pb.src_vertex] = pb.dt ** 2 * 2.5 * _ricker(0.0, pb.f0, pb.t0) / o.Mbar[pb.src_vertex]
    assert np.abs(U - expect).max() <= 1e-15 * abs(expect).max()
    assert (Up == 0).all()


def test_linear_in_amplitude_and_zero_source():
    pb = mg.config("C1", scale=4)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    U1, _ = o.leapfrog(pb.dt, 60, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=0.0)
    U3, _ = o.leapfrog(pb.dt, 60, src=pb.src_vertex, A=3.0, f0=pb.f0, t0=0.0)
    assert np.abs(U3 - 3 * U1).max() < 1e-13 * np.abs(U3).max()
    U0, _ = o.leapfrog(pb.dt, 60, src=pb.src_vertex, A=0.0, f0=pb.f0, t0=0.0)
    assert (U0 == 0).all()


def _vertex_field(pb_mesh, U, nat_nv):
    """Vertex-node values mapped to natural vertex ids."""
    out = np.empty(nat_nv)
    vp = pb_mesh.vert_perm if pb_mesh.vert_perm is not None else np.arange(nat_nv)
    out[vp] = U[: nat_nv]
    return out


def test_relabelling_invariance_natural_shuffled_sfc():
    pb = mg.config("C1", scale=2)
    nat, sh = pb.natural, pb.mesh
    steps = 80
    # natural labelling
    on = OracleSEM(nat.vxy, nat.tri, pb.P, pb.c_natural)
    src_nat = int(sh.vert_perm[pb.src_vertex])
    Un, _ = on.leapfrog(pb.dt, steps, src=src_nat, f0=pb.f0, t0=0.02)
    # shuffled labelling
    os_ = OracleSEM(sh.vxy, sh.tri, pb.P, pb.c)
    Us, _ = os_.leapfrog(pb.dt, steps, src=pb.src_vertex, f0=pb.f0, t0=0.02)
    # SFC element order of the shuffled file (vertex ids unchanged)
    key, perm, grid = core.hilbert_order(sh.vxy, sh.tri)
    oh = OracleSEM(sh.vxy, sh.tri[perm], pb.P, pb.c[perm])
    Uh, _ = oh.leapfrog(pb.dt, steps, src=pb.src_vertex, f0=pb.f0, t0=0.02)
    ref = Un[: nat.nv]
    scale = np.abs(ref).max()
    assert scale > 0
    assert np.abs(_vertex_field(sh, Us, nat.nv) - ref).max() < 1e-12 * scale
    assert np.abs(_vertex_field(sh, Uh, nat.nv) - ref).max() < 1e-12 * scale
    # full node sets agree when matched by coordinates
    for o, U in ((os_, Us), (oh, Uh)):
        a = np.lexsort(np.round(on.node_xy() * 1e9).T[::-1])
        b = np.lexsort(np.round(o.node_xy() * 1e9).T[::-1])
        assert np.abs(U[b] - Un[a]).max() < 1e-12 * scale


def test_first_touch_relabelled_run_matches():
    """Field on (SFC elements, first-touch nodes) mapped back = canonical field."""
    pb = mg.config("C1", scale=2)
    sh = pb.mesh
    o = OracleSEM(sh.vxy, sh.tri, pb.P, pb.c)
    U, _ = o.leapfrog(pb.dt, 50, src=pb.src_vertex, f0=pb.f0, t0=0.02)
    key, perm, grid = core.hilbert_order(sh.vxy, sh.tri)
    node_perm, mu_ft = core.first_touch(o.mu[perm], o.N)
    # mu_ft is a valid relabelling: canonical node of new node k is node_perm[k]
    assert (node_perm[mu_ft] == o.mu[perm]).all()
    assert sorted(node_perm.tolist()) == list(range(o.N))
