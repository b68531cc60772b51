"""The seeded input recipe (paper_2104_08416_b200/meshgen.py) produces what
DESIGN.md "Input recipe" promises: valid CCW meshes of the configured sizes,
layered speeds, a centred source, and a time step below half the leapfrog
stability limit (checked with the oracle's operator on reduced sizes)."""
import math

import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg


def test_full_size_counts():
    # element counts of BASELINE.json configs (computed from the recipe, not built)
    assert 2 * 32 * 32 == 2048
    assert 2 * 512 * 512 == 524288
    assert 2 * 2000 * 1000 == 4_000_000
    assert 2 * 2048 * 2048 == 8_388_608
    assert 2 * 16384 * 8192 == 268_435_456


def test_c1_exact():
    pb = mg.config("C1")
    assert pb.mesh.ne == 2048 and pb.P == 2 and pb.n_steps == 200
    assert abs(pb.dt - 0.2 * mg.min_edge(pb.natural)) < 1e-18
    # shuffled: elements and vertices permuted, same geometry
    assert not (pb.mesh.elem_perm == np.arange(2048)).all()
    v = pb.mesh.vxy
    assert abs(v[pb.src_vertex] - [0.5, 0.5]).max() < 0.25 / 32 + 1e-12


def _lam_max(o, iters=300):
    x = np.random.default_rng(0).standard_normal(o.N)
    for _ in range(iters):
        y = o.apply_K(x) / o.Mbar
        x = y / np.linalg.norm(y)
    return float(x @ o.apply_K(x) / (x @ (o.Mbar * x)))


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C2", 16), ("C3", 40), ("C4", 64), ("C5", 256)])
def test_dt_below_half_cfl(name, scale):
    pb = mg.config(name, scale)
    m = pb.mesh
    assert (mg._signed_area2(m.vxy, m.tri) > 0).all()
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    dt_crit = 2.0 / math.sqrt(_lam_max(o))
    limit = 0.8 if name == "C1" else 0.5
    assert pb.dt < limit * dt_crit


def test_layers():
    pb = mg.config("C3", 40)
    assert set(np.unique(pb.c).tolist()) == {1500.0, 2500.0, 3500.0}
    cen = mg.centroids(pb.mesh)
    depth = 4000.0 - cen[:, 1]
    assert (pb.c[depth < 1000.0] == 1500.0).all() and (pb.c[depth >= 2500.0] == 3500.0).all()


@pytest.mark.parametrize("P", [4, 5, 6, 7])
def test_b1_dt_below_half_cfl_high_order(P):
    # the Benchmark 1 stand-in at orders 5 and 7 (reading R21 CFL factors)
    pb = mg.config("B1", 50, degree=P)
    assert pb.P == P and pb.mesh.ne == 2 * 20 * 10
    o = OracleSEM(pb.mesh.vxy, pb.mesh.tri, P, pb.c)
    assert pb.dt < 0.5 * 2.0 / math.sqrt(_lam_max(o))
    # with the C2 recipe at P5/P7 too (graded-free jittered square, alpha 0.25)
    pc = mg.config("C2", 32)
    o2 = OracleSEM(pc.mesh.vxy, pc.mesh.tri, P, pc.c)
    assert mg.cfl_dt(pc.natural, pc.c_natural, P) < 0.5 * 2.0 / math.sqrt(_lam_max(o2))
