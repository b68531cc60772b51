"""GPU parity at the paper's benchmark orders 5-7 and order 4 (NEXT-2;
PAPER.md:572, :746-776; readings R21, R21b): reordering bit-exact, leapfrog field within rel L2
1e-10 of the oracle, random-state steps within 1e-12 (every element's G and mu
row matters), on the Benchmark 1 recipe and the C2 recipe at reduced sizes."""
import numpy as np
import pytest

from oracle import core
from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = S.SemContext(0)
    yield c
    c.close()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("P", [4, 5, 6, 7])
@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_CONN, S.SEM_NODES_VISIT),
                                                   (S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH_DEGREE)])
def test_reorder_bit_exact_high_order(ctx, P, elem_order, node_order):
    pb = mg.config("B1", 25, degree=P)
    m = pb.mesh
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, P, elem_order, node_order)
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, P)
    assert r["n_nodes"] == N
    if elem_order == S.SEM_ORDER_CONN:
        ep, npm = core.strategy_order(mu, N, core.conn_key(mu, N))
    else:
        _, ep, _ = core.hilbert_order(m.vxy, m.tri)
        npm = (core.first_touch if node_order == S.SEM_NODES_FIRST_TOUCH else core.first_touch_degree)(mu[ep], N)[0]
    assert np.array_equal(r["elem_perm"], ep)
    assert np.array_equal(r["node_perm"], npm)


@pytest.mark.parametrize("P", [4, 5, 6, 7])
@pytest.mark.parametrize("name,scale,steps", [("B1", 25, 150), ("C2", 32, 120)])
def test_leapfrog_parity_high_order(ctx, P, name, scale, steps):
    pb = mg.config(name, scale, degree=P) if name == "B1" else mg.config(name, scale)
    m = pb.mesh
    dt = mg.cfl_dt(pb.natural, pb.c_natural, P)
    f0, t0 = 1.0 / (8 * dt), 10 * dt
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    Uo, _ = o.leapfrog(dt, steps, src=pb.src_vertex, A=1.0, f0=f0, t0=t0)
    ctx.sem_mesh_reorder(m.vxy, m.tri, P)
    ctx.sem_build_operators(pb.c, pb.src_vertex, f0, t0, 1.0, dt)
    ctx.sem_step_n(steps)
    Ug, n = ctx.sem_read_field()
    assert n == steps and np.abs(Uo).max() > 0
    assert rel(Ug, Uo) <= 1e-10, rel(Ug, Uo)


@pytest.mark.parametrize("P", [4, 5, 6, 7])
@pytest.mark.parametrize("steps", [1, 10])
def test_random_state_high_order(ctx, P, steps):
    pb = mg.config("B1", 30, degree=P)  # 33 x 16 cells: ragged last chunk at B = 128 and 64
    m = pb.mesh
    assert m.ne % 64 != 0
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(P)
    U, Up = rng.standard_normal(o.N), rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=2.0, f0=pb.f0, t0=0.0, U=U, Uprev=Up, step0=3)
    ctx.sem_mesh_reorder(m.vxy, m.tri, P)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 2.0, pb.dt)
    ctx.sem_write_state(U, Up)
    ctx.sem_set_step(3)
    ctx.sem_step_n(steps)
    Ug, _ = ctx.sem_read_field()
    assert rel(Ug, Uo) <= 1e-12, rel(Ug, Uo)


def test_unsupported_orders(ctx):
    pb = mg.config("B1", 50, degree=5)
    for P in (1, 8):
        with pytest.raises(S.SemError) as e:
            ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, P)
        assert e.value.status == S.SEM_E_UNSUPPORTED
    # Heun needs the nodal quadrature: not at the R21b orders
    for P in (4, 6):
        ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
        ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, P)
        with pytest.raises(S.SemError) as e:
            ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        assert e.value.status == S.SEM_E_UNSUPPORTED
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_LEAPFROG)
