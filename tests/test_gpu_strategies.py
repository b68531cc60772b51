"""GPU parity of the paper's other reordering strategies (NEXT-3): Conn. / Dist.
(reading R20) and the degree-sorted node renumbering
(reading R12).  Element and node permutations bit-exact
against the oracle; the field is ordering-invariant (rel L2 <= 1e-10)."""
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


def oracle_orders(m, P, elem_order, node_order):
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, P)
    npm = None
    if elem_order == S.SEM_ORDER_CONN:
        ep, npm = core.strategy_order(mu, N, core.conn_key(mu, N))
    elif elem_order == S.SEM_ORDER_DIST:
        ep, npm = core.strategy_order(mu, N, core.dist_key(m.vxy, t, mu, P))
    elif elem_order == S.SEM_ORDER_HILBERT:
        _, ep, _ = core.hilbert_order(m.vxy, m.tri)
    else:
        ep = np.arange(m.ne, dtype=np.int32)
    if node_order == S.SEM_NODES_FIRST_TOUCH:
        npm, _ = core.first_touch(mu[ep], N)
    elif node_order == S.SEM_NODES_FIRST_TOUCH_DEGREE:
        npm, _ = core.first_touch_degree(mu[ep], N)
    elif node_order == S.SEM_NODES_CANONICAL:
        npm = np.arange(N, dtype=np.int32)
    return ep, npm


COMBOS = [(S.SEM_ORDER_CONN, S.SEM_NODES_VISIT), (S.SEM_ORDER_DIST, S.SEM_NODES_VISIT),
          (S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH_DEGREE), (S.SEM_ORDER_CONN, S.SEM_NODES_FIRST_TOUCH),
          (S.SEM_ORDER_DIST, S.SEM_NODES_FIRST_TOUCH_DEGREE), (S.SEM_ORDER_INPUT, S.SEM_NODES_FIRST_TOUCH_DEGREE)]


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C2", 16), ("C3", 40), ("C5", 256)])
@pytest.mark.parametrize("elem_order,node_order", COMBOS)
def test_strategy_permutations_bit_exact(ctx, name, scale, elem_order, node_order):
    pb = mg.config(name, scale)
    m = pb.mesh
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, node_order)
    ep, npm = oracle_orders(m, pb.P, elem_order, node_order)
    assert np.array_equal(r["elem_perm"], ep)
    assert np.array_equal(r["node_perm"], npm)


@pytest.mark.parametrize("elem_order,node_order", COMBOS[:3])
def test_strategy_field_parity(ctx, elem_order, node_order):
    pb = mg.config("C2", 16)
    m = pb.mesh
    f0, t0 = 1.0 / (8 * pb.dt), 10 * pb.dt
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, 100, src=pb.src_vertex, A=1.0, f0=f0, t0=t0)
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, node_order)
    ctx.sem_build_operators(pb.c, pb.src_vertex, f0, t0, 1.0, pb.dt)
    ctx.sem_step_n(100)
    Ug, _ = ctx.sem_read_field()
    assert np.linalg.norm(Ug - Uo) / np.linalg.norm(Uo) <= 1e-10


def test_visit_needs_strategy(ctx):
    pb = mg.config("C1", 4)
    with pytest.raises(S.SemError) as e:
        ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_VISIT)
    assert e.value.status == S.SEM_E_UNSUPPORTED


@pytest.mark.parametrize("P", [3, 7])
@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_CONN, S.SEM_NODES_VISIT),
                                                   (S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH_DEGREE)])
def test_high_valence_fan(ctx, P, elem_order, node_order):
    """A vertex held by 48 elements: more than 32 entries in one chunk (round 1's limit) and,
    at P7, more distinct neighbours than the node-graph kernel's local list (the rescan path).
    Permutations bit-exact; five steps from a random state within 1e-12 of the oracle."""
    m = mg.fan_mesh(48)
    c = np.full(m.ne, 1.0)
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, P, elem_order, node_order)
    ep, npm = oracle_orders(m, P, elem_order, node_order)
    assert np.array_equal(r["elem_perm"], ep)
    assert np.array_equal(r["node_perm"], npm)
    o = OracleSEM(m.vxy, m.tri, P, c)
    dt = mg.cfl_dt(m, c, P)
    rng = np.random.default_rng(P)
    U0, Up = rng.standard_normal(o.N), rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(dt, 5, src=0, A=1.0, f0=2.0, t0=0.0, U=U0, Uprev=Up)
    ctx.sem_build_operators(c, 0, 2.0, 0.0, 1.0, dt)
    ctx.sem_write_state(U0, Up)
    ctx.sem_step_n(5)
    Ug, _ = ctx.sem_read_field()
    assert np.linalg.norm(Ug - Uo) <= 1e-12 * np.linalg.norm(Uo)
