"""GPU parity of the paper's Heun integrator (NEXT-1; PAPER.md:269-291 with
Algorithms 1-3) against the oracle's orc_heun, through the C ABI.

Bars: U and V within relative L2 <= 1e-10 after the run (north_star tolerance);
one- and ten-step parity from seeded random (U, V) states <= 1e-12 (P-12 analog:
every element's F, sd and mu row matters, not only those near the source).
The GPU folds the predictor-corrector into one pass (heun.cu header); the
oracle follows the paper's two RHS evaluations literally.
"""
import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu

REL_L2 = 1e-10
REL_STATE = 1e-12


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    c = S.SemContext(0)
    yield c
    c.close()


def setup_gpu(ctx, pb, h, mesh=None, c=None, src=None, elem_order=S.SEM_ORDER_HILBERT,
              node_order=S.SEM_NODES_FIRST_TOUCH, f0=None, t0=None):
    m = pb.mesh if mesh is None else mesh
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, node_order, seed=11)
    ctx.sem_build_operators(pb.c if c is None else c, pb.src_vertex if src is None else src,
                            pb.f0 if f0 is None else f0, pb.t0 if t0 is None else t0, pb.amplitude, h)
    assert ctx.sem_get_info()["integrator"] == S.SEM_INTEGRATOR_HEUN


def shifted(pb, h):
    """Source peak moved to t0 = 10 h with f0 = 1/(8h) so short runs carry a field."""
    return 1.0 / (8 * h), 10 * h


@pytest.mark.parametrize("name,scale,steps", [("C1", 1, 200), ("C2", 16, 150), ("C3", 40, 120),
                                              ("C4", 64, 120), ("C5", 256, 100)])
def test_heun_run_parity(ctx, name, scale, steps):
    pb = mg.config(name, scale)
    h = mg.heun_h(pb)
    f0, t0 = shifted(pb, h)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=pb.amplitude, f0=f0, t0=t0)
    setup_gpu(ctx, pb, h, f0=f0, t0=t0)
    ctx.sem_step_n(steps)
    Ug, n = ctx.sem_read_field()
    Vg, n2 = ctx.sem_read_velocity()
    assert n == steps and n2 == steps
    assert np.abs(Uo).max() > 0 and np.abs(Vo).max() > 0
    assert rel_l2(Ug, Uo) <= REL_L2, rel_l2(Ug, Uo)
    assert rel_l2(Vg, Vo) <= REL_L2, rel_l2(Vg, Vo)


@pytest.mark.parametrize("name,scale,B_ragged", [("C2", 16, True), ("C1", 1, True), ("C3", 40, False)])
@pytest.mark.parametrize("steps", [1, 10])
def test_heun_random_state_parity(ctx, name, scale, B_ragged, steps):
    pb = mg.config(name, scale)
    m = pb.mesh
    if B_ragged:  # element count not a multiple of the chunk size
        nat = mg.grid_mesh(45, 37, 1.0, 0.8, alpha=0.2, seed=21)
        m = mg.shuffle(nat, 22, 23)
        pb = mg.Problem(**{**pb.__dict__, "mesh": m, "c": np.linspace(0.8, 1.6, m.ne),
                           "src_vertex": mg.source_vertex(m), "dt": mg.cfl_dt(m, np.full(m.ne, 1.6), pb.P)})
    h = mg.heun_h(pb)
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(5)
    U0 = rng.standard_normal(o.N)
    V0 = rng.standard_normal((m.ne, o.Np, 2))
    Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=3.0, f0=pb.f0, t0=0.0, U=U0, V=V0, step0=4)
    setup_gpu(ctx, pb, h, f0=pb.f0, t0=0.0)
    ctx2 = ctx
    # amplitude 3 through a rebuilt source
    ctx2.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 3.0, h)
    ctx2.sem_write_state(U0, None)
    ctx2.sem_write_velocity(V0)
    ctx2.sem_set_step(4)
    ctx2.sem_step_n(steps)
    Ug, _ = ctx2.sem_read_field()
    Vg, _ = ctx2.sem_read_velocity()
    assert rel_l2(Ug, Uo) <= REL_STATE, rel_l2(Ug, Uo)
    assert rel_l2(Vg, Vo) <= REL_STATE, rel_l2(Vg, Vo)


def test_heun_velocity_roundtrip_and_midrun_readout_is_bitwise(ctx):
    pb = mg.config("C2", 16)
    h = mg.heun_h(pb)
    f0, t0 = shifted(pb, h)
    setup_gpu(ctx, pb, h, f0=f0, t0=t0)
    V0 = np.random.default_rng(1).standard_normal((pb.mesh.ne, 10, 2))
    ctx.sem_write_velocity(V0)
    Vr, _ = ctx.sem_read_velocity()
    assert np.array_equal(Vr, V0)
    ctx.sem_step_n(30)
    Ua, _ = ctx.sem_read_field()
    Va, _ = ctx.sem_read_velocity()
    setup_gpu(ctx, pb, h, f0=f0, t0=t0)
    ctx.sem_write_velocity(V0)
    ctx.sem_step_n(12)
    ctx.sem_read_velocity()  # finalises the lagged V update mid-run
    ctx.sem_step_n(18)
    Ub, _ = ctx.sem_read_field()
    Vb, _ = ctx.sem_read_velocity()
    assert np.array_equal(Ua, Ub) and np.array_equal(Va, Vb)


@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
                                                   (S.SEM_ORDER_RANDOM, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_HILBERT, S.SEM_NODES_CANONICAL)])
def test_heun_orderings_same_field(ctx, elem_order, node_order):
    pb = mg.config("C1", 2)
    h = mg.heun_h(pb)
    f0, t0 = shifted(pb, h)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, Vo = o.heun(h, 80, src=pb.src_vertex, A=1.0, f0=f0, t0=t0)
    setup_gpu(ctx, pb, h, elem_order=elem_order, node_order=node_order, f0=f0, t0=t0)
    ctx.sem_step_n(80)
    Ug, _ = ctx.sem_read_field()
    Vg, _ = ctx.sem_read_velocity()
    assert rel_l2(Ug, Uo) <= REL_L2 and rel_l2(Vg, Vo) <= REL_L2


def test_heun_zero_source_stays_zero_and_errors(ctx):
    pb = mg.config("C1", 4)
    h = mg.heun_h(pb)
    setup_gpu(ctx, pb, h, src=-1)
    ctx.sem_step_n(25)
    U, _ = ctx.sem_read_field()
    V, _ = ctx.sem_read_velocity()
    assert (U == 0).all() and (V == 0).all()
    with pytest.raises(S.SemError) as e:
        ctx.sem_write_state(np.zeros(U.size), np.zeros(U.size))
    assert e.value.status == S.SEM_E_ARG
    with pytest.raises(S.SemError) as e:
        ctx.sem_set_integrator(7)
    assert e.value.status == S.SEM_E_UNSUPPORTED
    # back to the leapfrog: velocity calls are out of state
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_LEAPFROG)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    with pytest.raises(S.SemError) as e:
        ctx.sem_read_velocity()
    assert e.value.status == S.SEM_E_STATE


@pytest.mark.parametrize("world,name,scale,P", [(2, "C2", 8, None), (3, "C1", 1, None), (4, "C3", 20, None),
                                                 (8, "C5", 128, None), (3, "B1", 25, 5), (2, "B1", 30, 7)])
def test_heun_multirank_loopback(ctx, world, name, scale, P):
    """Heun across G partitions (SURVEY §8e with the (R(V), K U) payload, loopback
    transport on one GPU): equal to the oracle (<= 1e-10 after a Ricker run,
    <= 1e-12 from a random state) and to the one-rank run (rounding level)."""
    pb = mg.config(name, scale, degree=P) if P else mg.config(name, scale)
    m = pb.mesh
    h = mg.heun_h(pb)
    f0, t0 = shifted(pb, h)
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    steps = 60
    Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=1.0, f0=f0, t0=t0)
    setup_gpu(ctx, pb, h, f0=f0, t0=t0)
    ctx.sem_step_n(steps)
    U1, _ = ctx.sem_read_field()
    V1, _ = ctx.sem_read_velocity()
    g = S.LoopbackGroup(world)
    try:
        g.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
        g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        assert all(c.sem_get_info()["n_interface_nodes"] > 0 for c in g.ctxs)
        g.sem_build_operators(pb.c, pb.src_vertex, f0, t0, 1.0, h)
        g.sem_step_n(steps // 2)
        g.sem_read_velocity()  # mid-run finalise on every rank
        g.sem_step_n(steps - steps // 2)
        Ug, n = g.sem_read_field()
        Vg, _ = g.sem_read_velocity()
        assert n == steps and not np.isnan(Ug).any() and not np.isnan(Vg).any()
        assert rel_l2(Ug, Uo) <= REL_L2 and rel_l2(Vg, Vo) <= REL_L2
        assert rel_l2(Ug, U1) <= 1e-13 and rel_l2(Vg, V1) <= 1e-13
        # random state, 5 steps
        rng = np.random.default_rng(world)
        U0, V0 = rng.standard_normal(o.N), rng.standard_normal((m.ne, o.Np, 2))
        Uo, Vo = o.heun(h, 5, src=pb.src_vertex, A=1.0, f0=f0, t0=t0, U=U0, V=V0, step0=9)
        g.sem_write_state(U0, None)
        g.sem_write_velocity(V0)
        g.sem_set_step(9)
        g.sem_step_n(5)
        Ug, _ = g.sem_read_field()
        Vg, _ = g.sem_read_velocity()
        assert rel_l2(Ug, Uo) <= REL_STATE and rel_l2(Vg, Vo) <= REL_STATE
    finally:
        g.close()


@pytest.mark.parametrize("P", [5, 7])
@pytest.mark.parametrize("steps", [1, 10, 60])
def test_heun_p5_parity(ctx, steps, P):
    """The paper's Benchmark 1 orders 5 and 7 with its own
    integrator (P7: 4 threads per element, chunks of 64)."""
    pb = mg.config("B1", 30, degree=P)  # 33 x 16 cells: ragged last chunk of 128 / 64
    m = pb.mesh
    h = mg.heun_h(pb)
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(steps)
    U0 = rng.standard_normal(o.N)
    V0 = rng.standard_normal((m.ne, o.Np, 2))
    f0, t0 = shifted(pb, h)
    Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=1.0, f0=f0, t0=t0, U=U0, V=V0)
    setup_gpu(ctx, pb, h, f0=f0, t0=t0)
    ctx.sem_write_state(U0, None)
    ctx.sem_write_velocity(V0)
    ctx.sem_step_n(steps)
    Ug, _ = ctx.sem_read_field()
    Vg, _ = ctx.sem_read_velocity()
    tol = REL_STATE if steps <= 10 else REL_L2
    assert rel_l2(Ug, Uo) <= tol, rel_l2(Ug, Uo)
    assert rel_l2(Vg, Vo) <= tol, rel_l2(Vg, Vo)
