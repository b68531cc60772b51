"""NEXT-4 ablation scatters (fp64 atomics, and the paper's global
element colouring of Algorithm 2) against the oracle.  Both are
alternatives to the product path's chunk-owned scatter; the field must match
the oracle within rel L2 1e-10.  The colour scatter is deterministic (bitwise
repeatable), which also shows the colouring is conflict-free."""
import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu


@pytest.fixture()
def ctx():
    c = S.SemContext(0)
    yield c
    c.close()


def run(ctx, pb, mode, steps, f0, t0, elem_order=S.SEM_ORDER_HILBERT):
    m = pb.mesh
    ctx.sem_set_scatter(mode)
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, S.SEM_NODES_FIRST_TOUCH)
    ctx.sem_build_operators(pb.c, pb.src_vertex, f0, t0, 1.0, pb.dt)
    ctx.sem_step_n(steps)
    U, n = ctx.sem_read_field()
    assert n == steps
    return U, ctx.sem_get_info()


@pytest.mark.parametrize("mode", [S.SEM_SCATTER_ATOMIC, S.SEM_SCATTER_COLOR])
@pytest.mark.parametrize("name,scale,steps", [("C1", 1, 200), ("C2", 16, 120), ("C5", 256, 100)])
def test_ablation_parity(ctx, mode, name, scale, steps):
    pb = mg.config(name, scale)
    f0, t0 = 1.0 / (8 * pb.dt), 10 * pb.dt
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=f0, t0=t0)
    Ug, info = run(ctx, pb, mode, steps, f0, t0)
    assert info["scatter"] == mode
    if mode == S.SEM_SCATTER_COLOR:
        assert info["n_global_colors"] >= 3 and info["launches_per_step"] == info["n_global_colors"] + 1
    assert np.linalg.norm(Ug - Uo) / np.linalg.norm(Uo) <= 1e-10


def test_color_scatter_bitwise_repeatable(ctx):
    pb = mg.config("C2", 8)
    f0, t0 = 1.0 / (8 * pb.dt), 10 * pb.dt
    a, _ = run(ctx, pb, S.SEM_SCATTER_COLOR, 60, f0, t0, S.SEM_ORDER_RANDOM)
    b, _ = run(ctx, pb, S.SEM_SCATTER_COLOR, 60, f0, t0, S.SEM_ORDER_RANDOM)
    assert np.array_equal(a, b)


def test_ablation_errors(ctx):
    with pytest.raises(S.SemError) as e:
        ctx.sem_set_scatter(9)
    assert e.value.status == S.SEM_E_UNSUPPORTED
    pb = mg.config("C1", 4)
    ctx.sem_set_scatter(S.SEM_SCATTER_ATOMIC)
    ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P)
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
    with pytest.raises(S.SemError) as e:
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    assert e.value.status == S.SEM_E_UNSUPPORTED
