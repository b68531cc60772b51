"""K7 / KH7 with many chunks per persistent CTA ("What's weak" #2).

The product grid is every SM x the resident CTAs per SM (296 on a B200 at P3), so on the
small meshes the oracle finishes in seconds each CTA sees at most one chunk and the
pipeline's stage recycling (k >= kStages: the `empty` mbarrier waits and parity flips),
the single-buffered U^{n-1} / dt^2/M window hand-off (k >= 1: `wempty`) and the ids
barrier reuse never run.  SEM_K7_GRID caps the persistent grid, so a few-thousand-element
mesh walks 5-69 chunks per CTA -- the same code path the C4 bench times (about 110 chunks per
CTA).  Bars as in test_gpu_parity (P-12): random full-mesh states, rel L2 <= 1e-13 per
step at P2/P3 and <= 1e-12 at P5/P7 against the oracle (Alg. 1+2+3 + leapfrog,
PAPER.md:404-528), plus bitwise equality with the uncapped grid (each node's sums run in
a fixed order whatever CTA processes its chunk).
"""
import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def problem(P):
    # P3: C2 recipe at 64 x 64 cells (8192 elements, 32 chunks of 256); P2: C5 recipe (graded,
    # layered) at 64 x 32 cells (4096 elements, 16 chunks); P5 / P7: the paper's Benchmark 1
    # recipe at 66 x 33 cells (4356 elements: 35 chunks of 128 / 69 of 64, ragged tails)
    if P == 3:
        return mg.config("C2", 8)
    if P == 2:
        return mg.config("C5", 256)
    return mg.config("B1", 15, degree=P)


def gpu_run(pb, steps, U, Up, step0, grid_cap, monkeypatch, A=1.0, t0=0.0):
    if grid_cap:
        monkeypatch.setenv("SEM_K7_GRID", str(grid_cap))
    else:
        monkeypatch.delenv("SEM_K7_GRID", raising=False)
    m = pb.mesh
    with S.SemContext(0) as ctx:
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, t0, A, pb.dt)
        info = ctx.sem_get_info()
        ctx.sem_write_state(U, Up)
        ctx.sem_set_step(step0)
        ctx.sem_step_n(steps)
        Ug, n = ctx.sem_read_field()
    assert n == step0 + steps
    return Ug, info


@pytest.mark.parametrize("P", [2, 3, 5, 7])
@pytest.mark.parametrize("grid_cap", [1, 2, 3])
def test_leapfrog_many_chunks_per_cta(monkeypatch, P, grid_cap):
    pb = problem(P)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(100 + P)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    # 10 steps: stream launches; 40 steps: one 32-step CUDA-graph replay + 8 launches
    for steps in (10, 40):
        Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=2.0, f0=pb.f0, t0=0.0, U=U0, Uprev=Up, step0=5)
        Ug, info = gpu_run(pb, steps, U0, Up, 5, grid_cap, monkeypatch, A=2.0)
        assert info["n_chunks"] >= 4 * grid_cap, info["n_chunks"]  # several chunks per CTA
        tol = (1e-13 if P <= 3 else 1e-12) * steps
        assert rel_l2(Ug, Uo) <= tol, (P, grid_cap, steps, rel_l2(Ug, Uo))
        assert np.abs(Ug - Uo).max() <= 10 * tol * np.abs(Uo).max()
        if grid_cap == 2:
            Ufull, _ = gpu_run(pb, steps, U0, Up, 5, 0, monkeypatch, A=2.0)
            assert np.array_equal(Ug, Ufull)


@pytest.mark.parametrize("P", [2, 3, 5, 7])
@pytest.mark.parametrize("grid_cap", [1, 3])
def test_heun_many_chunks_per_cta(monkeypatch, P, grid_cap):
    monkeypatch.setenv("SEM_K7_GRID", str(grid_cap))
    pb = problem(P)
    m = pb.mesh
    h = mg.heun_h(pb)
    o = OracleSEM(m.vxy, m.tri, P, pb.c)
    rng = np.random.default_rng(7 + P)
    U0 = rng.standard_normal(o.N)
    V0 = rng.standard_normal((m.ne, o.Np, 2))
    for steps in (1, 10):
        Uo, Vo = o.heun(h, steps, src=pb.src_vertex, A=3.0, f0=pb.f0, t0=0.0, U=U0, V=V0, step0=4)
        with S.SemContext(0) as ctx:
            ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
            ctx.sem_mesh_reorder(m.vxy, m.tri, P)
            ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 3.0, h)
            assert ctx.sem_get_info()["n_chunks"] >= 4 * grid_cap
            ctx.sem_write_state(U0, None)
            ctx.sem_write_velocity(V0)
            ctx.sem_set_step(4)
            ctx.sem_step_n(steps)
            Ug, _ = ctx.sem_read_field()
            Vg, _ = ctx.sem_read_velocity()
        assert rel_l2(Ug, Uo) <= 1e-12, (P, steps, rel_l2(Ug, Uo))
        assert rel_l2(Vg, Vo) <= 1e-12, (P, steps, rel_l2(Vg, Vo))


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_many_chunks_per_cta(monkeypatch, world):
    """Multi-rank path (boundary chunks, then interior chunks from chunk lists) with the
    grid capped at 2 CTAs: list walks with stage reuse on every rank."""
    monkeypatch.setenv("SEM_K7_GRID", "2")
    pb = mg.config("C2", 8)  # 64 x 64 cells, P3
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(9)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, 10, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0, U=U0, Uprev=Up, step0=3)
    g = S.LoopbackGroup(world)
    try:
        g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        g.sem_write_state(U0, Up)
        g.sem_set_step(3)
        g.sem_step_n(10)
        Ug, n = g.sem_read_field()
    finally:
        g.close()
    assert n == 13 and not np.isnan(Ug).any()
    assert rel_l2(Ug, Uo) <= 1e-12, rel_l2(Ug, Uo)
