"""The GPU chunk builder (csrc/chunks_gpu.cu) against the host builder
(csrc/chunks.cpp): with SEM_CHUNK_CHECK=1 sem_mesh_reorder builds both and
fails with SEM_E_MESH naming the first array that differs (scalars, chunk
lists, cmeta, lidx, lpos, lptr, sh_pstart, shl_node, shl_slot, shl_cr,
int_of).  The host builder is the one every parity test validated before."""
import os

import pytest

from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu


@pytest.fixture()
def ctx(monkeypatch):
    monkeypatch.setenv("SEM_CHUNK_CHECK", "1")
    c = S.SemContext(0)
    yield c
    c.close()


@pytest.mark.parametrize("name,scale,deg", [("C1", 1, None), ("C2", 8, None), ("C3", 20, None), ("C4", 32, None),
                                            ("C5", 64, None), ("B1", 25, 5), ("B1", 30, 7)])
@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
                                                   (S.SEM_ORDER_RANDOM, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_CONN, S.SEM_NODES_VISIT)])
def test_gpu_chunks_equal_host(ctx, name, scale, deg, elem_order, node_order):
    pb = mg.config(name, scale, degree=deg) if deg else mg.config(name, scale)
    ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P, elem_order, node_order, seed=3)
    info = ctx.sem_get_info()
    assert info["n_chunks"] >= 1 and info["n_shared_nodes"] > 0


@pytest.mark.parametrize("B", ["128", "192", "256", "512"])
def test_gpu_chunks_equal_host_chunk_sizes(ctx, monkeypatch, B):
    monkeypatch.setenv("SEM_CHUNK", B)
    pb = mg.config("C2", 8)
    ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
    assert ctx.sem_get_info()["chunk_elems"] == int(B)


def test_single_element_and_tiny(ctx):
    import numpy as np
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    for tri in (np.array([[0, 1, 2]], np.int32), np.array([[0, 1, 2], [1, 3, 2]], np.int32)):
        for P in (2, 3, 5, 7):
            r = ctx.sem_mesh_reorder(vxy[:3] if len(tri) == 1 else vxy, tri, P)
            assert r["n_nodes"] > 0


def test_chunks_of_512_fall_back_to_256(monkeypatch):
    """P3 defaults to chunks of 512 (api.cu chunk_elems); a mesh whose largest chunks would
    not fit one K7 CTA's shared memory is rebuilt with 256 (SEM_K7_SMEM_CAP lowers the budget
    to force it).  Both builds keep the oracle parity of a few steps from a random state."""
    import numpy as np
    from oracle.core import OracleSEM

    monkeypatch.delenv("SEM_CHUNK", raising=False)
    pb = mg.config("C2", 8)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(11)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, 5, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=0.0, U=U0, Uprev=Up, step0=3)
    for cap, want in ((None, 512), ("150000", 256)):
        if cap:
            monkeypatch.setenv("SEM_K7_SMEM_CAP", cap)
        with S.SemContext(0) as c:
            c.sem_mesh_reorder(m.vxy, m.tri, pb.P)
            assert c.sem_get_info()["chunk_elems"] == want
            c.sem_build_operators(pb.c, pb.src_vertex, pb.f0, 0.0, 1.0, pb.dt)
            c.sem_write_state(U0, Up)
            c.sem_set_step(3)
            c.sem_step_n(5)
            Ug, n = c.sem_read_field()
        assert n == 8
        assert float(np.linalg.norm(Ug - Uo) / np.linalg.norm(Uo)) <= 1e-13
