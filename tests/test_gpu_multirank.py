"""Multi-GPU path on one B200: G in-process partitions (loopback transport).

The partitions run the multi-GPU kernels (interface partials, pack, rank-ordered
sums) with a device-to-device copy in place of NCCL send/recv; the host
sequences the ranks with events, so no kernel ever waits on another rank.
Results must match the oracle (rel L2 <= 1e-10) and the one-rank GPU run
(rounding-level: only the summation order of interface nodes differs).
"""
import os

import numpy as np
import pytest

from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def shifted(pb):
    return mg.Problem(**{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)})


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_loopback_matches_oracle_and_single_rank(world):
    pb = shifted(mg.config("C2", 4))  # 128 x 128 cells, P3
    m = pb.mesh
    steps = 150
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
    with S.SemContext(0) as one:
        one.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        one.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        one.sem_step_n(steps)
        U1, _ = one.sem_read_field()
    g = S.LoopbackGroup(world)
    try:
        g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        infos = [c.sem_get_info() for c in g.ctxs]
        assert sum(i["n_elements"] for i in infos) == m.ne
        assert all(i["n_interface_nodes"] > 0 for i in infos)
        g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        g.sem_step_n(steps)
        Ug, n = g.sem_read_field()
    finally:
        g.close()
    assert n == steps
    assert not np.isnan(Ug).any()  # every node written by exactly its owner
    assert rel_l2(Ug, Uo) <= 1e-10
    assert rel_l2(Ug, U1) <= 1e-13


@pytest.mark.parametrize("name,scale,world", [("C3", 20, 4), ("C5", 128, 8), ("C1", 1, 3)])
def test_loopback_random_state_steps(name, scale, world):
    pb = mg.config(name, scale)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(5)
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
    assert n == 13
    assert rel_l2(Ug, Uo) <= 1e-12


def test_loopback_bitwise_deterministic():
    pb = shifted(mg.config("C2", 8))
    m = pb.mesh
    outs = []
    for _ in range(2):
        g = S.LoopbackGroup(4)
        try:
            g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
            g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
            g.sem_step_n(60)
            outs.append(g.sem_read_field()[0])
        finally:
            g.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("name,scale", [("C2", 8), ("C5", 128)])
def test_gpu_partition_equals_host(monkeypatch, world, name, scale):
    """SEM_CHUNK_CHECK=1: every rank's GPU partition (partition_gpu.cu) and GPU
    chunk metadata are compared with the host builders (partition.cpp,
    chunks.cpp), array by array; sem_mesh_reorder fails on any difference."""
    monkeypatch.setenv("SEM_CHUNK_CHECK", "1")
    pb = mg.config(name, scale)
    g = S.LoopbackGroup(world)
    try:
        g.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P)
        infos = [c.sem_get_info() for c in g.ctxs]
        assert all(i["n_interface_nodes"] > 0 for i in infos)
    finally:
        g.close()


def test_nccl_unique_id_through_dlopen():
    """The NCCL transport of the multi-GPU path: libsem dlopens libnccl (torch's copy) and
    creates unique ids (the only NCCL step one GPU can run; the send/recv exchange needs
    two devices and runs in the driver's scaling bench)."""
    # in a subprocess: whichever libnccl this maps stays out of the pytest process
    import subprocess
    import sys
    code = ("from paper_2104_08416_b200 import sem as S\n"
            "a, b = S.nccl_unique_id(), S.nccl_unique_id()\n"
            "assert len(a) == 128 and len(b) == 128\n"
            "assert any(a) and a != b\n"
            "import torch\n"
            "assert torch.cuda.is_available()\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def _nccl_rank(rank, world, nccl_id, q):
    from paper_2104_08416_b200 import meshgen as mg_
    from paper_2104_08416_b200 import sem as S_
    pb = mg_.config("C2", 8)
    m = pb.mesh
    rng = np.random.default_rng(5)
    with S_.SemContext(rank, rank, world, nccl_id=nccl_id) as ctx:
        r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        U0 = rng.standard_normal(r["n_nodes"])
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        ctx.sem_write_state(U0, U0)
        ctx.sem_step_n(20)
        out = np.full(r["n_nodes"], np.nan)
        ctx.sem_read_field(out=out)
    q.put((rank, out))


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="the NCCL transport needs two GPUs (the driver's GPU runs have one)")
def test_nccl_two_gpus_bitwise_equal_to_loopback():
    """The real transport: two processes, one GPU each, a real NCCL unique id; the merged
    field must equal the in-process loopback group's bit for bit (same kernels, same
    rank-ordered sums; only the transport differs)."""
    import multiprocessing as mp
    nid = S.nccl_unique_id()
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    ps = [ctx_mp.Process(target=_nccl_rank, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    parts = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    Un = np.where(np.isnan(parts[0]), parts[1], parts[0])
    pb = mg.config("C2", 8)
    m = pb.mesh
    g = S.LoopbackGroup(2)
    try:
        r = g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        U0 = np.random.default_rng(5).standard_normal(g.ctxs[0].N)
        g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        g.sem_write_state(U0, U0)
        g.sem_step_n(20)
        Ul, _ = g.sem_read_field()
    finally:
        g.close()
    assert not np.isnan(Un).any()
    assert np.array_equal(Un, Ul)
