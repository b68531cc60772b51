"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): keys, permutations and renumbering bit-exact;
fp64 field within relative L2 <= 1e-10 (tolerance stated per test).  Inputs are
the seeded recipe of paper_2104_08416_b200/meshgen.py; nothing the oracle sees
comes from the GPU.
"""
import os

import numpy as np
import pytest

from oracle import core
from oracle.core import OracleSEM
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S

pytestmark = pytest.mark.gpu

REL_L2 = 1e-10


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    c = S.SemContext(0)
    yield c
    c.close()


def oracle_reorder(m, P, elem_order=S.SEM_ORDER_HILBERT, node_order=S.SEM_NODES_FIRST_TOUCH, seed=0):
    o_tri = core.orient(m.vxy, m.tri)
    mu_can, N = core.canonical_nodes(o_tri, m.nv, P)
    if elem_order == S.SEM_ORDER_HILBERT:
        key, perm, grid = core.hilbert_order(m.vxy, m.tri)
    elif elem_order == S.SEM_ORDER_RANDOM:
        perm = core.random_order(m.ne, seed)
        key, grid = np.zeros(m.ne, np.uint32), (0, 0)
    else:
        perm = np.arange(m.ne, dtype=np.int32)
        key, grid = np.zeros(m.ne, np.uint32), (0, 0)
    if node_order == S.SEM_NODES_FIRST_TOUCH:
        node_perm, _ = core.first_touch(mu_can[perm], N)
    else:
        node_perm = np.arange(N, dtype=np.int32)
    return key, perm, node_perm, N, grid


CASES = [("C1", 1), ("C2", 8), ("C3", 20), ("C4", 32), ("C5", 128), ("C2", 1)]


@pytest.mark.parametrize("name,scale", CASES)
def test_reorder_bit_exact(ctx, name, scale):
    pb = mg.config(name, scale)
    m = pb.mesh
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
    key, perm, node_perm, N, grid = oracle_reorder(m, pb.P)
    assert r["grid"] == grid
    assert r["n_nodes"] == N
    assert np.array_equal(r["keys"], key)
    assert np.array_equal(r["elem_perm"], perm)
    assert np.array_equal(r["node_perm"], node_perm)


def test_reorder_caller_buffers(ctx):
    """Outputs written into caller-owned (pinned) arrays, or skipped with None,
    carry the same bits as the binding's own arrays."""
    import torch
    pb = mg.config("C3", 8)
    m = pb.mesh
    ref = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
    nmax = m.nv + 3 * m.ne * (pb.P - 1) + m.ne * (pb.P - 1) * (pb.P - 2) // 2
    out = {"keys": torch.full((m.ne,), -1, dtype=torch.int32).pin_memory().numpy().view(np.uint32),
           "elem_perm": np.full(m.ne, -1, np.int32),
           "node_perm": torch.full((nmax + 5,), -1, dtype=torch.int32).pin_memory().numpy()}
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, out=out)
    for k in ("keys", "elem_perm", "node_perm"):
        assert np.array_equal(r[k], ref[k]), k
    assert np.all(out["node_perm"][r["n_nodes"]:] == -1)  # nothing written past N
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, out={"keys": None, "elem_perm": None})
    assert r["keys"] is None and r["elem_perm"] is None
    assert np.array_equal(r["node_perm"], ref["node_perm"])
    with pytest.raises(ValueError):
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, out={"elem_perm": np.zeros(m.ne - 1, np.int32)})


@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
                                                   (S.SEM_ORDER_RANDOM, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_HILBERT, S.SEM_NODES_CANONICAL),
                                                   (S.SEM_ORDER_INPUT, S.SEM_NODES_FIRST_TOUCH)])
def test_reorder_variants_bit_exact(ctx, elem_order, node_order):
    pb = mg.config("C2", 16)
    m = pb.mesh
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, node_order, seed=1234)
    key, perm, node_perm, N, grid = oracle_reorder(m, pb.P, elem_order, node_order, seed=1234)
    assert np.array_equal(r["elem_perm"], perm)
    assert np.array_equal(r["node_perm"], node_perm)


def run_gpu(ctx, pb, steps, elem_order=S.SEM_ORDER_HILBERT, node_order=S.SEM_NODES_FIRST_TOUCH,
            mesh=None, c=None, src=None, state=None, step0=0):
    m = pb.mesh if mesh is None else mesh
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, elem_order, node_order, seed=7)
    ctx.sem_build_operators(pb.c if c is None else c, pb.src_vertex if src is None else src,
                            pb.f0, pb.t0, pb.amplitude, pb.dt)
    if state is not None:
        ctx.sem_write_state(state[0], state[1])
        ctx.sem_set_step(step0)
    ctx.sem_step_n(steps)
    U, n = ctx.sem_read_field()
    assert n == step0 + steps
    return U


def test_c1_full_run_parity(ctx):
    pb = mg.config("C1")
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, pb.n_steps, src=pb.src_vertex, A=pb.amplitude, f0=pb.f0, t0=pb.t0)
    Ug = run_gpu(ctx, pb, pb.n_steps)
    assert np.abs(Uo).max() > 0
    assert rel_l2(Ug, Uo) <= REL_L2


@pytest.mark.parametrize("elem_order,node_order", [(S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
                                                   (S.SEM_ORDER_RANDOM, S.SEM_NODES_FIRST_TOUCH),
                                                   (S.SEM_ORDER_HILBERT, S.SEM_NODES_CANONICAL)])
def test_c1_orderings_same_field(ctx, elem_order, node_order):
    pb = mg.config("C1")
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, 120, src=pb.src_vertex, A=pb.amplitude, f0=pb.f0, t0=0.05)
    pb2 = mg.Problem(**{**pb.__dict__, "t0": 0.05})
    Ug = run_gpu(ctx, pb2, 120, elem_order, node_order)
    assert rel_l2(Ug, Uo) <= REL_L2


@pytest.mark.parametrize("name,scale,steps", [("C2", 4, 300), ("C3", 10, 200), ("C4", 16, 200), ("C5", 64, 150)])
def test_reduced_configs_run_parity(ctx, name, scale, steps):
    # shifted source peak (t0 = 10 dt) so the short run carries a real wavefield
    pb = mg.config(name, scale)
    pb = mg.Problem(**{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)})
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
    Ug = run_gpu(ctx, pb, steps)
    assert np.count_nonzero(Uo) > 0.05 * Uo.size
    assert rel_l2(Ug, Uo) <= REL_L2


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C2", 1), ("C3", 4), ("C4", 4), ("C5", 32)])
def test_random_state_steps_parity(ctx, name, scale):
    """P-12: one and ten steps from seeded random full-mesh states."""
    pb = mg.config(name, scale)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(42)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    for steps in (1, 10):
        Uo, _ = o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0,
                           U=U0, Uprev=Up, step0=37)
        Ug = run_gpu(ctx, pb, steps, state=(U0, Up), step0=37)
        assert rel_l2(Ug, Uo) <= 1e-13 * steps, (name, steps, rel_l2(Ug, Uo))
        assert np.abs(Ug - Uo).max() <= 1e-12 * np.abs(Uo).max()


def test_read_internal_numbering(ctx):
    pb = mg.config("C1")
    r = ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, pb.P)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    rng = np.random.default_rng(0)
    U = rng.standard_normal(r["n_nodes"])
    ctx.sem_write_state(U, None)
    Ui, _ = ctx.sem_read_field(S.SEM_NUMBERING_INTERNAL)
    assert np.array_equal(Ui, U[r["node_perm"]])
    Uc, _ = ctx.sem_read_field(S.SEM_NUMBERING_CANONICAL)
    assert np.array_equal(Uc, U)


def test_bitwise_deterministic(ctx):
    pb = mg.config("C2", 4)
    a = run_gpu(ctx, pb, 50)
    b = run_gpu(ctx, pb, 50)
    assert np.array_equal(a, b)


def test_errors(ctx):
    pb = mg.config("C1", 4)
    m = pb.mesh
    with pytest.raises(S.SemError) as e:
        ctx.sem_mesh_reorder(m.vxy, m.tri, 8)
    assert e.value.status == S.SEM_E_UNSUPPORTED
    bad = m.vxy.copy()
    t = m.tri[5]
    bad[t[2]] = bad[t[0]]  # coincident vertices: exactly zero area
    with pytest.raises(S.SemError) as e:
        ctx.sem_mesh_reorder(bad, m.tri, 2)
    assert e.value.status == S.SEM_E_MESH and "zero area" in e.value.msg
    for v in (m.nv, -1, 2**31 - 1):  # vertex ids outside [0, V): checked on the GPU before any access
        tri = m.tri.copy()
        tri[7, 1] = v
        tri[9, 2] = v
        with pytest.raises(S.SemError) as e:
            ctx.sem_mesh_reorder(m.vxy, tri, 2)
        assert e.value.status == S.SEM_E_MESH and "element 7 has a vertex id out of range" in e.value.msg
    ctx.sem_mesh_reorder(m.vxy, m.tri, 2)
    with pytest.raises(S.SemError) as e:
        ctx.sem_step_n(1)
    assert e.value.status == S.SEM_E_STATE
    c = pb.c.copy()
    c[3] = -1.0
    with pytest.raises(S.SemError) as e:
        ctx.sem_build_operators(c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    assert e.value.status == S.SEM_E_ARG and "element 3" in e.value.msg
    for k, v in ((9, np.nan), (11, 0.0), (12, np.inf)):  # checked on the device: the smallest bad index
        c = pb.c.copy()
        c[k] = v
        c[k + 5] = -2.0
        with pytest.raises(S.SemError) as e:
            ctx.sem_build_operators(c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        assert e.value.status == S.SEM_E_ARG and ("element %d " % k) in e.value.msg, e.value.msg
    with pytest.raises(S.SemError) as e:
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, -1.0)
    assert e.value.status == S.SEM_E_ARG


def test_nonfinite_reported(ctx):
    pb = mg.config("C1", 4)
    ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, 2)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt * 50)  # unstable dt
    ctx.sem_step_n(3000)
    with pytest.raises(S.SemError) as e:
        ctx.sem_read_field()
    assert e.value.status == S.SEM_E_NONFINITE and "step 3000" in e.value.msg


def test_single_element_and_tiny(ctx):
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    tri = np.array([[0, 2, 1]], np.int32)  # clockwise: fixed by the library
    for P in (2, 3):
        r = ctx.sem_mesh_reorder(vxy, tri, P)
        assert r["n_nodes"] == (6 if P == 2 else 10)
        o = OracleSEM(vxy, tri, P)
        ctx.sem_build_operators(np.ones(1), 0, 5.0, 0.0, 1.0, 0.01)
        U0 = np.random.default_rng(P).standard_normal(o.N)
        ctx.sem_write_state(U0, U0)
        ctx.sem_step_n(5)
        Ug, _ = ctx.sem_read_field()
        Uo, _ = o.leapfrog(0.01, 5, src=0, A=1.0, f0=5.0, t0=0.0, U=U0, Uprev=U0)
        assert rel_l2(Ug, Uo) <= 1e-13


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_bench_configuration(ctx, name):
    """Full BASELINE.json size in the launch configuration bench.py times
    (one rank, default chunks): one step from a seeded random state over the
    whole mesh, and the configured Ricker run for 10 steps from zero."""
    pb = mg.config(name)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    rng = np.random.default_rng(7)
    U0 = rng.standard_normal(o.N)
    Up = U0 + 0.1 * rng.standard_normal(o.N)
    Uo, _ = o.leapfrog(pb.dt, 1, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0, U=U0, Uprev=Up, step0=5)
    Ug = run_gpu(ctx, pb, 1, state=(U0, Up), step0=5)
    assert ctx.sem_get_info()["chunk_elems"] == 512  # the P3 default (api.cu chunk_elems)
    assert rel_l2(Ug, Uo) <= 1e-13, rel_l2(Ug, Uo)
    pb2 = mg.Problem(**{**pb.__dict__, "t0": 3 * pb.dt, "f0": 1.0 / (8 * pb.dt)})
    Uo, _ = o.leapfrog(pb2.dt, 10, src=pb2.src_vertex, A=1.0, f0=pb2.f0, t0=pb2.t0)
    Ug = run_gpu(ctx, pb2, 10)
    assert np.abs(Uo).max() > 0
    assert rel_l2(Ug, Uo) <= REL_L2, rel_l2(Ug, Uo)


_GRAPH_CHILD = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2104_08416_b200 import meshgen as mg, sem as S
pb = mg.config("C2", 16)
pb = mg.Problem(**{{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)}})
m = pb.mesh
with S.SemContext(0) as c:
    c.sem_mesh_reorder(m.vxy, m.tri, pb.P)
    c.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    for n in (70, 3, 77):
        c.sem_step_n(n)
    U, n = c.sem_read_field()
    assert n == 150
    np.save({out!r}, U)
"""


def test_graph_step_loop_bitwise_equal(tmp_path):
    """The CUDA-graph step loop (32 captured steps per replay, the remainder from the
    16/8/4/2/1-step graphs, device step counter) gives the same bits as launching step by step (SEM_GRAPH=0, read once
    per process: a child process), with and without the kernel-timing events in
    the graph and with a capture-only sem_step_n(0), and matches the oracle."""
    import subprocess
    import sys
    pb = mg.config("C2", 16)
    pb = mg.Problem(**{**pb.__dict__, "t0": 10 * pb.dt, "f0": 1.0 / (8 * pb.dt)})
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    Uo, _ = o.leapfrog(pb.dt, 150, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
    out = []
    for timing in (False, True):
        with S.SemContext(0) as c:
            c.sem_mesh_reorder(m.vxy, m.tri, pb.P)
            c.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
            c.sem_step_n(0)    # capture only: advances nothing
            assert c.sem_read_field()[1] == 0
            c.sem_set_kernel_timing(timing)  # timing: the graph with event-record nodes
            c.sem_step_n(70)   # 2 replays of the 32-step graph + the 4- and 2-step graphs (timing: 6 plain steps)
            c.sem_step_n(3)    # the 2- and 1-step graphs: the parity flips
            c.sem_step_n(77)   # odd parity at entry: the other captured graphs (64 + 8 + 4 + 1)
            U, n = c.sem_read_field()
            assert n == 150
            if timing:
                kt = c.sem_kernel_times()
                assert kt["k7_launches"] == 150 and kt["k7_ms"] > 0
            out.append(U)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    f = str(tmp_path / "plain.npy")
    env = dict(os.environ, SEM_GRAPH="0")
    r = subprocess.run([sys.executable, "-c", _GRAPH_CHILD.format(root=root, out=f)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out.append(np.load(f))
    assert np.array_equal(out[0], out[1])
    assert np.array_equal(out[0], out[2])
    assert rel_l2(out[0], Uo) <= REL_L2


@pytest.mark.skipif(os.environ.get("SEM_TEST_FULL_C5") != "1", reason="full C5 (268M elements) is opt-in: SEM_TEST_FULL_C5=1")
def test_full_size_c5_properties(ctx):
    """BASELINE.json configs[4] at its full size on one GPU (268M elements, P2,
    537M nodes): properties that hold at any size.  A constant field with no
    source stays constant (K 1 = 0 through every element's G and mu row), the
    preparation is deterministic (two reorders give the same permutations), and
    the configured run stays finite."""
    pb = mg.config("C5")
    m = pb.mesh
    r = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
    info = ctx.sem_get_info()
    assert info["n_elements"] == 268_435_456 and r["n_nodes"] == info["n_nodes"]
    ctx.sem_build_operators(pb.c, -1, pb.f0, pb.t0, 1.0, pb.dt)
    U = np.full(r["n_nodes"], 3.0)
    ctx.sem_write_state(U, U)
    ctx.sem_step_n(5)
    Ug, _ = ctx.sem_read_field()
    assert np.abs(Ug - 3.0).max() <= 1e-11
    r2 = ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P)
    assert np.array_equal(r["elem_perm"], r2["elem_perm"]) and np.array_equal(r["node_perm"], r2["node_perm"])
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
    ctx.sem_step_n(20)
    Ug, n = ctx.sem_read_field()
    assert n == 20 and np.isfinite(Ug).all()


def test_degenerate_inputs(ctx):
    """Empty mesh, zero steps, unused vertices, more ranks than elements."""
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [5.0, 5.0]])
    tri = np.array([[0, 1, 2]], np.int32)
    with pytest.raises(S.SemError) as e:
        ctx.sem_mesh_reorder(vxy, np.zeros((0, 3), np.int32), 2)
    assert e.value.status == S.SEM_E_ARG
    with pytest.raises(S.SemError) as e:  # vertex 3 is used by no element: its M-bar would be 0
        ctx.sem_mesh_reorder(vxy, tri, 2)
    assert e.value.status == S.SEM_E_MESH and "vertex 3" in e.value.msg
    bad = tri.copy()
    bad[0, 2] = 7
    with pytest.raises(S.SemError) as e:
        ctx.sem_mesh_reorder(vxy[:3], bad, 2)
    assert e.value.status == S.SEM_E_MESH
    ctx.sem_mesh_reorder(vxy[:3], tri, 3)
    ctx.sem_build_operators(np.ones(1), 0, 5.0, 0.0, 1.0, 0.01)
    ctx.sem_step_n(0)
    U, n = ctx.sem_read_field()
    assert n == 0 and (U == 0).all()
    with pytest.raises(S.SemError) as e:
        ctx.sem_step_n(-1)
    assert e.value.status == S.SEM_E_ARG
    with pytest.raises(S.SemError) as e:
        S.LoopbackGroup(2).sem_mesh_reorder(vxy[:3], tri, 2)  # 1 element, 2 ranks
    assert e.value.status == S.SEM_E_ARG


def test_torch_allocator_hook_bitwise():
    """SURVEY §8(b)'s allocator hook: with PyTorch's caching allocator behind sem_allocator,
    every device array of the context is torch memory (torch.cuda.memory_allocated grows by
    at least the mesh and operator arrays while the context lives and returns when it is
    freed) and the field is bitwise the same as with the library's own pool."""
    import torch
    pb = mg.config("C2", 8)
    m = pb.mesh
    rng = np.random.default_rng(3)

    def run(allocator):
        with S.SemContext(0, allocator=allocator) as c:
            r = c.sem_mesh_reorder(m.vxy, m.tri, pb.P)
            c.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
            U0 = np.random.default_rng(3).standard_normal(r["n_nodes"])
            c.sem_write_state(U0, U0)
            c.sem_step_n(40)
            held = torch.cuda.memory_allocated(0)
            U, _ = c.sem_read_field()
        return U, held

    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    Ua, _ = run(None)
    Ut, held = run("torch")
    torch.cuda.synchronize()
    assert np.array_equal(Ua, Ut)
    # mu-sized chunk tables, G, U^n, U^{n-1}, dt^2/M at least: > 24 B per element
    assert held - base > 24 * m.ne
    assert torch.cuda.memory_allocated(0) == base
    g = S.LoopbackGroup(2, allocator="torch")
    try:
        g.sem_mesh_reorder(m.vxy, m.tri, pb.P)
        g.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, 1.0, pb.dt)
        g.sem_step_n(5)
        Ug, _ = g.sem_read_field()
        assert not np.isnan(Ug).any()
    finally:
        g.close()
    del rng
