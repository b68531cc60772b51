"""Multi-GPU partition logic, host side, on CPU.

The library's partition (paper_2104_08416_b200/csrc/partition.cpp, reached through
the host-only `sem_debug_partition`) is checked against what the decomposition
must satisfy, using the oracle's reordered connectivity as input:
* contiguous element ranges covering the mesh; local nodes = nodes of the
  local elements;
* symmetric neighbour relation and identical per-pair interface lists (the
  message layout both sides of a send/recv agree on);
* every node owned by exactly one rank;
* emulated exchange: every rank's interface sum equals the sum over ranks in
  ascending rank order, bit-for-bit identical on all replicas.
A world_size-2 gloo run repeats the exchange check across real processes.
"""
import os

import numpy as np
import pytest

from oracle import core
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem


def global_mu(name="C2", scale=16):
    pb = mg.config(name, scale)
    m = pb.mesh
    tri = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(tri, m.nv, pb.P)
    key, perm, grid = core.hilbert_order(m.vxy, m.tri)
    node_perm, mu_ft = core.first_touch(mu[perm], N)
    return mu_ft, N


def emulate_exchange(parts, values):
    """values[r][i]: rank r's partial of its interface node i.  Returns each rank's totals."""
    world = len(parts)
    totals = []
    for r, P in enumerate(parts):
        nif = len(P["if_glob"])
        xbuf = np.empty(nif + len(P["send_glob"]))
        xbuf[:nif] = values[r]
        for k, q in enumerate(P["nbr"]):
            Q = parts[q]
            kq = list(Q["nbr"]).index(r)
            # what q packs for r: its partials of the nodes in its list for r
            sent_glob = Q["send_glob"][Q["nbr_off"][kq]:Q["nbr_off"][kq + 1]]
            qpos = {g: i for i, g in enumerate(Q["if_glob"])}
            blk = np.array([values[q][qpos[g]] for g in sent_glob])
            xbuf[nif + P["nbr_off"][k]: nif + P["nbr_off"][k + 1]] = blk
        tot = np.empty(nif)
        for i in range(nif):
            acc = 0.0
            for j in range(P["sum_start"][i], P["sum_start"][i + 1]):
                acc += xbuf[P["sum_src"][j]]
            tot[i] = acc
        totals.append(tot)
    return totals


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partition_invariants(world):
    mu, N = global_mu()
    E = mu.shape[0]
    parts = [sem.sem_debug_partition(mu, N, r, world) for r in range(world)]
    # contiguous element ranges
    assert parts[0]["e0"] == 0 and parts[-1]["e1"] == E
    for r in range(world - 1):
        assert parts[r]["e1"] == parts[r + 1]["e0"]
        assert parts[r]["e1"] == (r + 1) * E // world
    # ranks touching each node
    touch = [set() for _ in range(N)]
    for r, P in enumerate(parts):
        loc = np.unique(mu[P["e0"]:P["e1"]])
        assert np.array_equal(P["loc2glob"], loc)
        for g in loc:
            touch[g].add(r)
    # ownership: exactly one owner (the lowest toucher)
    assert sum(P["n_owned"] for P in parts) == N
    # interface nodes and neighbour lists
    for r, P in enumerate(parts):
        expect_if = [g for g in P["loc2glob"] if len(touch[g]) > 1]
        assert list(P["if_glob"]) == expect_if
        expect_nbr = sorted(set().union(*[touch[g] for g in expect_if]) - {r}) if expect_if else []
        assert list(P["nbr"]) == expect_nbr
        for k, q in enumerate(P["nbr"]):
            mine = list(P["send_glob"][P["nbr_off"][k]:P["nbr_off"][k + 1]])
            Q = parts[q]
            kq = list(Q["nbr"]).index(r)
            theirs = list(Q["send_glob"][Q["nbr_off"][kq]:Q["nbr_off"][kq + 1]])
            assert mine == theirs == sorted(g for g in expect_if if q in touch[g])
    # emulated exchange: rank-ordered sums, bitwise identical on all replicas
    rng = np.random.default_rng(world)
    val = {}
    values = []
    for r, P in enumerate(parts):
        v = rng.standard_normal(len(P["if_glob"]))
        values.append(v)
        for g, x in zip(P["if_glob"], v):
            val[(r, int(g))] = x
    totals = emulate_exchange(parts, values)
    seen = {}
    for r, P in enumerate(parts):
        for g, t in zip(P["if_glob"], totals[r]):
            acc = 0.0
            for q in sorted(touch[g]):
                acc += val[(q, int(g))]
            assert t == acc
            if int(g) in seen:
                assert seen[int(g)] == t  # every replica has the same bits
            seen[int(g)] = t
    max_mult = max(len(touch[g]) for g in range(N))
    assert 2 <= max_mult <= 4 or world == 2


def _gloo_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mu, N = global_mu()
    P = sem.sem_debug_partition(mu, N, rank, world)
    rng = np.random.default_rng(100 + rank)
    mine = rng.standard_normal(len(P["if_glob"]))
    # real exchange over gloo: each rank sends its packed partials per neighbour
    pos = {int(g): i for i, g in enumerate(P["if_glob"])}
    packed = {int(q): [mine[pos[int(g)]] for g in P["send_glob"][P["nbr_off"][k]:P["nbr_off"][k + 1]]]
              for k, q in enumerate(P["nbr"])}
    allp = [None] * world
    dist.all_gather_object(allp, packed)
    nif = len(P["if_glob"])
    xbuf = np.empty(nif + len(P["send_glob"]))
    xbuf[:nif] = mine
    for k, q in enumerate(P["nbr"]):
        xbuf[nif + P["nbr_off"][k]: nif + P["nbr_off"][k + 1]] = allp[q][rank]
    tot = [sum(xbuf[P["sum_src"][j]] for j in range(P["sum_start"][i], P["sum_start"][i + 1])) for i in range(nif)]
    allv = [None] * world
    dist.all_gather_object(allv, {int(g): float(x) for g, x in zip(P["if_glob"], mine)})
    ok = True
    for i, g in enumerate(P["if_glob"]):
        acc = 0.0
        for q in range(world):
            if int(g) in allv[q]:
                acc += allv[q][int(g)]
        ok &= (acc == tot[i])
    np.save(os.path.join(out_dir, "r%d.npy" % rank), np.array([ok, nif, len(P["nbr"])], dtype=np.int64))
    dist.destroy_process_group()


def test_gloo_world2_exchange(tmp_path):
    import socket

    import torch.multiprocessing as tmp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tmp.spawn(_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert r0[0] == 1 and r1[0] == 1
    assert r0[1] == r1[1] > 0 and r0[2] == r1[2] == 1
