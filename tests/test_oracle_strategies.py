"""Pins for the oracle's other reordering strategies (NEXT-3 of SURVEY §8f):
node degrees, the degree-sorted node renumbering
(PAPER.md:312-321 steps 1-2), the Node Connectivity / Node Distance strategies
(reading R20) and the canonical node coordinates they use.

Independent anchors:
* closed-form degrees of the structured 2-triangles-per-cell grid (counting
  spokes, far vertices, outer edges and interior nodes of a vertex star);
* brute force with Python sets / lists on tiny shuffled meshes, written from
  the paper's text (not from the C code);
* invariants: permutations, BFS property, first node = smallest key, element
  list sorted by the first visited node, same first-touch groups.
"""
import numpy as np
import pytest

from oracle import core
from paper_2104_08416_b200 import meshgen as mg


def setup(m, P):
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, P)
    return t, mu, N


@pytest.mark.parametrize("P", [2, 3])
def test_degree_closed_forms_structured_grid(P):
    nx, ny = 6, 5
    m = mg.grid_mesh(nx, ny, 1.0, 1.0)  # unjittered
    t, mu, N = setup(m, P)
    deg = core.node_degree(mu, N)
    Np = (P + 1) * (P + 2) // 2
    nI = (P - 1) * (P - 2) // 2
    # interior vertex: 6 triangles, 6 spokes: 6 (P-1) spoke-edge nodes + 6 far vertices
    # + 6 (P-1) outer-edge nodes + 6 nI interior nodes
    v = 2 * (nx + 1) + 3
    assert deg[v] == 6 * (P - 1) * 2 + 6 + 6 * nI
    # boundary vertex on the bottom side (not a corner): 3 triangles, 4 spokes
    vb = 2
    assert deg[vb] == 4 * (P - 1) + 4 + 3 * (P - 1) + 3 * nI
    # corner (0,0): 2 triangles sharing the diagonal; corner (nx, 0): 1 triangle
    assert deg[0] == 2 * Np - (P + 1) - 1
    assert deg[nx] == Np - 1
    # edge nodes: interior edge 2 Np - (P+1) - 1, boundary edge Np - 1; interior nodes Np - 1
    nv = m.nv
    edge_deg = deg[nv:nv + (N - nv - m.ne * nI)]
    assert set(np.unique(edge_deg)) == {Np - 1, 2 * Np - (P + 1) - 1}
    nb_edges = 2 * (nx + ny)
    assert (edge_deg == Np - 1).sum() == nb_edges * (P - 1)
    if nI:
        assert (deg[N - m.ne * nI:] == Np - 1).all()


def brute_degree(mu, N):
    nb = [set() for _ in range(N)]
    for row in mu:
        for a in row:
            nb[a].update(int(b) for b in row if b != a)
    return np.array([len(s) for s in nb]), nb


@pytest.mark.parametrize("P", [2, 3])
def test_degree_brute_force(P):
    m = mg.shuffle(mg.grid_mesh(5, 4, 1.3, 1.0, alpha=0.2, seed=2), 3, 4)
    t, mu, N = setup(m, P)
    d, _ = brute_degree(mu, N)
    assert np.array_equal(core.node_degree(mu, N), d)


@pytest.mark.parametrize("P", [2, 3])
def test_first_touch_degree_brute_force(P):
    m = mg.shuffle(mg.grid_mesh(5, 4, 1.3, 1.0, alpha=0.2, seed=2), 3, 4)
    t, mu, N = setup(m, P)
    _, perm_h, _ = core.hilbert_order(m.vxy, m.tri)
    mu_h = mu[perm_h]
    d, _ = brute_degree(mu, N)
    # PAPER.md:316-318 written out: N^(e) = nodes of e not seen before; sort by degree
    seen, order = set(), []
    for row in mu_h:
        grp = []
        for g in row:
            g = int(g)
            if g not in seen and g not in grp:
                grp.append(g)
        seen.update(grp)
        order += sorted(grp, key=lambda g: (d[g], g))
    perm, mu_new = core.first_touch_degree(mu_h, N)
    assert np.array_equal(perm, np.array(order, np.int32))
    inv = np.empty(N, np.int64)
    inv[perm] = np.arange(N)
    assert np.array_equal(mu_new, inv[mu_h])
    # same groups as plain first touch
    p0, _ = core.first_touch(mu_h, N)
    assert sorted(p0.tolist()) == list(range(N))
    starts = [0]
    for row in mu_h:
        starts.append(starts[-1] + len({int(g) for g in row} - set(p0[:starts[-1]].tolist())))
    for a, b in zip(starts[:-1], starts[1:]):
        assert set(p0[a:b].tolist()) == set(perm[a:b].tolist())


def brute_cm(mu, N, key):
    """Cuthill-McKee traversal from the paper's text (R20), Python lists."""
    _, nb = brute_degree(mu, N)
    vis = [False] * N
    order = []
    while len(order) < N:
        s = min((g for g in range(N) if not vis[g]), key=lambda g: (key[g], g))
        vis[s] = True
        order.append(s)
        h = len(order) - 1
        while h < len(order):
            u = order[h]
            h += 1
            new = sorted((w for w in nb[u] if not vis[w]), key=lambda g: (key[g], g))
            for w in new:
                vis[w] = True
                order.append(w)
    elems = []
    done = set()
    for g in order:
        for e in range(mu.shape[0]):
            if e not in done and g in mu[e]:
                done.add(e)
                elems.append(e)
    return np.array(elems, np.int32), np.array(order, np.int32)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("strategy", ["conn", "dist"])
def test_strategy_brute_force(P, strategy):
    m = mg.shuffle(mg.grid_mesh(5, 4, 1.3, 1.0, alpha=0.2, seed=6), 7, 8)
    t, mu, N = setup(m, P)
    key = core.conn_key(mu, N) if strategy == "conn" else core.dist_key(m.vxy, t, mu, P)
    ep, npm = core.strategy_order(mu, N, key)
    be, bn = brute_cm(mu, N, key)
    assert np.array_equal(npm, bn)
    assert np.array_equal(ep, be)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("strategy", ["conn", "dist"])
def test_strategy_invariants(P, strategy):
    m = mg.shuffle(mg.grid_mesh(13, 9, 2.0, 1.0, alpha=0.2, seed=1), 2, 3)
    t, mu, N = setup(m, P)
    key = core.conn_key(mu, N) if strategy == "conn" else core.dist_key(m.vxy, t, mu, P)
    ep, npm = core.strategy_order(mu, N, key)
    assert sorted(ep.tolist()) == list(range(m.ne))
    assert sorted(npm.tolist()) == list(range(N))
    pos = np.empty(N, np.int64)
    pos[npm] = np.arange(N)
    # first node has the smallest (key, id); Dist. starts at the lower-left corner vertex
    assert npm[0] == min(range(N), key=lambda g: (key[g], g))
    if strategy == "dist":
        x0, y0 = m.vxy[:, 0].min(), m.vxy[:, 1].min()
        assert np.array_equal(m.vxy[npm[0]], [x0, y0])
    # BFS: every node but the first has a neighbour visited before it
    _, nb = brute_degree(mu, N)
    for g in range(N):
        if pos[g] > 0:
            assert min(pos[w] for w in nb[g]) < pos[g]
    # element list sorted by (first visited node, element id)
    first = pos[mu].min(axis=1)
    assert np.array_equal(ep, np.lexsort((np.arange(m.ne), first)).astype(np.int32))


@pytest.mark.parametrize("P", [2, 3])
def test_node_coords(P):
    m = mg.shuffle(mg.grid_mesh(6, 5, 1.5, 1.0, alpha=0.2, seed=4), 5, 6)
    t, mu, N = setup(m, P)
    xy = core.node_coords(m.vxy, t, mu, P)
    assert np.isfinite(xy).all()
    assert np.array_equal(xy[:m.nv], m.vxy)  # vertex nodes are the vertices, bit for bit
    o = core.OracleSEM(m.vxy, m.tri, P)
    assert np.abs(xy - o.node_xy()).max() < 1e-14  # element map F^(e)(x^_p)
    if P == 2:  # edge nodes are the midpoints
        mids = 0.5 * (m.vxy[t[:, 0]] + m.vxy[t[:, 1]])
        assert np.abs(xy[mu[:, 1]] - mids).max() < 1e-15
