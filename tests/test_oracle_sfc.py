"""Pins for the oracle's SFC ordering and node renumbering
(PAPER.md:312-321).

Fixed by the paper: Listing 1 is executable (order-1 path, order-5 positions);
the generalized curve equals Listing 1 on 2^k squares; the grid
formula w_b = sqrt(n_e), h_b = sqrt(n_e)/r (n_e = 250000, r = 2
gives 500 x 250).  Fixed by combinatorics: bijection and adjacency
of the path on every rectangle up to 64 x 64, with a diagonal step only where
a corner-to-corner Hamiltonian path cannot exist (bipartite parity).
"""
import numpy as np
import pytest

from oracle import core
from oracle.listing1 import listing1_path
from paper_2104_08416_b200 import meshgen as mg


def test_listing1_pins():
    assert listing1_path(1) == [(0, 0), (0, 1), (1, 1), (1, 0)]
    p = listing1_path(5)
    d = {c: i for i, c in enumerate(p)}
    assert len(p) == 1024 and len(d) == 1024
    assert d[(16, 16)] == 512 and d[(0, 31)] == 341 and d[(5, 9)] == 216 and d[(31, 0)] == 1023
    for k in range(1, 6):
        pk = listing1_path(k)
        assert pk[0] == (0, 0) and pk[-1] == (2 ** k - 1, 0)
        # first move alternates with the parity of the order
        assert pk[1] == ((0, 1) if k % 2 == 1 else (1, 0))


@pytest.mark.parametrize("k", range(0, 7))
def test_generalized_equals_listing1_on_powers_of_two(k):
    p = core.gilbert_path(2 ** k, 2 ** k)
    if k == 0:
        assert p.tolist() == [[0, 0]]
        return
    assert p.tolist() == [list(c) for c in listing1_path(k)]


def test_generalized_bijection_and_adjacency_all_rectangles():
    for w in range(1, 65):
        for h in range(1, 65):
            p = core.gilbert_path(w, h)
            assert p.shape == (w * h, 2)
            assert p[0].tolist() == [0, 0]
            assert (p[:, 0] >= 0).all() and (p[:, 0] < w).all() and (p[:, 1] >= 0).all() and (p[:, 1] < h).all()
            assert len(np.unique(p[:, 1].astype(np.int64) * w + p[:, 0])) == w * h
            if w * h > 1:
                d = np.abs(np.diff(p, axis=0))
                assert d.max() == 1, (w, h)  # Chebyshev distance 1
                ndiag = int((d.sum(axis=1) == 2).sum())
                assert ndiag <= 1, (w, h)
                if ndiag:
                    forced = (w >= h and w % 2 == 1 and h % 2 == 0) or (w < h and h % 2 == 1 and w % 2 == 0)
                    assert forced, (w, h)


def test_straight_runs():
    assert core.gilbert_path(1, 5).tolist() == [[0, i] for i in range(5)]
    assert core.gilbert_path(5, 1).tolist() == [[i, 0] for i in range(5)]


def test_grid_dims_paper_example():
    # n_e = 250000 on a 2:1 domain -> w_b = 500, h_b = 250
    m = mg.grid_mesh(500, 250, 2.0, 1.0)
    assert m.ne == 250000
    key, perm, grid = core.hilbert_order(m.vxy, m.tri)
    assert grid == (500, 250)


def _quadrant_mesh(order):
    """One small triangle inside each quadrant of the unit square."""
    tris, vxy = [], []
    for (i, j) in order:
        b = len(vxy)
        x0, y0 = i * 0.5, j * 0.5
        vxy += [(x0, y0), (x0 + 0.5, y0), (x0, y0 + 0.5)]
        tris.append((b, b + 1, b + 2))
    return np.array(vxy), np.array(tris, np.int32)


def test_quadrant_order_follows_order1_curve():
    # 4 elements -> w_b = h_b = 2: quadrants visited LL, UL, UR, LR (Listing 1 order 1)
    order = [(1, 0), (0, 1), (0, 0), (1, 1)]  # input: LR, UL, LL, UR
    vxy, tri = _quadrant_mesh(order)
    key, perm, grid = core.hilbert_order(vxy, tri)
    assert grid == (2, 2)
    assert [order[e] for e in perm] == [(0, 0), (0, 1), (1, 1), (1, 0)]
    assert key.tolist() == [3, 1, 0, 2]


def test_single_element():
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    tri = np.array([[0, 1, 2]], np.int32)
    key, perm, grid = core.hilbert_order(vxy, tri)
    assert perm.tolist() == [0] and key.tolist() == [0] and grid == (1, 1)


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_small_meshes(seed):
    rng = np.random.default_rng(seed)
    nx, ny = int(rng.integers(1, 6)), int(rng.integers(1, 5))
    m = mg.shuffle(mg.grid_mesh(nx, ny, float(rng.uniform(0.5, 3)), 1.0, alpha=0.2, seed=seed), seed + 10, seed + 20)
    key, perm, (wb, hb) = core.hilbert_order(m.vxy, m.tri)
    E = m.ne
    assert sorted(perm.tolist()) == list(range(E))
    # brute force: every element's key is the path position of the cell its
    # centroid falls in; L lists elements by (key, input id)
    path = core.gilbert_path(wb, hb)
    pos = {(int(x), int(y)): s for s, (x, y) in enumerate(path)}
    lo = m.vxy.min(axis=0)
    hi = m.vxy.max(axis=0)
    for e in range(E):
        c = m.vxy[m.tri[e]]
        cx = ((c[0, 0] + c[1, 0]) + c[2, 0]) / 3.0
        cy = ((c[0, 1] + c[1, 1]) + c[2, 1]) / 3.0
        i = min(int(np.floor((cx - lo[0]) * (wb / (hi[0] - lo[0])))), wb - 1)
        j = min(int(np.floor((cy - lo[1]) * (hb / (hi[1] - lo[1])))), hb - 1)
        assert key[e] == pos[(i, j)]
    expect = sorted(range(E), key=lambda e: (int(key[e]), e))
    assert perm.tolist() == expect


def test_random_order_is_bijection_and_seeded():
    a = core.random_order(1000, 7)
    b = core.random_order(1000, 7)
    c = core.random_order(1000, 8)
    assert sorted(a.tolist()) == list(range(1000))
    assert (a == b).all() and not (a == c).all()


def test_splitmix64_published_sequence():
    # Reading R16 keys the library-side random order by SplitMix64 (Steele, Lea and Flood 2014).
    # The generator's published reference output for state 0 starts e220a8397b1dcdaf,
    # 6e789e6aa1b965f4: output k is the mixer of k times the golden-ratio increment.
    g = 0x9E3779B97F4A7C15
    assert core.splitmix64(0) == 0xE220A8397B1DCDAF
    assert core.splitmix64(g) == 0x6E789E6AA1B965F4
    # the order is the stable sort of ids by splitmix64(seed ^ id)
    perm = core.random_order(300, 5)
    keys = [core.splitmix64(5 ^ e) for e in range(300)]
    assert perm.tolist() == sorted(range(300), key=lambda e: (keys[e], e))


def test_first_touch_brute_force():
    rng = np.random.default_rng(3)
    N = 40
    mu = rng.integers(0, N, size=(25, 6)).astype(np.int32)
    mu[0, :] = np.arange(6)
    used = np.unique(mu)
    remap = {int(g): k for k, g in enumerate(used)}
    mu = np.vectorize(remap.get)(mu).astype(np.int32)
    N = len(used)
    perm, mu2 = core.first_touch(mu, N)
    assert sorted(perm.tolist()) == list(range(N))
    # relabelling is consistent
    assert (perm[mu2] == mu).all()
    # labels appear in increasing order of first occurrence
    seen = []
    for g in mu2.ravel():
        if g not in seen:
            seen.append(int(g))
    assert seen == list(range(N))
