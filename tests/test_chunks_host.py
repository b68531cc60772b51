"""Host logic of the chunk builder (csrc/chunks.cpp, the twin of the GPU
builder) on CPU through sem_debug_chunk_stats: the interior / shared split, the
internal numbering and the slot count against brute force with Python sets."""
import numpy as np
import pytest

from oracle import core
from paper_2104_08416_b200 import meshgen as mg
from paper_2104_08416_b200 import sem as S


def reordered_mu(name, scale, P=None):
    pb = mg.config(name, scale, degree=P) if P else mg.config(name, scale)
    m = pb.mesh
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, pb.P)
    _, perm, _ = core.hilbert_order(m.vxy, m.tri)
    _, mu_ft = core.first_touch(mu[perm], N)
    return mu_ft, N


@pytest.mark.parametrize("name,scale,P,B", [("C1", 1, None, 256), ("C2", 16, None, 256), ("C2", 16, None, 128),
                                            ("C3", 40, None, 192), ("B1", 30, 5, 128), ("B1", 40, 7, 64)])
def test_chunk_builder_brute_force(name, scale, P, B):
    mu, N = reordered_mu(name, scale, P)
    E, Np = mu.shape
    st = S.sem_debug_chunk_stats(mu, N, B, want_maps=True)
    nch = (E + B - 1) // B
    assert st["nchunks"] == nch
    touching = [set() for _ in range(N)]
    for c in range(nch):
        for g in np.unique(mu[c * B:(c + 1) * B]):
            touching[g].add(c)
    interior = np.array([len(s) == 1 for s in touching])
    nsh = int((~interior).sum())
    assert st["N_sh"] == nsh
    assert st["sum_nint"] == int(interior.sum())
    assert st["n_slots"] == sum(len(s) for s in touching if len(s) > 1)
    int_of, cm = st["int_of"], st["cmeta"]
    # internal ids: distinct; interior nodes inside their chunk's window, shared after N_int
    assert len(set(int_of.tolist())) == N
    N_int = st["N_int"]
    assert (int_of[~interior] >= N_int).all() and (int_of[~interior] < N_int + nsh).all()
    for g in np.nonzero(interior)[0][:: max(1, N // 2000)]:
        c = next(iter(touching[g]))
        i0, nint = cm[c, 0], cm[c, 1]
        assert i0 % 2 == 0 and i0 <= int_of[g] < i0 + nint
    # shared nodes by (owner = last touching chunk, id) (no rank-interface nodes here), so
    # each chunk owns a contiguous range of shared indices
    sh_ids = np.nonzero(~interior)[0]
    owner = np.array([max(touching[g]) for g in sh_ids])
    order = np.lexsort((sh_ids, owner))
    assert np.array_equal(int_of[sh_ids[order]], N_int + np.arange(nsh))
    own0 = st["own0"]
    assert own0.shape == (nch + 1,) and own0[0] == 0 and own0[-1] == nsh
    assert np.array_equal(np.diff(own0), np.bincount(owner, minlength=nch))
    # per-chunk counts and element counts
    for c in range(nch):
        ne = min(E, (c + 1) * B) - c * B
        assert cm[c, 5] == ne
        nodes = set(np.unique(mu[c * B:c * B + ne]).tolist())
        assert cm[c, 1] == sum(1 for g in nodes if interior[g])
        assert cm[c, 3] == sum(1 for g in nodes if not interior[g])
        assert cm[c, 6] == cm[c, 1] + (cm[c, 1] & 1)


def lattice_interior_positions(P):
    """Local positions p (lattice order: row j outer, i inner) of the element's own
    interior nodes: 1 <= i, 1 <= j, i + j <= P - 1."""
    out, p = [], 0
    for j in range(P + 1):
        for i in range(P + 1 - j):
            if i >= 1 and j >= 1 and i + j <= P - 1:
                out.append(p)
            p += 1
    return out


@pytest.mark.parametrize("name,scale,P,B", [("C2", 16, None, 192), ("C3", 40, None, 256), ("B1", 30, 5, 128)])
def test_element_interior_nodes_close_the_interior_segment(name, scale, P, B):
    """K7 finalises each element's own interior nodes in the element phase and its node
    phase covers only the first nint - ne * nI interior ids of a chunk: the builder must
    place exactly those nodes (one entry each) at the end of every chunk's window, and
    keep the other interior nodes in descending entry count."""
    mu, N = reordered_mu(name, scale, P)
    E, Np = mu.shape
    deg = int(round((np.sqrt(8 * Np + 1) - 3) / 2))
    inner_p = lattice_interior_positions(deg)
    assert len(inner_p) == (deg - 1) * (deg - 2) // 2
    st = S.sem_debug_chunk_stats(mu, N, B, want_maps=True)
    int_of, cm = st["int_of"], st["cmeta"]
    nch = (E + B - 1) // B
    for c in list(range(0, nch, max(1, nch // 25))) + [nch - 1]:
        i0, nint, ne = cm[c, 0], cm[c, 1], cm[c, 5]
        rows = mu[c * B:c * B + ne]
        inner = rows[:, inner_p].ravel()
        assert len(np.unique(inner)) == inner.size  # one entry each
        tail0 = i0 + nint - inner.size
        assert np.array_equal(np.sort(int_of[inner]), np.arange(tail0, i0 + nint))
        # the rest of the window: descending entry count
        ids, cnt = np.unique(rows, return_counts=True)
        win = (int_of[ids] >= i0) & (int_of[ids] < tail0)
        order = np.argsort(int_of[ids[win]])
        assert (np.diff(cnt[win][order]) <= 0).all()


def test_high_valence_fan_fits_a_chunk():
    """A vertex held by 48 elements of one chunk (more than round 1's limit of 32 entries per
    node and chunk): the chunk builder accepts it (kJdsW = 64) and counts its entries."""
    m = mg.fan_mesh(48)
    t = core.orient(m.vxy, m.tri)
    mu, N = core.canonical_nodes(t, m.nv, 3)
    _, perm, _ = core.hilbert_order(m.vxy, m.tri)
    _, mu_ft = core.first_touch(mu[perm], N)
    st = S.sem_debug_chunk_stats(mu_ft, N, 256)
    assert st["max_count"] == 48
