// chunks.cpp -- host-side chunk metadata for the deterministic, conflict-free
// scatter of the step kernel (product path).
//
// The paper avoids the scatter race of Algorithm 2 by
// colouring the whole mesh and running colours one after another.  On the GPU
// we keep the colouring idea at CTA scale: elements are cut into chunks of B
// consecutive elements (consecutive along the Hilbert order, so a chunk is a
// compact patch of the domain) and each chunk is processed by one CTA:
//   * nodes touched by a single chunk ("interior") are summed in shared memory
//     in a fixed colour order and finalised by that CTA;
//   * nodes touched by several chunks ("shared") get one SLOT per touching
//     chunk, node-major.  The step kernel's producer warp gathers the U^n of
//     a chunk's shared nodes with cp.async; its consumers write the chunk's
//     partial K U sums into the slots; the fix-up kernel adds a node's slots
//     (a contiguous run, ascending chunk order) and updates the node.
// Both summation orders are fixed, so results are bitwise reproducible.
// (Slot layout: node-major -- see below.)
//
// Internal node numbering: interior nodes of chunk c occupy [i0_c, i0_c+nint_c),
// i0_c even (16-byte aligned for TMA bulk copies, one hole at most per chunk),
// in ascending incoming id; shared nodes follow at [N_int, N_int+N_sh).
#include <algorithm>
#include <cstring>

#include "sem_internal.h"

namespace sem {

static inline int64_t align2(int64_t v) { return (v + 1) & ~int64_t(1); }

bool build_chunks(const int32_t *mu, int64_t E, int Np, int64_t N, int B, ChunkMeta &m,
                  std::string &err, const uint8_t *force_shared) {
    if (E <= 0 || N <= 0 || B <= 0 || B > 1024 || (B % 16) != 0 || Np > kMaxNp) {
        err = "build_chunks: bad arguments";
        return false;
    }
    if ((int64_t)B * Np > 32767) {
        err = "build_chunks: chunk too large for 16-bit local indices";
        return false;
    }
    m = ChunkMeta();
    m.B = B;
    m.Np = Np;
    m.E = E;
    m.N = N;
    const int64_t nch = (E + B - 1) / B;
    m.nchunks = nch;

    // Pass 1: first chunk and number of distinct chunks touching each node.
    std::vector<int32_t> firstc(N, -1), lastc(N, -1), nref(N, 0);
    std::vector<uint8_t> refcnt(N, 0);  // element entries per node (saturating)
    for (int64_t e = 0; e < E; e++) {
        const int32_t c = (int32_t)(e / B);
        for (int p = 0; p < Np; p++) {
            const int32_t g = mu[e * Np + p];
            if (g < 0 || g >= N) {
                err = "build_chunks: node id out of range in element " + std::to_string(e);
                return false;
            }
            if (refcnt[g] < 255) refcnt[g]++;
            if (lastc[g] != c) {  // chunks are visited in increasing order
                if (firstc[g] < 0) firstc[g] = c;
                lastc[g] = c;
                nref[g]++;
            }
        }
    }
    for (int64_t g = 0; g < N; g++)
        if (firstc[g] < 0) {
            err = "node " + std::to_string(g) + " is not used by any element";
            return false;
        }

    // Nodes touched by another rank (multi-GPU interface) are shared even when a
    // single local chunk touches them; they go last in the shared range.
    if (force_shared)
        for (int64_t g = 0; g < N; g++)
            if (force_shared[g] && nref[g] == 1) nref[g] = -1;  // marker: 1 local chunk, forced
    auto is_interior = [&](int64_t g) { return nref[g] == 1; };
    auto forced = [&](int64_t g) { return force_shared && force_shared[g]; };
    auto nref_local = [&](int64_t g) { return nref[g] < 0 ? 1 : nref[g]; };

    // Interior windows (even-aligned starts).
    std::vector<int64_t> nint(nch, 0);
    int64_t nsh = 0, nif = 0;
    for (int64_t g = 0; g < N; g++) {
        if (is_interior(g)) nint[firstc[g]]++;
        else { nsh++; if (forced(g)) nif++; }
    }
    m.i0.assign(nch + 1, 0);
    for (int64_t c = 0; c < nch; c++) m.i0[c + 1] = (int32_t)align2(m.i0[c] + nint[c]);
    m.N_int = m.i0[nch];
    m.N_sh = nsh;
    m.N_if = nif;
    m.N_tot = m.N_int + nsh;
    m.int_of.assign(N, -1);
    std::vector<int32_t> sh_index(N, -1);
    {
        // interior nodes of a chunk: descending entry count, then ascending id
        // (warps of the reduction then see nodes of equal degree)
        std::vector<int32_t> cur(m.i0.begin(), m.i0.end() - 1), order(m.N_int > 0 ? m.N_int : 1);
        int64_t s = 0, sf = nsh - nif;
        for (int64_t g = 0; g < N; g++) {
            if (is_interior(g)) order[cur[firstc[g]]++] = (int32_t)g;
            else if (!forced(g)) { sh_index[g] = (int32_t)s; m.int_of[g] = (int32_t)(m.N_int + s); s++; }
            else { sh_index[g] = (int32_t)sf; m.int_of[g] = (int32_t)(m.N_int + sf); sf++; }
        }
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t c = 0; c < nch; c++) {
            std::stable_sort(order.begin() + m.i0[c], order.begin() + m.i0[c] + nint[c],
                             [&](int32_t a, int32_t b) { return refcnt[a] > refcnt[b]; });
            for (int64_t k = m.i0[c]; k < m.i0[c] + nint[c]; k++) m.int_of[order[k]] = (int32_t)k;
        }
    }

    // Per-chunk shared lists (sorted, unique).
    std::vector<std::vector<int32_t>> lists(nch);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nch; c++) {
        std::vector<int32_t> &L = lists[c];
        const int64_t e0 = c * B, e1 = std::min<int64_t>(E, e0 + B);
        for (int64_t e = e0; e < e1; e++)
            for (int p = 0; p < Np; p++) {
                const int32_t s = sh_index[mu[e * Np + p]];
                if (s >= 0) L.push_back(s);
            }
        // by descending local entry count, then ascending shared index
        std::sort(L.begin(), L.end());
        std::vector<std::pair<int32_t, int32_t>> cnt;  // (-count, s)
        for (size_t k = 0; k < L.size();) {
            size_t j = k;
            while (j < L.size() && L[j] == L[k]) j++;
            cnt.push_back({-(int32_t)(j - k), L[k]});
            k = j;
        }
        std::sort(cnt.begin(), cnt.end());
        L.clear();
        for (auto &pr : cnt) L.push_back(pr.second);
    }
    // Boundary chunks (touching a rank-interface node) run first so that the
    // interface exchange overlaps the interior chunks.
    for (int64_t c = 0; c < nch; c++) {
        bool bnd = false;
        for (int32_t sidx : lists[c]) bnd |= sidx >= nsh - nif;
        (bnd ? m.bnd_chunks : m.int_chunks).push_back((int32_t)c);
    }
    // Slots are node-major: shared node s owns [sh_pstart[s], sh_pstart[s+1]),
    // one per touching chunk in ascending chunk order (so the fix-up sums a
    // contiguous run).  Each chunk lists, contiguously, the shared index and the
    // slot of every shared node it touches (block start 16-byte aligned).
    m.sh_pstart.assign(nsh + 1, 0);
    for (int64_t g = 0; g < N; g++)
        if (sh_index[g] >= 0) m.sh_pstart[sh_index[g] + 1] = nref_local(g);
    for (int64_t s = 0; s < nsh; s++) m.sh_pstart[s + 1] += m.sh_pstart[s];
    m.n_slots = nsh ? m.sh_pstart[nsh] : 0;
    m.s0.assign(nch + 1, 0);
    for (int64_t c = 0; c < nch; c++) m.s0[c + 1] = (int32_t)((m.s0[c] + (int64_t)lists[c].size() + 3) & ~int64_t(3));
    for (int64_t c = 0; c < nch; c++) m.max_nsh = std::max(m.max_nsh, (int)((lists[c].size() + 3) & ~size_t(3)));
    m.shl_node.assign((size_t)m.s0[nch] + 4, 0);
    m.shl_slot.assign((size_t)m.s0[nch] + 4, 0);
    {
        std::vector<int32_t> cursor(nsh, 0);
        for (int64_t c = 0; c < nch; c++) {  // ascending chunk order -> slot order within a node
            int32_t k = m.s0[c];
            for (int32_t sidx : lists[c]) {
                m.shl_node[k] = sidx;
                m.shl_slot[k] = m.sh_pstart[sidx] + cursor[sidx]++;
                k++;
            }
        }
    }

    // Local indices, the per-chunk node CSR (local node -> entries p*B + t in
    // ascending order; this fixes the summation order), a per-chunk greedy
    // colouring (first fit in element order; used by diagnostics only), and
    // the per-chunk descriptor.
    m.lidx.assign((size_t)nch * Np * B, 0);
    m.color.assign((size_t)nch * B, 255);
    m.cmeta.assign((size_t)nch * 8, 0);
    m.lp0.assign(nch + 1, 0);
    std::vector<int32_t> nlocal(nch, 0);
    int max_local = 0, max_win = 0, max_col = 0;
    bool bad_color = false;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : max_local, max_win, max_col)
    for (int64_t c = 0; c < nch; c++) {
        const int64_t e0 = c * B, e1 = std::min<int64_t>(E, e0 + B);
        const int32_t i0 = m.i0[c];
        const int32_t ni = (int32_t)nint[c];
        const int32_t ni_al = (int32_t)align2(ni);
        const std::vector<int32_t> &L = lists[c];
        const int32_t ns = (int32_t)L.size();
        const int nl = ni_al + (int)align2(ns);  // u-buffer length (TMA sizes are even)
        nlocal[c] = ni_al + ns;
        if (nl > max_local) max_local = nl;
        if (ni_al > max_win) max_win = ni_al;
        std::vector<uint32_t> used(nl, 0u);
        std::vector<std::pair<int32_t, int32_t>> pos_of;  // (shared index, local position)
        pos_of.reserve(L.size());
        for (int32_t k = 0; k < ns; k++) pos_of.push_back({L[k], k});
        std::sort(pos_of.begin(), pos_of.end());
        int ncol = 0;
        for (int64_t e = e0; e < e1; e++) {
            const int t = (int)(e - e0);
            uint32_t forb = 0;
            uint16_t li[kMaxNp];
            for (int p = 0; p < Np; p++) {
                const int32_t g = mu[e * Np + p];
                int loc;
                if (sh_index[g] < 0) loc = m.int_of[g] - i0;
                else loc = ni_al + std::lower_bound(pos_of.begin(), pos_of.end(),
                                                    std::make_pair(sh_index[g], (int32_t)-1))->second;
                li[p] = (uint16_t)loc;
                m.lidx[(size_t)c * Np * B + (size_t)p * B + t] = (uint16_t)loc;
                forb |= used[loc];
            }
            if (forb == 0xFFFFFFFFu) {
                bad_color = true;
                continue;
            }
            int col = 0;
            while (forb & (1u << col)) col++;
            m.color[(size_t)c * B + t] = (uint8_t)col;
            for (int p = 0; p < Np; p++) used[li[p]] |= (1u << col);
            if (col + 1 > ncol) ncol = col + 1;
        }
        int32_t *cm = &m.cmeta[(size_t)c * 8];
        cm[0] = i0;
        cm[1] = ni;
        cm[2] = m.s0[c];
        cm[3] = ns;
        cm[4] = ncol;
        cm[5] = (int32_t)(e1 - e0);
        cm[6] = ni_al;
        if (ncol > max_col) max_col = ncol;
    }
    if (bad_color) {
        err = "build_chunks: more than 32 colours needed inside a chunk";
        return false;
    }
    // CSR blocks: chunk c owns lptr[lp0[c] .. lp0[c] + nlocal+1) (start aligned
    // to 8 entries = 16 bytes for TMA) and lpos[c*Np*B .. (c+1)*Np*B).
    for (int64_t c = 0; c < nch; c++) m.lp0[c + 1] = (int32_t)((m.lp0[c] + nlocal[c] + 1 + 7) & ~7);
    m.lptr.assign((size_t)m.lp0[nch] + 8, 0);
    m.lpos.assign((size_t)nch * Np * B, 0);
    int max_lp = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : max_lp)
    for (int64_t c = 0; c < nch; c++) {
        const int nl = nlocal[c];
        const int ne = (int)(std::min<int64_t>(E, (c + 1) * B) - c * B);
        std::vector<int> cnt(nl + 1, 0);
        const uint16_t *li = &m.lidx[(size_t)c * Np * B];
        for (int p = 0; p < Np; p++)
            for (int t = 0; t < ne; t++) cnt[li[p * B + t] + 1]++;
        for (int i = 0; i < nl; i++) cnt[i + 1] += cnt[i];
        uint16_t *lp = &m.lptr[m.lp0[c]];
        for (int i = 0; i <= nl; i++) lp[i] = (uint16_t)cnt[i];
        // entries visited in ascending e = p*B + t order -> each node's run is
        // ascending; lpos[e] = CSR position of entry e (where y_e[p] goes)
        uint16_t *lpo = &m.lpos[(size_t)c * Np * B];
        for (int p = 0; p < Np; p++)
            for (int t = 0; t < ne; t++) lpo[p * B + t] = (uint16_t)(cnt[li[p * B + t]]++);
        m.cmeta[(size_t)c * 8 + 7] = m.lp0[c];
        const int w = (nl + 1 + 7) & ~7;
        if (w > max_lp) max_lp = w;
    }
    m.max_lptr = max_lp;
    m.max_local = max_local;
    m.max_win = max_win;
    m.max_colors = max_col;
    return true;
}

}  // namespace sem
