// chunks.cpp -- host-side chunk metadata for the deterministic, conflict-free
// scatter of the step kernel (product path).
//
// The paper avoids the scatter race of Algorithm 2 by
// colouring the whole mesh and running colours one after another.  On the GPU
// the race is removed at CTA scale instead: elements are cut into chunks of B
// consecutive elements (consecutive along the Hilbert order, so a chunk is a
// compact patch of the domain) and each chunk is processed by one CTA:
//   * nodes touched by a single chunk ("interior") are reduced in shared memory
//     through a per-chunk node CSR (each node's element contributions form a
//     contiguous run, summed in ascending entry order) and finalised there;
//   * nodes touched by several chunks ("shared") get one SLOT per touching
//     chunk, node-major.  The step kernel's producer warp gathers the U^n of
//     a chunk's shared nodes with cp.async; its consumers write the chunk's
//     partial K U sums into the slots; the fix-up kernel adds a node's slots
//     (a contiguous run, ascending chunk order) and updates the node.
// Every summation order is fixed, so results are bitwise reproducible.
//
// Internal node numbering: interior nodes of chunk c occupy [i0_c, i0_c+nint_c),
// i0_c even (16-byte aligned for TMA bulk copies, at most one hole per chunk),
// ordered by descending entry count then ascending incoming id (so warps of
// the reduction see nodes of equal degree); shared nodes follow at
// [N_int, N_int+N_sh): non-interface ones by (owner chunk, id) -- the owner is
// the last chunk touching the node, and a chunk's owned nodes form the range
// [own0[c], own0[c+1]) -- then the rank-interface ones (multi-GPU) in
// ascending id.
//
// Parallel structure: one pass sorts every chunk's node ids (OpenMP over
// chunks); the per-node facts (first chunk, number of touching chunks) come
// from atomics on those per-chunk unique lists; everything per chunk after that
// is again independent.  Only cheap loops over nodes/slots are serial.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sem_internal.h"

namespace sem {

namespace {
struct Trace {  // SEM_TRACE=1: phase timings of the builder on stderr
    bool on = getenv("SEM_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[sem build_chunks] %-28s %8.1f ms\n", what,
                std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

inline int64_t align2(int64_t v) { return (v + 1) & ~int64_t(1); }

struct Uniq {  // unique node of a chunk
    int32_t g;    // incoming node id
    int32_t cnt;  // entries of the chunk that reference it
};
}  // namespace

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
    Trace tr;

    // ---- per chunk: sorted unique node ids with entry counts; per node: first
    //      touching chunk and number of touching chunks (atomics, order-free) ----
    std::vector<std::vector<Uniq>> uq(nch);
    std::vector<int32_t> firstc(N, INT32_MAX), lastc(N, -1), nref(N, 0);
    bool bad_id = false;
#pragma omp parallel
    {
    std::vector<int32_t> ids;
    ids.reserve((size_t)B * Np);
#pragma omp for schedule(dynamic, 64)
    for (int64_t c = 0; c < nch; c++) {
        const int64_t e0 = c * B, e1 = std::min<int64_t>(E, e0 + B);
        ids.assign(mu + e0 * Np, mu + e1 * Np);
        std::sort(ids.begin(), ids.end());
        std::vector<Uniq> &U = uq[c];
        U.reserve(ids.size() / 2 + 16);
        for (size_t k = 0; k < ids.size();) {
            size_t j = k;
            while (j < ids.size() && ids[j] == ids[k]) j++;
            U.push_back({ids[k], (int32_t)(j - k)});
            k = j;
        }
        if (U.front().g < 0 || U.back().g >= N) {
            bad_id = true;
            continue;
        }
        for (const Uniq &u : U) {
            __atomic_fetch_add(&nref[u.g], 1, __ATOMIC_RELAXED);
            int32_t cur = __atomic_load_n(&firstc[u.g], __ATOMIC_RELAXED);
            while ((int32_t)c < cur &&
                   !__atomic_compare_exchange_n(&firstc[u.g], &cur, (int32_t)c, true, __ATOMIC_RELAXED,
                                                __ATOMIC_RELAXED)) {
            }
            int32_t hi = __atomic_load_n(&lastc[u.g], __ATOMIC_RELAXED);
            while ((int32_t)c > hi &&
                   !__atomic_compare_exchange_n(&lastc[u.g], &hi, (int32_t)c, true, __ATOMIC_RELAXED,
                                                __ATOMIC_RELAXED)) {
            }
        }
        U.shrink_to_fit();
    }
    }
    if (bad_id) {
        err = "build_chunks: node id out of range";
        return false;
    }
    for (int64_t g = 0; g < N; g++)
        if (nref[g] == 0) {
            err = "node " + std::to_string(g) + " is not used by any element";
            return false;
        }
    tr.mark("chunk sort + node facts");

    // ---- classification: nodes touched by another rank are always shared ----
    auto forced = [&](int64_t g) { return force_shared && force_shared[g]; };
    auto interior = [&](int64_t g) { return nref[g] == 1 && !forced(g); };

    std::vector<int64_t> nint(nch, 0);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nch; c++) {
        int64_t n = 0;
        for (const Uniq &u : uq[c]) n += interior(u.g);
        nint[c] = n;
    }
    m.i0.assign(nch + 1, 0);
    for (int64_t c = 0; c < nch; c++) m.i0[c + 1] = (int32_t)align2(m.i0[c] + nint[c]);
    m.N_int = m.i0[nch];

    // shared indices: non-interface by (owner chunk = last touching chunk, id) -- the nodes a
    // chunk owns form the contiguous range [own0[c], own0[c+1]) that K7 finalises after
    // the chunk (one launch walks the chunks in ascending order, so the owner comes last) --
    // then interface in ascending id
    m.int_of.assign(N, -1);
    std::vector<int32_t> sh_index(N, -1);
    int64_t nsh = 0, nif = 0;
    m.own0.assign(nch + 1, 0);
    for (int64_t g = 0; g < N; g++)
        if (!interior(g)) {
            nsh++;
            nif += forced(g);
            if (!forced(g)) m.own0[lastc[g] + 1]++;
        }
    for (int64_t c = 0; c < nch; c++) m.own0[c + 1] += m.own0[c];
    {
        std::vector<int32_t> cur(m.own0.begin(), m.own0.end() - 1);
        int64_t sf = nsh - nif;
        for (int64_t g = 0; g < N; g++) {  // ascending g within each owner
            if (interior(g)) continue;
            const int64_t k = forced(g) ? sf++ : cur[lastc[g]]++;
            sh_index[g] = (int32_t)k;
            m.int_of[g] = (int32_t)(m.N_int + k);
        }
    }
    m.N_sh = nsh;
    m.N_if = nif;
    m.N_tot = m.N_int + nsh;

    // interior ids: per chunk, descending entry count then ascending id (stable counting
    // sort; the unique list is ascending in id).  Element-interior nodes (lattice-interior
    // local p) come after the count-1 nodes: K7 finalises them per element.
    std::vector<uint8_t> inner;
    if (lattice_n_interior(Np) > 0) {
        inner.assign(N, 0);
        for (int p = 0; p < Np; p++)
            if (lattice_interior(Np, p))
                for (int64_t e = 0; e < E; e++) inner[mu[e * Np + p]] = 1;
    }
    auto bucket = [&](const Uniq &u) { return (!inner.empty() && inner[u.g]) ? 255 : 255 - std::min(u.cnt, 255); };
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t c = 0; c < nch; c++) {
        int off[256] = {0};
        for (const Uniq &u : uq[c])
            if (interior(u.g)) off[bucket(u)]++;
        int acc = 0;
        for (int b = 0; b < 256; b++) { const int h = off[b]; off[b] = acc; acc += h; }
        for (const Uniq &u : uq[c])
            if (interior(u.g)) m.int_of[u.g] = (int32_t)(m.i0[c] + off[bucket(u)]++);
    }
    tr.mark("internal numbering");

    // ---- per-chunk shared lists: descending local count, then ascending index ----
    std::vector<std::vector<int32_t>> lists(nch);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nch; c++) {
        std::vector<std::pair<int32_t, int32_t>> key;  // (-count, s)
        for (const Uniq &u : uq[c])
            if (!interior(u.g)) key.push_back({-u.cnt, sh_index[u.g]});
        std::sort(key.begin(), key.end());
        lists[c].reserve(key.size());
        for (auto &pr : key) lists[c].push_back(pr.second);
    }
    // Boundary chunks (touching a rank-interface node) run first so that the
    // interface exchange overlaps the interior chunks.
    for (int64_t c = 0; c < nch; c++) {
        bool bnd = false;
        for (int32_t sidx : lists[c]) bnd |= sidx >= nsh - nif;
        (bnd ? m.bnd_chunks : m.int_chunks).push_back((int32_t)c);
    }
    tr.mark("shared lists");

    // ---- node-major slots: shared node s owns [sh_pstart[s], sh_pstart[s+1]),
    //      one per touching chunk in ascending chunk order ----
    m.sh_pstart.assign(nsh + 1, 0);
    for (int64_t g = 0; g < N; g++)
        if (sh_index[g] >= 0) m.sh_pstart[sh_index[g] + 1] = nref[g];
    for (int64_t s = 0; s < nsh; s++) m.sh_pstart[s + 1] += m.sh_pstart[s];
    m.n_slots = nsh ? m.sh_pstart[nsh] : 0;
    m.s0.assign(nch + 1, 0);
    // chunk blocks of the per-chunk lists start on multiples of 8 entries (16-byte
    // aligned TMA copies of the u16 shl_cr block)
    for (int64_t c = 0; c < nch; c++) m.s0[c + 1] = (int32_t)((m.s0[c] + (int64_t)lists[c].size() + 7) & ~int64_t(7));
    for (int64_t c = 0; c < nch; c++) m.max_nsh = std::max(m.max_nsh, (int)((lists[c].size() + 7) & ~size_t(7)));
    m.shl_node.assign((size_t)m.s0[nch] + 8, 0);
    m.shl_slot.assign((size_t)m.s0[nch] + 8, 0);
    m.shl_cr.assign((size_t)m.s0[nch] + 8, 0);
    {
        std::vector<int32_t> cursor(nsh, 0);
        for (int64_t c = 0; c < nch; c++) {  // ascending chunk order -> slot order within a node
            int32_t k = m.s0[c];
            for (int32_t sidx : lists[c]) {
                const int32_t cnt = m.sh_pstart[sidx + 1] - m.sh_pstart[sidx];
                if (cnt > 255) {
                    err = "build_chunks: a node is shared by more than 255 chunks";
                    return false;
                }
                m.shl_node[k] = sidx;
                m.shl_cr[k] = (uint16_t)((cnt << 8) | cursor[sidx]);
                m.shl_slot[k] = m.sh_pstart[sidx] + cursor[sidx]++;
                k++;
            }
        }
    }
    tr.mark("slots");

    // ---- local indices, the per-chunk node CSR and the chunk descriptor ----
    m.lidx.assign((size_t)nch * Np * B, 0);
    m.lpos.assign((size_t)nch * Np * B, 0);
    m.cmeta.assign((size_t)nch * 8, 0);
    std::vector<int32_t> nlocal(nch, 0);
    int max_local = 0, max_win = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : max_local, max_win)
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
        std::vector<std::pair<int32_t, int32_t>> pos_of;  // (shared index, local position)
        pos_of.reserve(L.size());
        for (int32_t k = 0; k < ns; k++) pos_of.push_back({L[k], k});
        std::sort(pos_of.begin(), pos_of.end());
        for (int64_t e = e0; e < e1; e++) {
            const int t = (int)(e - e0);
            for (int p = 0; p < Np; p++) {
                const int32_t g = mu[e * Np + p];
                int loc;
                if (interior(g)) loc = m.int_of[g] - i0;
                else loc = ni_al + std::lower_bound(pos_of.begin(), pos_of.end(),
                                                    std::make_pair(sh_index[g], (int32_t)-1))->second;
                m.lidx[(size_t)c * Np * B + (size_t)p * B + t] = (uint16_t)loc;
            }
        }
        int32_t *cm = &m.cmeta[(size_t)c * 8];
        cm[0] = i0;
        cm[1] = ni;
        cm[2] = m.s0[c];
        cm[3] = ns;
        cm[4] = 0;
        cm[5] = (int32_t)(e1 - e0);
        cm[6] = ni_al;
    }
    tr.mark("local indices");
    // Jagged diagonals (JDS) of the per-chunk node sums.  The local nodes of a
    // segment (interior [0, nint), shared [ni_al, ni_al + ns)) are sorted by
    // entry count, descending; diagonal d holds the d-th entry of every node
    // with more than d entries, nodes in local order.  jds[c][32 s + d] = start
    // of diagonal d of segment s in the chunk's entry buffer (absolute);
    // cmeta[4] / cmeta[7] = end of segment 0 / 1.  lpos[e] = jds[...][rank] +
    // node index in its segment, rank = position of entry e = p*B + t among
    // its node's entries in ascending e.  A node's sum runs over d in order:
    // the same order as a CSR run, and a warp's lanes read consecutive words.
    m.jds.assign((size_t)nch * kJdsW * 2, 0);
    int max_cnt = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : max_cnt)
    for (int64_t c = 0; c < nch; c++) {
        const int nl = nlocal[c];
        const int ne = (int)(std::min<int64_t>(E, (c + 1) * B) - c * B);
        int32_t *cm = &m.cmeta[(size_t)c * 8];
        const int ni = cm[1], ni_al = cm[6];
        std::vector<int> cnt(nl, 0), rank(nl, 0);
        const uint16_t *li = &m.lidx[(size_t)c * Np * B];
        for (int p = 0; p < Np; p++)
            for (int t = 0; t < ne; t++) cnt[li[p * B + t]]++;
        uint16_t *jd = &m.jds[(size_t)c * kJdsW * 2];
        int base = 0;
        for (int sg = 0; sg < 2; sg++) {
            const int a = sg == 0 ? 0 : ni_al, b = sg == 0 ? ni : nl;
            int nd[kJdsW + 1] = {0};
            for (int i = a; i < b; i++) {
                if (cnt[i] > max_cnt) max_cnt = cnt[i];
                for (int d = 0; d < cnt[i] && d < kJdsW; d++) nd[d]++;
            }
            for (int d = 0; d < kJdsW; d++) { jd[sg * kJdsW + d] = (uint16_t)base; base += nd[d]; }
            cm[sg == 0 ? 4 : 7] = base;
        }
        uint16_t *lpo = &m.lpos[(size_t)c * Np * B];
        for (int p = 0; p < Np; p++)
            for (int t = 0; t < ne; t++) {
                const int i = li[p * B + t];
                const int sg = i < ni_al ? 0 : 1;
                const int r = rank[i]++;
                if (r < kJdsW) lpo[p * B + t] = (uint16_t)(jd[sg * kJdsW + r] + (sg == 0 ? i : i - ni_al));
            }
    }
    if (max_cnt > kJdsW) {
        err = "build_chunks: a node has more than 64 entries in one chunk";
        return false;
    }
    m.max_local = max_local;
    m.max_win = max_win;
    m.max_count = max_cnt;
    m.max_colors = 0;
    tr.mark("JDS");
    return true;
}

}  // namespace sem
