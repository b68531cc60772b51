// chunks.cpp -- host-side chunk metadata for the deterministic, conflict-free
// scatter of the step kernel (product path).
//
// The paper avoids the scatter race of Algorithm 2 by
// colouring the whole mesh and running colours one after another.  On the GPU
// we keep the colouring idea but at CTA scale: elements are cut into chunks of
// B consecutive elements (consecutive along the Hilbert order, so a chunk is a
// compact patch of the domain), each chunk is one CTA, and
//   * nodes touched by a single chunk ("interior") are summed in shared memory
//     in a fixed colour order and finalised by that CTA;
//   * nodes touched by several chunks ("shared") receive one partial sum per
//     chunk in a slot of their own; a fix-up kernel adds the slots in
//     ascending chunk order.
// Both orders are fixed, so results are bitwise reproducible run to run.
//
// Internal node numbering: interior nodes of chunk c occupy the contiguous id
// range [int_start[c], int_start[c+1]) (ordered by their incoming id); shared
// nodes follow at [N_int, N) in ascending incoming id.  With first-touch input
// numbering this is a small perturbation of that order.
#include <algorithm>
#include <cstring>

#include "sem_internal.h"

namespace sem {

bool build_chunks(const int32_t *mu, int64_t E, int Np, int64_t N, int B, ChunkMeta &m,
                  std::string &err) {
    if (E <= 0 || N <= 0 || B <= 0 || B > 1024 || Np > kMaxNp) {
        err = "build_chunks: bad arguments";
        return false;
    }
    if ((int64_t)B * Np > 65535) {
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
    for (int64_t e = 0; e < E; e++) {
        const int32_t c = (int32_t)(e / B);
        for (int p = 0; p < Np; p++) {
            const int32_t g = mu[e * Np + p];
            if (g < 0 || g >= N) {
                err = "build_chunks: node id out of range in element " + std::to_string(e);
                return false;
            }
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

    // Internal numbering.
    m.int_start.assign(nch + 1, 0);
    int64_t nsh = 0;
    for (int64_t g = 0; g < N; g++) {
        if (nref[g] == 1) m.int_start[firstc[g] + 1]++;
        else nsh++;
    }
    for (int64_t c = 0; c < nch; c++) m.int_start[c + 1] += m.int_start[c];
    m.N_int = m.int_start[nch];
    m.N_sh = nsh;
    m.int_of.assign(N, -1);
    std::vector<int32_t> sh_index(N, -1);
    {
        std::vector<int32_t> cur(m.int_start.begin(), m.int_start.end() - 1);
        int64_t s = 0;
        for (int64_t g = 0; g < N; g++) {
            if (nref[g] == 1) m.int_of[g] = cur[firstc[g]]++;
            else { sh_index[g] = (int32_t)s; m.int_of[g] = (int32_t)(m.N_int + s); s++; }
        }
    }

    // Shared slots: node s owns [sh_pstart[s], sh_pstart[s+1]), one per chunk.
    m.sh_pstart.assign(nsh + 1, 0);
    for (int64_t g = 0; g < N; g++)
        if (sh_index[g] >= 0) m.sh_pstart[sh_index[g] + 1] = nref[g];
    for (int64_t s = 0; s < nsh; s++) m.sh_pstart[s + 1] += m.sh_pstart[s];
    m.n_slots = nsh ? m.sh_pstart[nsh] : 0;

    // Per-chunk shared lists (sorted, unique) -- independent per chunk.
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
        std::sort(L.begin(), L.end());
        L.erase(std::unique(L.begin(), L.end()), L.end());
    }
    m.shl_start.assign(nch + 1, 0);
    for (int64_t c = 0; c < nch; c++) m.shl_start[c + 1] = m.shl_start[c] + (int32_t)lists[c].size();
    m.shl_node.resize(m.shl_start[nch]);
    m.shl_slot.resize(m.shl_start[nch]);
    {
        std::vector<int32_t> cursor(nsh, 0);
        for (int64_t c = 0; c < nch; c++) {  // ascending chunk order -> slot order
            int64_t k = m.shl_start[c];
            for (int32_t s : lists[c]) {
                m.shl_node[k] = s;
                m.shl_slot[k] = m.sh_pstart[s] + cursor[s]++;
                k++;
            }
        }
    }

    // Local indices and per-chunk greedy colouring (first fit in element order).
    m.lidx.assign((size_t)nch * Np * B, 0);
    m.color.assign((size_t)nch * B, 255);
    m.ncolors.assign(nch, 0);
    int max_local = 0, max_col = 0;
    bool bad_color = false;
#pragma omp parallel for schedule(dynamic, 64) reduction(max : max_local, max_col)
    for (int64_t c = 0; c < nch; c++) {
        const int64_t e0 = c * B, e1 = std::min<int64_t>(E, e0 + B);
        const int32_t i0 = m.int_start[c];
        const int32_t nint = m.int_start[c + 1] - i0;
        const std::vector<int32_t> &L = lists[c];
        const int nl = nint + (int)L.size();
        if (nl > max_local) max_local = nl;
        std::vector<uint32_t> used(nl, 0u);
        int ncol = 0;
        for (int64_t e = e0; e < e1; e++) {
            const int t = (int)(e - e0);
            uint32_t forb = 0;
            uint16_t li[kMaxNp];
            for (int p = 0; p < Np; p++) {
                const int32_t g = mu[e * Np + p];
                int loc;
                if (sh_index[g] < 0) loc = m.int_of[g] - i0;
                else loc = nint + (int)(std::lower_bound(L.begin(), L.end(), sh_index[g]) - L.begin());
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
        m.ncolors[c] = (uint8_t)ncol;
        if (ncol > max_col) max_col = ncol;
    }
    if (bad_color) {
        err = "build_chunks: more than 32 colours needed inside a chunk";
        return false;
    }
    m.max_local = max_local;
    m.max_colors = max_col;
    return true;
}

}  // namespace sem
