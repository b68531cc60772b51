// sem_internal.h -- private declarations of libsem.so (product path).
// Nothing here is shared with oracle/.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sem.h"

namespace sem {

constexpr int kMaxNp = 36;  // P = 7
#ifndef SEM_JDSW
#define SEM_JDSW 64
#endif
constexpr int kJdsW = SEM_JDSW;  // jagged diagonals per segment = max entries of a node in a chunk

#ifdef __CUDACC__
#define SEM_HD __host__ __device__
#else
#define SEM_HD
#endif

// Local node p of the lattice order (refelem.cpp: row j outer, i inner) is interior to
// the element when 1 <= i, 1 <= j, i + j <= P - 1; folded at compile time in unrolled loops.
SEM_HD constexpr int lattice_degree(int np) {
    int P = 0;
    while ((P + 1) * (P + 2) / 2 < np) P++;
    return P;
}
SEM_HD constexpr bool lattice_interior(int np, int p) {
    const int P = lattice_degree(np);
    int q = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, q++)
            if (q == p) return i >= 1 && j >= 1 && i + j <= P - 1;
    return false;
}
// Reflection r <-> s of the reference triangle on the lattice order: node (i, j) -> (j, i).
// The stiffness factors satisfy Sss = Pi Srr Pi and Srs = Pi Srs Pi under it (bit for bit at
// P4-P7, to one ulp at P2/P3, where the tables come from a different derivation).
SEM_HD constexpr int lattice_mirror(int np, int p) {
    const int P = lattice_degree(np);
    int q = 0, pi = 0, pj = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, q++)
            if (q == p) { pi = i; pj = j; }
    q = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, q++)
            if (i == pj && j == pi) return q;
    return -1;
}
// Pairs (p <= q) of K^e's upper triangle grouped with their mirror pair (sorted (pi p, pi q)):
// MirrorTable<NP>: the canonical pairs (the lexicographically smaller of the two) in order,
// p, q and the mirror pair mp, mq of each; n = their number.
constexpr int kMirMax = 128;  // canonical pairs held in constant memory (P <= 5: at most 123)
template <int NP>
struct MirrorTable {
    int n = 0;
    int p[kMirMax] = {}, q[kMirMax] = {}, mp[kMirMax] = {}, mq[kMirMax] = {};
    constexpr MirrorTable() {
        int pi[NP] = {};
        for (int k = 0; k < NP; k++) pi[k] = lattice_mirror(NP, k);
        for (int a = 0; a < NP; a++)
            for (int b = a; b < NP; b++) {
                int x = pi[a], y = pi[b];
                if (x > y) { const int z = x; x = y; y = z; }
                if ((a < x || (a == x && b <= y)) && n < kMirMax) {
                    p[n] = a; q[n] = b; mp[n] = x; mq[n] = y;
                    n++;
                }
            }
    }
};

SEM_HD constexpr int lattice_n_interior(int np) {
    const int P = lattice_degree(np);
    return P >= 3 ? (P - 1) * (P - 2) / 2 : 0;
}

// ---------------------------------------------------------------------------
// Reference triangle tables, derived on the host in long double (refelem.cpp).
// Readings R3 (node sets, lattice order) and R4 (weights) of DESIGN.md.
// ---------------------------------------------------------------------------
struct RefTables {
    int P = 0, Np = 0;
    double node[kMaxNp][2];
    double wK[kMaxNp];         // stiffness quadrature weights  = int N_p
    double wM[kMaxNp];         // mass lumping weights (HRZ for P2)
    double Dr[kMaxNp][kMaxNp]; // Dr[k][p] = dN_p/dr at node k
    double Ds[kMaxNp][kMaxNp];
    // Element stiffness factors: K^e = Grr*Srr + Gss*Sss + Grs*Srs with
    // G = c^2 detJ J^-1 J^-T (Grs = off-diagonal entry).
    double Srr[kMaxNp][kMaxNp], Sss[kMaxNp][kMaxNp], Srs[kMaxNp][kMaxNp];
    bool consistent = false;  // reading R21b (P = 4, 6): exact S, HRZ mass; no nodal quadrature
};
bool build_ref_tables(int P, RefTables &out);
bool degree_supported(int P);  // P in 2..7 (readings R21, R21b)

// Local node kinds of the lattice order (R3): kind 0 = vertex (which = local
// vertex), 1 = edge (which = local edge 0:v0v1 1:v0v2 2:v1v2, m = position from
// the edge's first listed vertex), 2 = interior (m = index).
struct LocalNode { int kind, which, m; };
const LocalNode *local_nodes(int P);

// ---------------------------------------------------------------------------
// Chunk metadata for the deterministic chunk-owned scatter (chunks.cpp).
// Elements are cut into chunks of B consecutive elements (one CTA iteration
// each).  Nodes touched by exactly one chunk are "interior": contiguous
// internal ids per chunk, window start even.  All other nodes are "shared":
// internal ids [N_int, N_int+N_sh); every (chunk, shared node) pair owns one
// slot (node-major: a shared node's slots are contiguous, in chunk order).
// ---------------------------------------------------------------------------
struct ChunkMeta {
    int B = 0, Np = 0;
    int64_t E = 0, N = 0, nchunks = 0;
    int64_t N_int = 0, N_sh = 0, N_tot = 0, n_slots = 0;
    int64_t N_if = 0;                // forced-shared (rank-interface) nodes, last N_if of the shared range
    int max_local = 0, max_win = 0, max_colors = 0, max_count = 0, max_nsh = 0;  // max_nsh: multiple of 8
    std::vector<int32_t> i0;         // [nchunks+1] interior window starts (even)
    std::vector<int32_t> s0;         // [nchunks+1] chunk blocks in shl_node / shl_slot / shl_cr (multiple of 8)
    std::vector<int32_t> shl_node;   // shared index s of each chunk-local shared node
    std::vector<int32_t> shl_slot;   // node-major slot written by that chunk
    std::vector<uint16_t> shl_cr;    // (slots of the node << 8) | this chunk's rank among them
    std::vector<int32_t> cmeta;      // [nchunks][8] {i0, nint, s0, nsh, end0, ne, nint_al, end1}
    std::vector<uint16_t> jds;       // [nchunks][2 kJdsW] start of each jagged diagonal per segment
    std::vector<uint16_t> lpos;      // [nchunks][Np*B] entry-buffer position of entry p*B + t (JDS)
    std::vector<int32_t> sh_pstart;  // [N_sh+1] slots of shared node s (node-major, chunk order)
    std::vector<int32_t> own0;       // [nchunks+1] shared indices owned (last touched) by chunk c:
                                     // [own0[c], own0[c+1]) (non-interface nodes only)
    std::vector<uint16_t> lidx;      // [nchunks][Np][B] chunk-local node index
    std::vector<uint8_t> color;      // [nchunks*B] colour within the chunk (255 = pad)
    std::vector<int32_t> int_of;     // [N] node id (numbering of mu) -> internal id
    std::vector<int32_t> bnd_chunks; // chunks touching a rank-interface node (ascending)
    std::vector<int32_t> int_chunks; // all other chunks (ascending)
};
// mu: [E][Np] node ids in [0, N) (elements in their final order).  Nodes with
// force_shared[g] != 0 (touched by another rank) are always shared; they take
// the last N_if ids of the shared range, in ascending g.
bool build_chunks(const int32_t *mu, int64_t E, int Np, int64_t N, int B, ChunkMeta &m,
                  std::string &err, const uint8_t *force_shared = nullptr);

// ---------------------------------------------------------------------------
// Multi-GPU partition (partition.cpp).  Rank r owns the global
// elements [e0, e1) = [floor(rE/G), floor((r+1)E/G)) of the reordered mesh.
// Local nodes are the global nodes its elements touch, in ascending global id.
// Interface nodes (touched by >= 2 ranks) are exchanged every step: the rank
// sends its local partial to every other rank touching the node (one buffer
// per neighbour, nodes in ascending global id) and sums all ranks' partials
// in ascending rank order, so every replica computes the same bits.
// ---------------------------------------------------------------------------
struct Partition {
    int rank = 0, world = 1;
    int64_t e0 = 0, e1 = 0;
    std::vector<int32_t> loc2glob;      // [N_loc] ascending global node id
    std::vector<int32_t> mu_local;      // [(e1-e0)][Np] local node ids
    std::vector<uint8_t> remote;        // [N_loc] touched by another rank
    std::vector<uint8_t> owned;         // [N_loc] this rank is the lowest toucher (I/O owner)
    std::vector<int32_t> if_local;      // [n_if] local id of interface node i (ascending global)
    std::vector<int32_t> nbr;           // neighbour ranks, ascending
    std::vector<int32_t> nbr_off;       // [nnbr+1] blocks of the send / recv arrays
    std::vector<int32_t> send_if;       // [n_send] interface index sent at each send position
    std::vector<int32_t> sum_start;     // [n_if+1]
    std::vector<int32_t> sum_src;       // parts index in ascending rank order: own = i (< n_if),
                                        // received = n_if + recv position
};
bool build_partition(const int32_t *mu_global, int64_t E, int Np, int64_t N, int rank, int world,
                     Partition &P, std::string &err);

}  // namespace sem
