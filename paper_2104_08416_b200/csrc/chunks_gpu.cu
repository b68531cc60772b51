// chunks_gpu.cu -- the chunk builder of chunks.cpp on the GPU (product path).
//
// Same metadata, bit for bit (tests/test_gpu_chunks.py compares every array
// with the host builder): chunks of B consecutive elements; nodes touched by
// one chunk are interior (contiguous window per chunk, descending entry count
// then ascending id), the others shared (non-interface by (owner = last
// touching chunk, id), then interface ascending id) with one node-major slot per touching chunk in
// ascending chunk order; per-chunk local indices, jagged-diagonal starts and
// entry positions.  Built from three radix sorts:
//   1. entries (chunk, node) in [chunk][p][t] order -> (chunk, node) runs,
//      entries of a run ascending in p*B + t (stable sort);
//   2. runs by (chunk, shared?, 255 - count, id or shared index) -> the local
//      order of every chunk (interior first, then shared) and its jagged
//      diagonals;
//   3. runs by (node, chunk) -> the rank of a chunk among a shared node's chunks
//      (its slot).
// Everything else is scans and scatters.  Replaces ~0.8 s of host work and
// the 0.3 GB connectivity round trip on C4.
#include <cub/cub.cuh>

#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace sem {

namespace {

constexpr int kT = 256;

inline unsigned nb(int64_t n) {
    int64_t b = (n + kT - 1) / kT;
    return (unsigned)(b < 1 ? 1 : b);
}

inline int bits_for(int64_t v) {  // smallest b with v < 2^b
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) <= v) b++;
    return b;
}

struct Tmp {
    void *p = nullptr;
    cudaStream_t s;
    explicit Tmp(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t n) { return dev_malloc(&p, n ? n : 16, s); }
    template <typename T> T *as() { return (T *)p; }
    ~Tmp() { if (p) dev_free(p, s); }
};

#define RET(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)

template <typename T>
cudaError_t excl_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    Tmp t(s);
    RET(t.alloc(bytes));
    return cub::DeviceScan::ExclusiveSum(t.p, bytes, in, out, n, s);
}

template <typename T>
cudaError_t incl_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, s));
    Tmp t(s);
    RET(t.alloc(bytes));
    return cub::DeviceScan::InclusiveSum(t.p, bytes, in, out, n, s);
}

cudaError_t sort_u64(const uint64_t *k, const int32_t *v, uint64_t *k2, int32_t *v2, int64_t n, int end_bit,
                     cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, k2, v, v2, n, 0, end_bit, s));
    Tmp t(s);
    RET(t.alloc(bytes));
    return cub::DeviceRadixSort::SortPairs(t.p, bytes, k, k2, v, v2, n, 0, end_bit, s);
}

// 1. entries in [chunk][p][t] order; padding entries get the largest key
__global__ void k_entry_keys(const int32_t *__restrict__ mu, int64_t E, int Np, int B, int64_t n_ent, int bn,
                             uint64_t pad_key, uint64_t *key, int32_t *val) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n_ent) return;
    const int64_t c = k / ((int64_t)Np * B);
    const int r = (int)(k % ((int64_t)Np * B));
    const int p = r / B, t = r % B;
    const int64_t e = c * B + t;
    key[k] = (e < E) ? (((uint64_t)c << bn) | (uint32_t)mu[e * Np + p]) : pad_key;
    val[k] = (int32_t)k;
}

__global__ void k_heads64(const uint64_t *__restrict__ key, int64_t n, int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// run r starts at sorted position start[r]; rid = inclusive scan of heads
__global__ void k_run_starts(const int32_t *__restrict__ flag, const int32_t *__restrict__ rid, int64_t n,
                             int32_t *start) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flag[i]) start[rid[i] - 1] = (int32_t)i;
}

__global__ void k_run_info(const uint64_t *__restrict__ key, const int32_t *__restrict__ start, int64_t nruns,
                           int64_t n, int bn, int32_t *rc, int32_t *rg, int32_t *rlen, int32_t *nref,
                           int32_t *lastc) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const uint64_t k = key[start[r]];
    const int32_t g = (int32_t)(k & (((uint64_t)1 << bn) - 1));
    rc[r] = (int32_t)(k >> bn);
    rg[r] = g;
    rlen[r] = (int32_t)((r + 1 < nruns ? start[r + 1] : n) - start[r]);
    atomicAdd(&nref[g], 1);
    atomicMax(&lastc[g], rc[r]);
}

__global__ void k_node_class(const int32_t *__restrict__ nref, const uint8_t *__restrict__ forced, int64_t N,
                             int32_t *a, int32_t *b, int32_t *unused) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= N) return;
    const bool f = forced && forced[g];
    a[g] = (nref[g] > 1 && !f) ? 1 : 0;
    b[g] = f ? 1 : 0;
    if (nref[g] == 0) atomicMin(unused, (int32_t)g);
}

// shared index of g: non-interface ascending id, then interface ascending id (-1 interior)
__global__ void k_shared_index(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                               const int32_t *__restrict__ ea, const int32_t *__restrict__ eb, int64_t N,
                               int32_t na, int32_t *s_of, int32_t *node_of_s) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= N) return;
    int32_t s = -1;
    if (a[g]) s = ea[g];
    else if (b[g]) s = na + eb[g];
    s_of[g] = s;
    if (s >= 0) node_of_s[s] = (int32_t)g;
}

// non-interface shared nodes (old index i < na, ascending id) keyed by (owner chunk, id)
__global__ void k_owner_keys(const int32_t *__restrict__ node_of_s, const int32_t *__restrict__ lastc, int64_t na,
                             int bn, uint64_t *key, int32_t *val) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int32_t g = node_of_s[i];
    key[i] = ((uint64_t)(uint32_t)lastc[g] << bn) | (uint32_t)g;
    val[i] = g;
}

__global__ void k_owner_index(const int32_t *__restrict__ gs, int64_t na, int32_t *s_of, int32_t *node_of_s) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int32_t g = gs[i];
    s_of[g] = (int32_t)i;
    node_of_s[i] = g;
}

// own0[c] = first owner-sorted position whose owner chunk is >= c (c = 0..nch)
__global__ void k_own0(const uint64_t *__restrict__ key, int64_t na, int bn, int64_t nch, int32_t *own0) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c > nch) return;
    int64_t lo = 0, hi = na;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)(key[mid] >> bn) < c) lo = mid + 1;
        else hi = mid;
    }
    own0[c] = (int32_t)lo;
}

// 2. local-order key of every run; per-chunk interior / shared counts
// Local order key: (chunk, shared?, 255 - entry count, id).  Element-interior nodes (the
// run's entry sits at a lattice-interior p, inner_mask bit p) take the bucket after the
// count-1 nodes, so they close the interior segment (K7 finalises them per element).
__global__ void k_local_keys(const int32_t *__restrict__ rc, const int32_t *__restrict__ rg,
                             const int32_t *__restrict__ rlen, const int32_t *__restrict__ s_of,
                             const int32_t *__restrict__ v1s, const int32_t *__restrict__ rstart, int Np, int B,
                             uint64_t inner_mask, int64_t nruns, int bx, uint64_t *key, int32_t *val, int32_t *nint,
                             int32_t *nsh) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int32_t c = rc[r], g = rg[r], s = s_of[g];
    const bool sh = s >= 0;
    const int p = (int)((v1s[rstart[r]] % ((int64_t)Np * B)) / B);
    const uint32_t bucket = (!sh && ((inner_mask >> p) & 1)) ? 255u : 255u - (uint32_t)min(rlen[r], 255);
    const uint64_t x = sh ? (uint32_t)s : (uint32_t)g;
    key[r] = ((uint64_t)c << (9 + bx)) | ((uint64_t)(sh ? 1 : 0) << (8 + bx)) | ((uint64_t)bucket << bx) | x;
    val[r] = (int32_t)r;
    // runs come in (chunk, node) order: lanes of a warp mostly share (c, sh), so
    // aggregate the count per warp before the atomic
    const int tag = 2 * c + (sh ? 1 : 0);
    const unsigned peers = __match_any_sync(__activemask(), tag);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(sh ? &nsh[c] : &nint[c], __popc(peers));
}

__global__ void k_chunk_sizes(const int32_t *__restrict__ nint, const int32_t *__restrict__ nsh, int64_t nch,
                              int32_t *tot, int32_t *ni_al, int32_t *nsh8) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int32_t ni = nint[c], ns = nsh[c];
    const int32_t al = (ni + 1) & ~1;
    tot[c] = ni + ns;
    ni_al[c] = al;
    nsh8[c] = (ns + 7) & ~7;
}

// local index of every run; int_of of every node
__global__ void k_local_index(const int32_t *__restrict__ order, const int32_t *__restrict__ rc,
                              const int32_t *__restrict__ rg, const int32_t *__restrict__ s_of,
                              const int32_t *__restrict__ cs, const int32_t *__restrict__ nint,
                              const int32_t *__restrict__ ni_al, const int32_t *__restrict__ i0, int64_t nruns,
                              int64_t N_int, int32_t *local, int32_t *int_of) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nruns) return;
    const int32_t r = order[j], c = rc[r], g = rg[r];
    const int32_t pos = (int32_t)(j - cs[c]);
    const int32_t s = s_of[g];
    if (s < 0) {
        local[r] = pos;
        int_of[g] = i0[c] + pos;
    } else {
        local[r] = ni_al[c] + (pos - nint[c]);
        int_of[g] = (int32_t)(N_int + s);
    }
}

// 3. rank of the chunk among the chunks of its node
__global__ void k_node_chunk_keys(const int32_t *__restrict__ rc, const int32_t *__restrict__ rg, int64_t nruns,
                                  int bc, uint64_t *key, int32_t *val) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    key[r] = ((uint64_t)(uint32_t)rg[r] << bc) | (uint32_t)rc[r];
    val[r] = (int32_t)r;
}

__global__ void k_count_of_s(const int32_t *__restrict__ node_of_s, const int32_t *__restrict__ nref, int64_t nsh,
                             int32_t *cnt) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s < nsh) cnt[s] = nref[node_of_s[s]];
}

__global__ void k_slots(const uint64_t *__restrict__ key3, const int32_t *__restrict__ order3, int64_t nruns, int bc,
                        const int32_t *__restrict__ s_of, const int32_t *__restrict__ nref,
                        const int32_t *__restrict__ pstart, const int32_t *__restrict__ rc,
                        const int32_t *__restrict__ local, const int32_t *__restrict__ ni_al,
                        const int32_t *__restrict__ s0, int32_t *shl_node, int32_t *shl_slot, uint16_t *shl_cr) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nruns) return;
    const int32_t g = (int32_t)(key3[j] >> bc);
    const int32_t s = s_of[g];
    if (s < 0) return;
    const int32_t n = nref[g];
    // the node's runs are consecutive in key3 order: rank = j - first position
    int32_t rank = 0;
    while (rank < n && j - rank - 1 >= 0 && (int32_t)(key3[j - rank - 1] >> bc) == g) rank++;
    const int32_t r = order3[j], c = rc[r];
    const int64_t k = (int64_t)s0[c] + (local[r] - ni_al[c]);
    shl_node[k] = s;
    shl_slot[k] = pstart[s] + rank;
    shl_cr[k] = (uint16_t)((n << 8) | rank);
}

// Jagged diagonals (chunks.cpp): nodes of a segment with more than d entries
// per diagonal d (order-free integer counts), then the diagonal starts.
__global__ void k_jds_counts(const int32_t *__restrict__ rc, const int32_t *__restrict__ rlen,
                             const int32_t *__restrict__ local, const int32_t *__restrict__ nint, int64_t nruns,
                             int32_t *nd, int32_t *mx) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int32_t c = rc[r], len = rlen[r];
    const int sg = local[r] < nint[c] ? 0 : 1;
    atomicMax(&mx[2], len);  // max_count
    for (int d = 0; d < len && d < kJdsW; d++) atomicAdd(&nd[((int64_t)c * 2 + sg) * kJdsW + d], 1);
}

__global__ void k_jds_starts(const int32_t *__restrict__ nd, int64_t nch, uint16_t *jds, int32_t *end0,
                             int32_t *end1) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    int base = 0;
    for (int sg = 0; sg < 2; sg++) {
        for (int d = 0; d < kJdsW; d++) {
            jds[(c * 2 + sg) * kJdsW + d] = (uint16_t)base;
            base += nd[(c * 2 + sg) * kJdsW + d];
        }
        (sg == 0 ? end0 : end1)[c] = base;
    }
}

__global__ void k_entry_local(const int32_t *__restrict__ flag_rid, const int32_t *__restrict__ v1,
                              const int32_t *__restrict__ rstart, const int32_t *__restrict__ rc,
                              const int32_t *__restrict__ local, const int32_t *__restrict__ nint,
                              const int32_t *__restrict__ ni_al, const uint16_t *__restrict__ jds, int64_t n,
                              uint16_t *lidx, uint16_t *lpos) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t r = flag_rid[i] - 1, k = v1[i];
    const int32_t l = local[r], c = rc[r], rank = (int32_t)(i - rstart[r]);
    lidx[k] = (uint16_t)l;
    if (rank >= kJdsW) return;  // reported through max_count
    const int sg = l < nint[c] ? 0 : 1;
    lpos[k] = (uint16_t)(jds[((int64_t)c * 2 + sg) * kJdsW + rank] + (sg == 0 ? l : l - ni_al[c]));
}

__global__ void k_cmeta(const int32_t *__restrict__ i0, const int32_t *__restrict__ nint,
                        const int32_t *__restrict__ s0, const int32_t *__restrict__ nsh,
                        const int32_t *__restrict__ ni_al, const int32_t *__restrict__ end0,
                        const int32_t *__restrict__ end1, int64_t nch, int64_t E, int B, int32_t *cmeta, int32_t *mx) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    int32_t *cm = cmeta + 8 * c;
    const int64_t e1 = min(E, (c + 1) * (int64_t)B);
    cm[0] = i0[c];
    cm[1] = nint[c];
    cm[2] = s0[c];
    cm[3] = nsh[c];
    cm[4] = end0[c];
    cm[5] = (int32_t)(e1 - c * B);
    cm[6] = ni_al[c];
    cm[7] = end1[c];
    const int32_t ns = nsh[c];
    atomicMax(&mx[0], ni_al[c] + ((ns + 1) & ~1));    // max_local
    atomicMax(&mx[1], ni_al[c]);                      // max_win
    atomicMax(&mx[3], (ns + 7) & ~7);                 // max_nsh
}

__global__ void k_bnd_flag(const int32_t *__restrict__ rc, const int32_t *__restrict__ rg,
                           const uint8_t *__restrict__ forced, int64_t nruns, int32_t *bnd) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < nruns && forced && forced[rg[r]]) bnd[rc[r]] = 1;
}

__global__ void k_iota32(int32_t *a, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

struct SubTrace {  // SEM_TRACE=1: wall time of each builder section on stderr
    bool on = getenv("SEM_TRACE") != nullptr;
    double t = ms();
    static double ms() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    void mark(cudaStream_t s, const char *what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const double n = ms();
        fprintf(stderr, "[sem chunk builder]   %-28s %8.1f ms\n", what, n - t);
        t = n;
    }
};

}  // namespace

cudaError_t build_chunks_gpu(const int32_t *d_mu, int64_t E, int Np, int64_t N, int B, const uint8_t *d_forced,
                             const DeviceAlloc &dalloc, ChunkMeta &m, DevChunks &d, int32_t **d_int_of,
                             int32_t **d_bnd, int32_t **d_intc, std::string &err, cudaStream_t s) {
    m = ChunkMeta();
    m.B = B;
    m.Np = Np;
    m.E = E;
    m.N = N;
    const int64_t nch = (E + B - 1) / B;
    m.nchunks = nch;
    const int64_t n_ent = nch * Np * B, n = E * Np;
    const int bn = bits_for(N), bc = bits_for(nch + 1);
    if (bc + bn > 62 || bc + 9 + bn > 64) { err = "build_chunks_gpu: mesh too large for 64-bit keys"; return cudaSuccess; }
    const uint64_t pad_key = ((uint64_t)1 << (bc + bn)) - 1;
    SubTrace tr;

    // ---- 1. entries -> (chunk, node) runs ----
    Tmp k1(s), v1(s), k1s(s), v1s(s), flag(s), rid(s);
    RET(k1.alloc(8 * n_ent));
    RET(v1.alloc(4 * n_ent));
    RET(k1s.alloc(8 * n_ent));
    RET(v1s.alloc(4 * n_ent));
    k_entry_keys<<<nb(n_ent), kT, 0, s>>>(d_mu, E, Np, B, n_ent, bn, pad_key, k1.as<uint64_t>(), v1.as<int32_t>());
    RET(sort_u64(k1.as<uint64_t>(), v1.as<int32_t>(), k1s.as<uint64_t>(), v1s.as<int32_t>(), n_ent, bc + bn, s));
    RET(flag.alloc(4 * n));
    RET(rid.alloc(4 * n));
    k_heads64<<<nb(n), kT, 0, s>>>(k1s.as<uint64_t>(), n, flag.as<int32_t>());
    RET(incl_scan(flag.as<int32_t>(), rid.as<int32_t>(), n, s));
    int32_t nr32 = 0;
    RET(cudaMemcpyAsync(&nr32, rid.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    const int64_t nruns = nr32;
    Tmp rstart(s), rc(s), rg(s), rlen(s), nref(s), lastc(s);
    RET(rstart.alloc(4 * nruns));
    RET(rc.alloc(4 * nruns));
    RET(rg.alloc(4 * nruns));
    RET(rlen.alloc(4 * nruns));
    RET(nref.alloc(4 * N));
    RET(lastc.alloc(4 * N));
    RET(cudaMemsetAsync(nref.p, 0, 4 * N, s));
    RET(cudaMemsetAsync(lastc.p, 0xff, 4 * N, s));
    k_run_starts<<<nb(n), kT, 0, s>>>(flag.as<int32_t>(), rid.as<int32_t>(), n, rstart.as<int32_t>());
    k_run_info<<<nb(nruns), kT, 0, s>>>(k1s.as<uint64_t>(), rstart.as<int32_t>(), nruns, n, bn, rc.as<int32_t>(),
                                        rg.as<int32_t>(), rlen.as<int32_t>(), nref.as<int32_t>(),
                                        lastc.as<int32_t>());

    tr.mark(s, "runs");
    // ---- classification and shared indices ----
    Tmp fa(s), fb(s), ea(s), eb(s), s_of(s), bad(s);
    RET(fa.alloc(4 * (N + 1)));
    RET(fb.alloc(4 * (N + 1)));
    RET(ea.alloc(4 * (N + 1)));
    RET(eb.alloc(4 * (N + 1)));
    RET(s_of.alloc(4 * N));
    RET(bad.alloc(4));
    int32_t big = INT_MAX;
    RET(cudaMemcpyAsync(bad.p, &big, 4, cudaMemcpyHostToDevice, s));
    RET(cudaMemsetAsync(fa.as<int32_t>() + N, 0, 4, s));
    RET(cudaMemsetAsync(fb.as<int32_t>() + N, 0, 4, s));
    k_node_class<<<nb(N), kT, 0, s>>>(nref.as<int32_t>(), d_forced, N, fa.as<int32_t>(), fb.as<int32_t>(),
                                      bad.as<int32_t>());
    RET(excl_scan(fa.as<int32_t>(), ea.as<int32_t>(), N + 1, s));
    RET(excl_scan(fb.as<int32_t>(), eb.as<int32_t>(), N + 1, s));
    int32_t hb[3];
    RET(cudaMemcpyAsync(&hb[0], ea.as<int32_t>() + N, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaMemcpyAsync(&hb[1], eb.as<int32_t>() + N, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaMemcpyAsync(&hb[2], bad.p, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    if (hb[2] != INT_MAX) {
        err = "node " + std::to_string(hb[2]) + " is not used by any element";
        return cudaSuccess;
    }
    const int64_t na = hb[0], nif = hb[1], nsh_tot = na + nif;
    m.N_sh = nsh_tot;
    m.N_if = nif;
    Tmp node_of_s(s);
    RET(node_of_s.alloc(4 * (nsh_tot + 1)));
    k_shared_index<<<nb(N), kT, 0, s>>>(fa.as<int32_t>(), fb.as<int32_t>(), ea.as<int32_t>(), eb.as<int32_t>(), N,
                                        (int32_t)na, s_of.as<int32_t>(), node_of_s.as<int32_t>());
    // non-interface shared nodes renumbered by (owner chunk, id): a chunk's owned nodes are the
    // contiguous range [own0[c], own0[c+1])
    int32_t *own0 = nullptr;
    RET(dalloc((void **)&own0, 4 * (size_t)(nch + 1)));
    {
        Tmp ok(s), ov(s), oks(s), ovs(s);
        RET(ok.alloc(8 * (na + 1)));
        RET(ov.alloc(4 * (na + 1)));
        RET(oks.alloc(8 * (na + 1)));
        RET(ovs.alloc(4 * (na + 1)));
        if (na > 0) {
            k_owner_keys<<<nb(na), kT, 0, s>>>(node_of_s.as<int32_t>(), lastc.as<int32_t>(), na, bn,
                                               ok.as<uint64_t>(), ov.as<int32_t>());
            RET(sort_u64(ok.as<uint64_t>(), ov.as<int32_t>(), oks.as<uint64_t>(), ovs.as<int32_t>(), na, bc + bn, s));
            k_owner_index<<<nb(na), kT, 0, s>>>(ovs.as<int32_t>(), na, s_of.as<int32_t>(), node_of_s.as<int32_t>());
        }
        k_own0<<<nb(nch + 1), kT, 0, s>>>(oks.as<uint64_t>(), na, bn, nch, own0);
        RET(cudaStreamSynchronize(s));
    }

    tr.mark(s, "classification");
    // ---- 2. local order per chunk ----
    Tmp k2(s), v2(s), k2s(s), order(s), nint(s), nsh(s);
    RET(k2.alloc(8 * nruns));
    RET(v2.alloc(4 * nruns));
    RET(k2s.alloc(8 * nruns));
    RET(order.alloc(4 * nruns));
    RET(nint.alloc(4 * (nch + 1)));
    RET(nsh.alloc(4 * (nch + 1)));
    RET(cudaMemsetAsync(nint.p, 0, 4 * (nch + 1), s));
    RET(cudaMemsetAsync(nsh.p, 0, 4 * (nch + 1), s));
    uint64_t inner_mask = 0;
    for (int p = 0; p < Np; p++)
        if (lattice_interior(Np, p)) inner_mask |= (uint64_t)1 << p;
    k_local_keys<<<nb(nruns), kT, 0, s>>>(rc.as<int32_t>(), rg.as<int32_t>(), rlen.as<int32_t>(), s_of.as<int32_t>(),
                                          v1s.as<int32_t>(), rstart.as<int32_t>(), Np, B, inner_mask, nruns, bn,
                                          k2.as<uint64_t>(), v2.as<int32_t>(), nint.as<int32_t>(), nsh.as<int32_t>());
    RET(sort_u64(k2.as<uint64_t>(), v2.as<int32_t>(), k2s.as<uint64_t>(), order.as<int32_t>(), nruns, bc + 9 + bn, s));
    Tmp tot(s), ni_al(s), nsh8(s), cs(s), i0(s), s0(s);
    for (Tmp *t : {&tot, &ni_al, &nsh8, &cs, &i0, &s0}) RET(t->alloc(4 * (nch + 1)));
    for (Tmp *t : {&tot, &ni_al, &nsh8}) RET(cudaMemsetAsync(t->p, 0, 4 * (nch + 1), s));
    k_chunk_sizes<<<nb(nch), kT, 0, s>>>(nint.as<int32_t>(), nsh.as<int32_t>(), nch, tot.as<int32_t>(),
                                         ni_al.as<int32_t>(), nsh8.as<int32_t>());
    RET(excl_scan(tot.as<int32_t>(), cs.as<int32_t>(), nch + 1, s));
    RET(excl_scan(ni_al.as<int32_t>(), i0.as<int32_t>(), nch + 1, s));
    RET(excl_scan(nsh8.as<int32_t>(), s0.as<int32_t>(), nch + 1, s));
    int32_t hN_int = 0, hs0 = 0;
    RET(cudaMemcpyAsync(&hN_int, i0.as<int32_t>() + nch, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaMemcpyAsync(&hs0, s0.as<int32_t>() + nch, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    m.N_int = hN_int;
    m.N_tot = m.N_int + m.N_sh;
    tr.mark(s, "local order sort");
    Tmp local(s);
    RET(local.alloc(4 * nruns));
    int32_t *int_of = nullptr;
    RET(dalloc((void **)&int_of, 4 * (size_t)N));
    *d_int_of = int_of;
    k_local_index<<<nb(nruns), kT, 0, s>>>(order.as<int32_t>(), rc.as<int32_t>(), rg.as<int32_t>(),
                                           s_of.as<int32_t>(), cs.as<int32_t>(), nint.as<int32_t>(),
                                           ni_al.as<int32_t>(), i0.as<int32_t>(), nruns, m.N_int, local.as<int32_t>(),
                                           int_of);

    tr.mark(s, "local index");
    // ---- 3. slots: node-major, chunks of a node in ascending order ----
    int32_t *sh_pstart = nullptr, *shl_node = nullptr, *shl_slot = nullptr;
    uint16_t *shl_cr = nullptr;
    RET(dalloc((void **)&sh_pstart, 4 * (size_t)(nsh_tot + 1)));
    RET(dalloc((void **)&shl_node, 4 * (size_t)(hs0 + 8)));
    RET(dalloc((void **)&shl_slot, 4 * (size_t)(hs0 + 8)));
    RET(dalloc((void **)&shl_cr, 2 * (size_t)(hs0 + 8)));
    RET(cudaMemsetAsync(shl_node, 0, 4 * (size_t)(hs0 + 8), s));
    RET(cudaMemsetAsync(shl_slot, 0, 4 * (size_t)(hs0 + 8), s));
    RET(cudaMemsetAsync(shl_cr, 0, 2 * (size_t)(hs0 + 8), s));
    {
        Tmp cnt(s);
        RET(cnt.alloc(4 * (nsh_tot + 1)));
        RET(cudaMemsetAsync(cnt.p, 0, 4 * (nsh_tot + 1), s));
        k_count_of_s<<<nb(nsh_tot), kT, 0, s>>>(node_of_s.as<int32_t>(), nref.as<int32_t>(), nsh_tot,
                                                cnt.as<int32_t>());
        RET(excl_scan(cnt.as<int32_t>(), sh_pstart, nsh_tot + 1, s));
        int32_t hslots = 0;
        RET(cudaMemcpyAsync(&hslots, sh_pstart + nsh_tot, 4, cudaMemcpyDeviceToHost, s));
        Tmp k3(s), v3(s), k3s(s), o3(s);
        RET(k3.alloc(8 * nruns));
        RET(v3.alloc(4 * nruns));
        RET(k3s.alloc(8 * nruns));
        RET(o3.alloc(4 * nruns));
        k_node_chunk_keys<<<nb(nruns), kT, 0, s>>>(rc.as<int32_t>(), rg.as<int32_t>(), nruns, bc, k3.as<uint64_t>(),
                                                   v3.as<int32_t>());
        RET(sort_u64(k3.as<uint64_t>(), v3.as<int32_t>(), k3s.as<uint64_t>(), o3.as<int32_t>(), nruns, bc + bn, s));
        k_slots<<<nb(nruns), kT, 0, s>>>(k3s.as<uint64_t>(), o3.as<int32_t>(), nruns, bc, s_of.as<int32_t>(),
                                         nref.as<int32_t>(), sh_pstart, rc.as<int32_t>(), local.as<int32_t>(),
                                         ni_al.as<int32_t>(), s0.as<int32_t>(), shl_node, shl_slot, shl_cr);
        RET(cudaStreamSynchronize(s));
        m.n_slots = nsh_tot ? hslots : 0;
    }

    tr.mark(s, "slots");
    // ---- local indices, CSR row pointers and positions ----
    uint16_t *lidx = nullptr, *lpos = nullptr, *jds = nullptr;
    int32_t *cmeta = nullptr;
    RET(dalloc((void **)&lidx, 2 * (size_t)n_ent));
    RET(dalloc((void **)&lpos, 2 * (size_t)n_ent));
    RET(dalloc((void **)&jds, 2 * (size_t)(nch * 2 * kJdsW)));
    RET(dalloc((void **)&cmeta, 4 * 8 * (size_t)nch));
    RET(cudaMemsetAsync(lidx, 0, 2 * (size_t)n_ent, s));
    RET(cudaMemsetAsync(lpos, 0, 2 * (size_t)n_ent, s));
    Tmp mx(s), nd(s), end0(s), end1(s);
    RET(mx.alloc(16));
    RET(cudaMemsetAsync(mx.p, 0, 16, s));
    RET(nd.alloc(4 * (size_t)(nch * 2 * kJdsW)));
    RET(end0.alloc(4 * (nch + 1)));
    RET(end1.alloc(4 * (nch + 1)));
    RET(cudaMemsetAsync(nd.p, 0, 4 * (size_t)(nch * 2 * kJdsW), s));
    k_jds_counts<<<nb(nruns), kT, 0, s>>>(rc.as<int32_t>(), rlen.as<int32_t>(), local.as<int32_t>(), nint.as<int32_t>(),
                                          nruns, nd.as<int32_t>(), mx.as<int32_t>());
    k_jds_starts<<<nb(nch), kT, 0, s>>>(nd.as<int32_t>(), nch, jds, end0.as<int32_t>(), end1.as<int32_t>());
    k_entry_local<<<nb(n), kT, 0, s>>>(rid.as<int32_t>(), v1s.as<int32_t>(), rstart.as<int32_t>(), rc.as<int32_t>(),
                                       local.as<int32_t>(), nint.as<int32_t>(), ni_al.as<int32_t>(), jds, n, lidx,
                                       lpos);
    k_cmeta<<<nb(nch), kT, 0, s>>>(i0.as<int32_t>(), nint.as<int32_t>(), s0.as<int32_t>(), nsh.as<int32_t>(),
                                   ni_al.as<int32_t>(), end0.as<int32_t>(), end1.as<int32_t>(), nch, E, B, cmeta,
                                   mx.as<int32_t>());
    int32_t hmx[4];
    RET(cudaMemcpyAsync(hmx, mx.p, 16, cudaMemcpyDeviceToHost, s));

    tr.mark(s, "jds + entries");
    // ---- boundary (touching a rank-interface node) / interior chunk lists ----
    int32_t *bnd = nullptr, *intc = nullptr;
    std::vector<int32_t> hbnd;
    if (d_forced && nif > 0) {
        Tmp bf(s);
        RET(bf.alloc(4 * nch));
        RET(cudaMemsetAsync(bf.p, 0, 4 * nch, s));
        k_bnd_flag<<<nb(nruns), kT, 0, s>>>(rc.as<int32_t>(), rg.as<int32_t>(), d_forced, nruns, bf.as<int32_t>());
        hbnd.resize(nch);
        RET(cudaMemcpyAsync(hbnd.data(), bf.p, 4 * nch, cudaMemcpyDeviceToHost, s));
    }
    RET(cudaStreamSynchronize(s));
    m.max_local = hmx[0];
    m.max_win = hmx[1];
    m.max_count = hmx[2];
    if (m.max_count > kJdsW) {
        err = "build_chunks: a node has more than 64 entries in one chunk";
        return cudaSuccess;
    }
    m.max_nsh = hmx[3];
    m.max_colors = 0;
    for (int64_t c = 0; c < nch; c++)
        ((!hbnd.empty() && hbnd[c]) ? m.bnd_chunks : m.int_chunks).push_back((int32_t)c);
    RET(dalloc((void **)&bnd, 4 * (m.bnd_chunks.size() + 1)));
    RET(dalloc((void **)&intc, 4 * (m.int_chunks.size() + 1)));
    if (!m.bnd_chunks.empty())
        RET(cudaMemcpyAsync(bnd, m.bnd_chunks.data(), 4 * m.bnd_chunks.size(), cudaMemcpyHostToDevice, s));
    if (!m.int_chunks.empty())
        RET(cudaMemcpyAsync(intc, m.int_chunks.data(), 4 * m.int_chunks.size(), cudaMemcpyHostToDevice, s));
    *d_bnd = bnd;
    *d_intc = intc;

    tr.mark(s, "lists");
    d.B = B; d.Np = Np; d.E = E; d.N = N; d.nchunks = nch;
    d.N_int = m.N_int; d.N_sh = m.N_sh; d.N_tot = m.N_tot; d.n_slots = m.n_slots; d.N_if = m.N_if;
    d.max_local = m.max_local; d.max_win = m.max_win; d.max_count = m.max_count; d.max_nsh = m.max_nsh;
    d.cmeta = cmeta; d.lidx = lidx; d.lpos = lpos; d.jds = jds; d.sh_pstart = sh_pstart;
    d.shl_node = shl_node; d.shl_slot = shl_slot; d.shl_cr = shl_cr; d.own0 = own0;
    RET(cudaStreamSynchronize(s));
    return cudaGetLastError();
}

}  // namespace sem
