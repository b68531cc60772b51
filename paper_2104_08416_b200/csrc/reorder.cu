// reorder.cu -- sm_100a kernels for mesh preparation (product path):
// bounding box, orientation, K1 generalized-Hilbert keys, K2 radix sort,
// K4 canonical SEM nodes, K3 row permutation, K5 first-touch renumbering.
//
// Bit-exactness with the oracle rests on (a) integer-only work for nodes and
// labels, and (b) IEEE fp64 with explicit round-to-nearest intrinsics (no FMA
// contraction) wherever floating point decides an integer (centroid cell,
// orientation sign).  Reading R9 fixes the operation order.
#include <cub/cub.cuh>

#include <climits>

#include "kernels.h"

namespace sem {

namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 2147483647LL) b = 2147483647LL;
    return (unsigned)b;
}

__device__ __forceinline__ int isgn(int v) { return (v > 0) - (v < 0); }
__device__ __forceinline__ int half_floor(int v) { return (v >= 0) ? v / 2 : -((-v + 1) / 2); }

// Position of cell (px, py) on the generalized Hilbert curve over W x H
// (docs/hilbert.md), by descending the recursion instead of walking the path:
// at each level find the sub-rectangle holding the cell and add the sizes of
// the sub-rectangles walked before it.
__device__ uint32_t gilbert_d(int px, int py, int W, int H) {
    int ox = 0, oy = 0, ax, ay, bx, by;
    if (W >= H) { ax = W; ay = 0; bx = 0; by = H; }
    else { ax = 0; ay = H; bx = W; by = 0; }
    uint32_t d = 0;
    for (;;) {
        const int w = abs(ax + ay), h = abs(bx + by);
        const int dax = isgn(ax), day = isgn(ay), dbx = isgn(bx), dby = isgn(by);
        const int u = (px - ox) * dax + (py - oy) * day;  // offset along a
        const int v = (px - ox) * dbx + (py - oy) * dby;  // offset along b
        if (h == 1) return d + (uint32_t)u;  // rule 1
        if (w == 1) return d + (uint32_t)v;  // rule 2
        int ax2 = half_floor(ax), ay2 = half_floor(ay);
        int bx2 = half_floor(bx), by2 = half_floor(by);
        const int w2 = abs(ax2 + ay2), h2 = abs(bx2 + by2);
        if (2 * w > 3 * h) {  // rule 3a
            if ((w2 & 1) && w > 2) { ax2 += dax; ay2 += day; }
            const int wa2 = abs(ax2 + ay2);
            if (u < wa2) { ax = ax2; ay = ay2; continue; }
            d += (uint32_t)(wa2 * h);
            ox += ax2; oy += ay2; ax -= ax2; ay -= ay2;
        } else {  // rule 3b
            if ((h2 & 1) && h > 2) { bx2 += dbx; by2 += dby; }
            const int wa2 = abs(ax2 + ay2), hb2 = abs(bx2 + by2);
            if (v < hb2 && u < wa2) {  // first: R(o, b2, a2)
                const int nax = bx2, nay = by2;
                bx = ax2; by = ay2; ax = nax; ay = nay;
                continue;
            }
            d += (uint32_t)(hb2 * wa2);
            if (v >= hb2) {  // second: R(o + b2, a, b - b2)
                ox += bx2; oy += by2; bx -= bx2; by -= by2;
                continue;
            }
            d += (uint32_t)(w * (h - hb2));
            // third: R(o + (a - sgn a) + (b2 - sgn b), -b2, -(a - a2))
            const int nox = ox + (ax - dax) + (bx2 - dbx), noy = oy + (ay - day) + (by2 - dby);
            const int nbx = -(ax - ax2), nby = -(ay - ay2);
            ox = nox; oy = noy; ax = -bx2; ay = -by2; bx = nbx; by = nby;
        }
    }
}

__global__ void k_bbox_partial(const double *__restrict__ vxy, int64_t nv, double *part) {
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = reinterpret_cast<const double2 *>(vxy)[i];
        mnx = fmin(mnx, p.x); mxx = fmax(mxx, p.x);
        mny = fmin(mny, p.y); mxy = fmax(mxy, p.y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    __shared__ double sm[4][32];
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) { sm[0][w] = mnx; sm[1][w] = mny; sm[2][w] = mxx; sm[3][w] = mxy; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x / 32); k++) {
            mnx = fmin(mnx, sm[0][k]); mny = fmin(mny, sm[1][k]);
            mxx = fmax(mxx, sm[2][k]); mxy = fmax(mxy, sm[3][k]);
        }
        part[4 * blockIdx.x + 0] = mnx;
        part[4 * blockIdx.x + 1] = mny;
        part[4 * blockIdx.x + 2] = mxx;
        part[4 * blockIdx.x + 3] = mxy;
    }
}

__global__ void k_bbox_final(const double *part, int nb, double *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double r[4] = {INFINITY, INFINITY, -INFINITY, -INFINITY};
    for (int b = 0; b < nb; b++) {
        r[0] = fmin(r[0], part[4 * b]); r[1] = fmin(r[1], part[4 * b + 1]);
        r[2] = fmax(r[2], part[4 * b + 2]); r[3] = fmax(r[3], part[4 * b + 3]);
    }
    for (int k = 0; k < 4; k++) out[k] = r[k];
}

__global__ void k_orient(const double *__restrict__ vxy, const int32_t *__restrict__ tri, int64_t E, int64_t nv,
                         int32_t *__restrict__ tri_or, int32_t *bad) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
    if (v0 < 0 || v0 >= nv || v1 < 0 || v1 >= nv || v2 < 0 || v2 >= nv) {  // before any vertex access
        atomicMin(bad + 1, (int32_t)e);
        return;
    }
    const double x0 = vxy[2 * v0], y0 = vxy[2 * v0 + 1];
    const double x1 = vxy[2 * v1], y1 = vxy[2 * v1 + 1];
    const double x2 = vxy[2 * v2], y2 = vxy[2 * v2 + 1];
    const double det = __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(y2, y0)),
                                 __dmul_rn(__dsub_rn(x2, x0), __dsub_rn(y1, y0)));
    if (det == 0.0) atomicMin(bad, (int32_t)e);
    tri_or[3 * e] = v0;
    if (det < 0.0) { tri_or[3 * e + 1] = v2; tri_or[3 * e + 2] = v1; }
    else { tri_or[3 * e + 1] = v1; tri_or[3 * e + 2] = v2; }
}

// K1: centroid from the INPUT vertex order, sub-rectangle
// (i, j) of the w_b x h_b box, then its position on the curve.
__global__ void k_hilbert_keys(const double *__restrict__ vxy, const int32_t *__restrict__ tri,
                               int64_t E, double xm0, double xm1, double ws, double hs, int wb,
                               int hb, uint32_t *__restrict__ keys) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
    const double xc0 = __ddiv_rn(__dadd_rn(__dadd_rn(vxy[2 * v0], vxy[2 * v1]), vxy[2 * v2]), 3.0);
    const double xc1 =
        __ddiv_rn(__dadd_rn(__dadd_rn(vxy[2 * v0 + 1], vxy[2 * v1 + 1]), vxy[2 * v2 + 1]), 3.0);
    long long i = (long long)floor(__dmul_rn(__dsub_rn(xc0, xm0), ws));
    long long j = (long long)floor(__dmul_rn(__dsub_rn(xc1, xm1), hs));
    if (i > wb - 1) i = wb - 1;
    if (j > hb - 1) j = hb - 1;
    if (i < 0) i = 0;
    if (j < 0) j = 0;
    keys[e] = gilbert_d((int)i, (int)j, wb, hb);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void k_random_keys(int64_t E, uint64_t seed, uint64_t *keys) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < E) keys[e] = splitmix64(seed ^ (uint64_t)e);
}

__global__ void k_iota(int32_t *a, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

__global__ void k_fill_i32(int32_t *a, int64_t n, int32_t v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

// ---- K4 canonical nodes -----------------------------------------------------
__constant__ int c_edge_v[3][2] = {{0, 1}, {0, 2}, {1, 2}};
__constant__ int c_ln[kMaxNp][3];  // local node table of the current degree (R3)

__global__ void k_edge_keys(const int32_t *__restrict__ tri, int64_t E, uint64_t *keys,
                            int32_t *vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= 3 * E) return;
    const int64_t e = i / 3;
    const int l = (int)(i % 3);
    const int32_t a = tri[3 * e + c_edge_v[l][0]], b = tri[3 * e + c_edge_v[l][1]];
    const uint32_t lo = (uint32_t)min(a, b), hi = (uint32_t)max(a, b);
    keys[i] = ((uint64_t)lo << 32) | hi;
    vals[i] = (int32_t)i;
}

__global__ void k_heads(const uint64_t *__restrict__ keys, int64_t n, int32_t *flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_edge_scatter(const int32_t *__restrict__ vals, const int32_t *__restrict__ incl,
                               int64_t n, int32_t *eid) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) eid[vals[i]] = incl[i] - 1;
}

__global__ void k_mu_canonical(const int32_t *__restrict__ tri, const int32_t *__restrict__ eid,
                               int64_t E, int P, int Np, int64_t nv, int64_t nedges,
                               int32_t *__restrict__ mu) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int nI = (P - 1) * (P - 2) / 2;
    for (int p = 0; p < Np; p++) {
        const int kind = c_ln[p][0], which = c_ln[p][1], m = c_ln[p][2];
        int64_t g;
        if (kind == 0) {
            g = tri[3 * e + which];
        } else if (kind == 1) {
            const int32_t a = tri[3 * e + c_edge_v[which][0]], b = tri[3 * e + c_edge_v[which][1]];
            const int i = (a < b) ? m : (P - 2) - m;  // counted from the min-id end
            g = nv + (int64_t)eid[3 * e + which] * (P - 1) + i;
        } else {
            g = nv + nedges * (P - 1) + e * nI + m;
        }
        mu[e * Np + p] = (int32_t)g;
    }
}

__global__ void k_mark_used(const int32_t *__restrict__ tri, int64_t E, int32_t *used) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < 3 * E) used[tri[i]] = 1;
}

__global__ void k_first_unused(const int32_t *used, int64_t nv, int32_t *first) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nv && !used[i]) atomicMin(first, (int32_t)i);
}

__global__ void k_permute_rows(const int32_t *__restrict__ src, const int32_t *__restrict__ perm,
                               int64_t E, int w, int32_t *__restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= E * w) return;
    const int64_t k = i / w;
    const int c = (int)(i % w);
    dst[i] = src[(int64_t)perm[k] * w + c];
}

// ---- K5 first touch --------------------------------------------------------
__global__ void k_first_pos(const int32_t *__restrict__ mu, int64_t n, int32_t *firstpos) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) atomicMin(&firstpos[mu[i]], (int32_t)i);
}

__global__ void k_first_flags(const int32_t *__restrict__ mu, const int32_t *__restrict__ firstpos,
                              int64_t n, int32_t *flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flags[i] = (firstpos[mu[i]] == (int32_t)i) ? 1 : 0;
}

__global__ void k_first_label(const int32_t *__restrict__ mu, const int32_t *__restrict__ flags,
                              const int32_t *__restrict__ excl, int64_t n, int32_t *label_of,
                              int32_t *node_perm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flags[i]) {
        label_of[mu[i]] = excl[i];
        node_perm[excl[i]] = mu[i];
    }
}

__global__ void k_relabel(const int32_t *__restrict__ mu, const int32_t *__restrict__ label_of,
                          int64_t n, int32_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = label_of[mu[i]];
}

// ---- node graph, degrees ---------------------------------------
constexpr int kMaxCand = 384;  // candidate neighbour entries of one node (valence x Np)

__global__ void k_count_nodes(const int32_t *__restrict__ mu, int64_t n, int32_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(&cnt[mu[i]], 1);
}

__global__ void k_incidence(const int32_t *__restrict__ mu, int64_t n, const int32_t *__restrict__ ptr,
                            int32_t *fill, int32_t *inc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) inc[ptr[mu[i]] + atomicAdd(&fill[mu[i]], 1)] = (int32_t)i;  // entry index (order fixed later)
}

// More than kMaxCand distinct neighbours (high-valence fans, high orders): the ascending distinct
// list by repeated minimum search over the node's element entries, O(degree x entries), no list.
__device__ void node_nbrs_rescan(const int32_t *__restrict__ mu, int Np, const int32_t *__restrict__ iptr,
                                 const int32_t *__restrict__ inc, int64_t g, int32_t *deg,
                                 const int64_t *__restrict__ aptr, int32_t *__restrict__ adj) {
    int32_t prev = -1;
    int k = 0;
    for (;;) {
        int32_t best = INT_MAX;
        for (int j = iptr[g]; j < iptr[g + 1]; j++) {
            const int64_t e = inc[j] / Np;
            for (int q = 0; q < Np; q++) {
                const int32_t o = mu[e * Np + q];
                if (o != (int32_t)g && o > prev && o < best) best = o;
            }
        }
        if (best == INT_MAX) break;
        if (adj) adj[aptr[g] + k] = best;
        k++;
        prev = best;
    }
    if (!adj) deg[g] = k;
}

// Distinct other nodes of the elements holding g: count (adj == nullptr) or
// write them ascending at adj + aptr[g].  Nodes with more than kMaxCand of them take the
// rescan path (same result).  (*bad is no longer set.)
__global__ void k_node_nbrs(const int32_t *__restrict__ mu, int Np, const int32_t *__restrict__ iptr,
                            const int32_t *__restrict__ inc, int64_t N, int32_t *deg,
                            const int64_t *__restrict__ aptr, int32_t *__restrict__ adj, int32_t *bad) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= N) return;
    int32_t c[kMaxCand];
    int m = 0;
    for (int j = iptr[g]; j < iptr[g + 1]; j++) {
        const int64_t e = inc[j] / Np;
        for (int q = 0; q < Np; q++) {
            const int32_t o = mu[e * Np + q];
            if (o == (int32_t)g) continue;
            int k = m - 1;  // insertion into the ascending unique list
            while (k >= 0 && c[k] > o) k--;
            if (k >= 0 && c[k] == o) continue;
            if (m == kMaxCand) {  // a high-valence node: the slow path without the local list
                node_nbrs_rescan(mu, Np, iptr, inc, g, deg, aptr, adj);
                return;
            }
            for (int r = m; r > k + 1; r--) c[r] = c[r - 1];
            c[k + 1] = o;
            m++;
        }
    }
    if (adj) {
        for (int k = 0; k < m; k++) adj[aptr[g] + k] = c[k];
    } else {
        deg[g] = m;
    }
}

// ---- degree-sorted first-touch groups (PAPER.md:318 step 2) ----------------------
// Element e's newly touched nodes hold the labels [excl[e Np], excl[(e+1) Np]);
// sort them by (degree, old id).
__global__ void k_group_sort(const int32_t *__restrict__ excl, int64_t E, int Np, const int32_t *__restrict__ deg,
                             int32_t *node_perm) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int32_t a = excl[e * Np], b = excl[(e + 1) * Np];
    int32_t v[kMaxNp];
    const int n = b - a;
    for (int i = 0; i < n; i++) v[i] = node_perm[a + i];
    for (int i = 1; i < n; i++) {
        const int32_t x = v[i];
        int j = i - 1;
        while (j >= 0 && (deg[v[j]] > deg[x] || (deg[v[j]] == deg[x] && v[j] > x))) { v[j + 1] = v[j]; j--; }
        v[j + 1] = x;
    }
    for (int i = 0; i < n; i++) node_perm[a + i] = v[i];
}

__global__ void k_label_from_perm(const int32_t *__restrict__ node_perm, int64_t n, int32_t *label_of) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) label_of[node_perm[i]] = (int32_t)i;
}

// ---- Conn. / Dist. strategies (reading R20) -------------------
__global__ void k_key_degree(const int32_t *__restrict__ deg, int64_t N, uint64_t *key) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < N) key[g] = (uint64_t)(uint32_t)deg[g];
}

// Squared distance of every node to (x0, y0), from its canonical coordinates:
// vertices exact; edge node m (1..P-1) from the lower-id end a: a + t_m (b - a);
// P3 interior node: ((v0 + v1) + v2) / 3.  Explicit round-to-nearest, no FMA.
// A node written by several elements gets identical bits from each.
__constant__ double c_edge_t[8];
__global__ void k_key_dist(const double *__restrict__ vxy, const int32_t *__restrict__ tri,
                           const int32_t *__restrict__ mu, int64_t E, int P, double x0, double y0,
                           uint64_t *key) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int Np = (P + 1) * (P + 2) / 2;
    const int32_t v[3] = {tri[3 * e], tri[3 * e + 1], tri[3 * e + 2]};
    int p = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, p++) {
            double x, y;
            if ((i == 0 && j == 0) || (i == P && j == 0) || (i == 0 && j == P)) {
                const int32_t w = (j == P) ? v[2] : (i == P ? v[1] : v[0]);
                x = vxy[2 * w];
                y = vxy[2 * w + 1];
            } else if (j == 0 || i == 0 || i + j == P) {
                int32_t a, b;
                int m;
                if (j == 0) { a = v[0]; b = v[1]; m = i; }
                else if (i == 0) { a = v[0]; b = v[2]; m = j; }
                else { a = v[1]; b = v[2]; m = j; }
                if (a > b) { const int32_t t = a; a = b; b = t; m = P - m; }
                const double t = c_edge_t[m - 1];
                x = __dadd_rn(vxy[2 * a], __dmul_rn(t, __dsub_rn(vxy[2 * b], vxy[2 * a])));
                y = __dadd_rn(vxy[2 * a + 1], __dmul_rn(t, __dsub_rn(vxy[2 * b + 1], vxy[2 * a + 1])));
            } else {
                x = __ddiv_rn(__dadd_rn(__dadd_rn(vxy[2 * v[0]], vxy[2 * v[1]]), vxy[2 * v[2]]), 3.0);
                y = __ddiv_rn(__dadd_rn(__dadd_rn(vxy[2 * v[0] + 1], vxy[2 * v[1] + 1]), vxy[2 * v[2] + 1]), 3.0);
            }
            const double dx = __dsub_rn(x, x0), dy = __dsub_rn(y, y0);
            const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            key[mu[e * Np + p]] = (uint64_t)__double_as_longlong(d2);  // d2 >= +0: bits are monotone
        }
}

__global__ void k_scatter_rank(const int32_t *__restrict__ sorted_ids, int64_t N, int32_t *rank) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) rank[sorted_ids[i]] = (int32_t)i;
}

// Smallest-rank unvisited node.
__global__ void k_min_unvisited(const int32_t *__restrict__ pos, const int32_t *__restrict__ rank, int64_t N,
                                int32_t *best) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < N && pos[g] < 0) atomicMin(best, rank[g]);
}

__global__ void k_bfs_start(const int32_t *__restrict__ sorted_ids, const int32_t *best, int32_t q, int32_t *pos,
                            int32_t *order) {
    const int32_t s = sorted_ids[*best];
    pos[s] = q;
    order[q] = s;
}

// Frontier positions [a, b): every unvisited neighbour w of order[q] records
// the smallest such q (its Cuthill-McKee parent); the first claimer appends w.
__global__ void k_bfs_expand(const int32_t *__restrict__ order, int32_t a, int32_t b,
                             const int64_t *__restrict__ aptr, const int32_t *__restrict__ adj,
                             const int32_t *__restrict__ pos, int32_t *par, int32_t *cand, int32_t *cnt) {
    const int64_t q = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= b) return;
    const int32_t u = order[q];
    for (int64_t j = aptr[u]; j < aptr[u + 1]; j++) {
        const int32_t w = adj[j];
        if (pos[w] >= 0) continue;
        if (atomicMin(&par[w], (int32_t)q) == INT_MAX) cand[atomicAdd(cnt, 1)] = w;
    }
}

__global__ void k_bfs_keys(const int32_t *__restrict__ cand, const int32_t *cnt, const int32_t *__restrict__ par,
                           const int32_t *__restrict__ rank, uint64_t *key) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= *cnt) return;
    const int32_t w = cand[i];
    key[i] = ((uint64_t)(uint32_t)par[w] << 32) | (uint32_t)rank[w];
}

__global__ void k_bfs_assign(const int32_t *__restrict__ sorted, const int32_t *cnt, int32_t b, int32_t *pos,
                             int32_t *order) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= *cnt) return;
    const int32_t w = sorted[i];
    pos[w] = b + (int32_t)i;
    order[b + i] = w;
}

// Element list: an element is appended at the first of its nodes in visit
// order, elements of one node by ascending id -> key (min node position, e).
__global__ void k_elem_first_pos(const int32_t *__restrict__ mu, int64_t E, int Np, const int32_t *__restrict__ pos,
                                 uint64_t *key, int32_t *ids) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t m = INT_MAX;
    for (int p = 0; p < Np; p++) m = min(m, pos[mu[e * Np + p]]);
    key[e] = ((uint64_t)(uint32_t)m << 32) | (uint32_t)e;
    ids[e] = (int32_t)e;
}

__global__ void k_find_i32(const int32_t *__restrict__ a, int64_t n, int32_t v, int32_t *first) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && a[i] == v) atomicMin(first, (int32_t)i);
}

__global__ void k_i32_to_i64(const int32_t *__restrict__ a, int64_t n, int64_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i <= n) out[i] = (i < n) ? a[i] : 0;
}

// temporary device allocation on the stream
struct Tmp {
    void *p = nullptr;
    cudaStream_t s;
    explicit Tmp(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t n) { return dev_malloc(&p, n ? n : 16, s); }
    ~Tmp() { if (p) dev_free(p, s); }
};

#define RET(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)

}  // namespace

cudaError_t launch_bbox(const double *vxy, int64_t nv, double *out4, cudaStream_t s) {
    const int nb = 296;
    Tmp part(s);
    RET(part.alloc(sizeof(double) * 4 * nb));
    k_bbox_partial<<<nb, 256, 0, s>>>(vxy, nv, (double *)part.p);
    k_bbox_final<<<1, 32, 0, s>>>((double *)part.p, nb, out4);
    return cudaGetLastError();
}

cudaError_t launch_orient(const double *vxy, const int32_t *tri, int64_t E, int64_t nv, int32_t *tri_or,
                          int32_t *bad, cudaStream_t s) {
    k_orient<<<blocks_for(E), kThreads, 0, s>>>(vxy, tri, E, nv, tri_or, bad);
    return cudaGetLastError();
}

cudaError_t launch_hilbert_keys(const double *vxy, const int32_t *tri, int64_t E, double xm0,
                                double xm1, double ws, double hs, int32_t wb, int32_t hb,
                                uint32_t *keys, cudaStream_t s) {
    k_hilbert_keys<<<blocks_for(E), kThreads, 0, s>>>(vxy, tri, E, xm0, xm1, ws, hs, wb, hb, keys);
    return cudaGetLastError();
}

cudaError_t launch_random_keys(int64_t E, uint64_t seed, uint64_t *keys, cudaStream_t s) {
    k_random_keys<<<blocks_for(E), kThreads, 0, s>>>(E, seed, keys);
    return cudaGetLastError();
}

cudaError_t launch_iota(int32_t *a, int64_t n, cudaStream_t s) {
    k_iota<<<blocks_for(n), kThreads, 0, s>>>(a, n);
    return cudaGetLastError();
}

cudaError_t launch_fill_i32(int32_t *a, int64_t n, int32_t v, cudaStream_t s) {
    k_fill_i32<<<blocks_for(n), kThreads, 0, s>>>(a, n, v);
    return cudaGetLastError();
}

cudaError_t sort_pairs_u32(const uint32_t *keys, const int32_t *vals, uint32_t *keys_out,
                           int32_t *vals_out, int64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, vals, vals_out, n, 0,
                                        end_bit, s));
    Tmp t(s);
    RET(t.alloc(bytes));
    return cub::DeviceRadixSort::SortPairs(t.p, bytes, keys, keys_out, vals, vals_out, n, 0,
                                           end_bit, s);
}

cudaError_t sort_pairs_u64(const uint64_t *keys, const int32_t *vals, uint64_t *keys_out,
                           int32_t *vals_out, int64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, vals, vals_out, n, 0,
                                        end_bit, s));
    Tmp t(s);
    RET(t.alloc(bytes));
    return cub::DeviceRadixSort::SortPairs(t.p, bytes, keys, keys_out, vals, vals_out, n, 0,
                                           end_bit, s);
}

cudaError_t canonical_nodes(const int32_t *tri_or, int64_t nv, int64_t E, int P, int32_t *mu_can,
                            int64_t *n_edges, int64_t *n_unused, int32_t *first_unused,
                            cudaStream_t s) {
    const LocalNode *ln = local_nodes(P);
    if (!ln) return cudaErrorInvalidValue;
    const int Np = (P + 1) * (P + 2) / 2;
    int h_ln[kMaxNp][3] = {};
    for (int p = 0; p < Np; p++) { h_ln[p][0] = ln[p].kind; h_ln[p][1] = ln[p].which; h_ln[p][2] = ln[p].m; }
    RET(cudaMemcpyToSymbolAsync(c_ln, h_ln, sizeof(h_ln), 0, cudaMemcpyHostToDevice, s));
    const int64_t n = 3 * E;
    Tmp keys(s), keys2(s), vals(s), vals2(s), flags(s), incl(s), eid(s), used(s), cnt(s), scr(s);
    RET(keys.alloc(sizeof(uint64_t) * n));
    RET(keys2.alloc(sizeof(uint64_t) * n));
    RET(vals.alloc(sizeof(int32_t) * n));
    RET(vals2.alloc(sizeof(int32_t) * n));
    RET(flags.alloc(sizeof(int32_t) * n));
    RET(incl.alloc(sizeof(int32_t) * n));
    RET(eid.alloc(sizeof(int32_t) * n));
    k_edge_keys<<<blocks_for(n), kThreads, 0, s>>>(tri_or, E, (uint64_t *)keys.p, (int32_t *)vals.p);
    int vbits = 1;
    while (vbits < 32 && ((int64_t)1 << vbits) <= nv) vbits++;
    RET(sort_pairs_u64((uint64_t *)keys.p, (int32_t *)vals.p, (uint64_t *)keys2.p,
                       (int32_t *)vals2.p, n, 32 + vbits, s));
    k_heads<<<blocks_for(n), kThreads, 0, s>>>((uint64_t *)keys2.p, n, (int32_t *)flags.p);
    size_t bytes = 0;
    RET(cub::DeviceScan::InclusiveSum(nullptr, bytes, (int32_t *)flags.p, (int32_t *)incl.p, n, s));
    RET(scr.alloc(bytes));
    RET(cub::DeviceScan::InclusiveSum(scr.p, bytes, (int32_t *)flags.p, (int32_t *)incl.p, n, s));
    k_edge_scatter<<<blocks_for(n), kThreads, 0, s>>>((int32_t *)vals2.p, (int32_t *)incl.p, n,
                                                      (int32_t *)eid.p);
    int32_t ne32 = 0;
    RET(cudaMemcpyAsync(&ne32, (int32_t *)incl.p + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    *n_edges = ne32;
    k_mu_canonical<<<blocks_for(E), kThreads, 0, s>>>(tri_or, (int32_t *)eid.p, E, P, Np, nv, ne32,
                                                      mu_can);
    // every vertex must be used (a vertex no element touches would have M-bar = 0)
    RET(used.alloc(sizeof(int32_t) * (nv + 1)));
    RET(cudaMemsetAsync(used.p, 0, sizeof(int32_t) * (nv + 1), s));
    k_mark_used<<<blocks_for(3 * E), kThreads, 0, s>>>(tri_or, E, (int32_t *)used.p);
    int32_t *fu = (int32_t *)used.p + nv;
    k_fill_i32<<<1, 32, 0, s>>>(fu, 1, INT_MAX);
    k_first_unused<<<blocks_for(nv), kThreads, 0, s>>>((int32_t *)used.p, nv, fu);
    int32_t h_fu = 0;
    RET(cudaMemcpyAsync(&h_fu, fu, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    *first_unused = h_fu;
    *n_unused = (h_fu == INT_MAX) ? 0 : 1;
    return cudaGetLastError();
}

cudaError_t launch_permute_rows(const int32_t *src, const int32_t *perm, int64_t E, int w,
                                int32_t *dst, cudaStream_t s) {
    k_permute_rows<<<blocks_for(E * w), kThreads, 0, s>>>(src, perm, E, w, dst);
    return cudaGetLastError();
}

cudaError_t first_touch(const int32_t *mu, int64_t E, int Np, int64_t N, int32_t *node_perm,
                        int32_t *mu_out, int64_t *n_labels, cudaStream_t s, const int32_t *deg) {
    const int64_t n = E * Np;
    Tmp firstpos(s), flags(s), excl(s), label(s), scr(s);
    RET(firstpos.alloc(sizeof(int32_t) * N));
    RET(flags.alloc(sizeof(int32_t) * (n + 1)));
    RET(excl.alloc(sizeof(int32_t) * (n + 1)));
    RET(label.alloc(sizeof(int32_t) * N));
    k_fill_i32<<<blocks_for(N), kThreads, 0, s>>>((int32_t *)firstpos.p, N, INT_MAX);
    k_first_pos<<<blocks_for(n), kThreads, 0, s>>>(mu, n, (int32_t *)firstpos.p);
    k_first_flags<<<blocks_for(n), kThreads, 0, s>>>(mu, (int32_t *)firstpos.p, n, (int32_t *)flags.p);
    RET(cudaMemsetAsync((int32_t *)flags.p + n, 0, sizeof(int32_t), s));
    size_t bytes = 0;
    RET(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t *)flags.p, (int32_t *)excl.p, n + 1, s));
    RET(scr.alloc(bytes));
    RET(cub::DeviceScan::ExclusiveSum(scr.p, bytes, (int32_t *)flags.p, (int32_t *)excl.p, n + 1, s));
    k_first_label<<<blocks_for(n), kThreads, 0, s>>>(mu, (int32_t *)flags.p, (int32_t *)excl.p, n,
                                                     (int32_t *)label.p, node_perm);
    if (deg) {  // PAPER.md:318 step 2: each element's group sorted by (degree, old id)
        k_group_sort<<<blocks_for(E), kThreads, 0, s>>>((int32_t *)excl.p, E, Np, deg, node_perm);
        k_label_from_perm<<<blocks_for(N), kThreads, 0, s>>>(node_perm, N, (int32_t *)label.p);
    }
    k_relabel<<<blocks_for(n), kThreads, 0, s>>>(mu, (int32_t *)label.p, n, mu_out);
    int32_t cnt = 0;
    RET(cudaMemcpyAsync(&cnt, (int32_t *)excl.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    *n_labels = cnt;
    return cudaGetLastError();
}


cudaError_t build_node_graph(const int32_t *mu, int64_t E, int Np, int64_t N, bool want_adj, DevGraph &g,
                             int *bad, cudaStream_t s) {
    g = DevGraph{};
    const int64_t n = E * Np;
    Tmp cnt(s), iptr(s), fill(s), inc(s), scr(s), dbad(s);
    RET(cnt.alloc(sizeof(int32_t) * (N + 1)));
    RET(iptr.alloc(sizeof(int32_t) * (N + 1)));
    RET(fill.alloc(sizeof(int32_t) * (N + 1)));
    RET(inc.alloc(sizeof(int32_t) * (n + 1)));
    RET(dbad.alloc(sizeof(int32_t)));
    RET(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * (N + 1), s));
    RET(cudaMemsetAsync(fill.p, 0, sizeof(int32_t) * (N + 1), s));
    RET(cudaMemsetAsync(dbad.p, 0, sizeof(int32_t), s));
    k_count_nodes<<<blocks_for(n), kThreads, 0, s>>>(mu, n, (int32_t *)cnt.p);
    size_t bytes = 0;
    RET(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t *)cnt.p, (int32_t *)iptr.p, N + 1, s));
    RET(scr.alloc(bytes));
    RET(cub::DeviceScan::ExclusiveSum(scr.p, bytes, (int32_t *)cnt.p, (int32_t *)iptr.p, N + 1, s));
    k_incidence<<<blocks_for(n), kThreads, 0, s>>>(mu, n, (int32_t *)iptr.p, (int32_t *)fill.p, (int32_t *)inc.p);
    RET(dev_malloc((void **)&g.deg, sizeof(int32_t) * (N + 1), s));
    k_node_nbrs<<<blocks_for(N, 128), 128, 0, s>>>(mu, Np, (int32_t *)iptr.p, (int32_t *)inc.p, N, g.deg, nullptr,
                                                   nullptr, (int32_t *)dbad.p);
    if (want_adj) {
        RET(dev_malloc((void **)&g.aptr, sizeof(int64_t) * (N + 1), s));
        Tmp deg64(s), scr2(s);
        RET(deg64.alloc(sizeof(int64_t) * (N + 1)));
        k_i32_to_i64<<<blocks_for(N + 1), kThreads, 0, s>>>(g.deg, N, (int64_t *)deg64.p);
        bytes = 0;
        RET(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t *)deg64.p, g.aptr, N + 1, s));
        RET(scr2.alloc(bytes));
        RET(cub::DeviceScan::ExclusiveSum(scr2.p, bytes, (int64_t *)deg64.p, g.aptr, N + 1, s));
        RET(cudaMemcpyAsync(&g.nadj, g.aptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RET(cudaStreamSynchronize(s));
        RET(dev_malloc((void **)&g.adj, sizeof(int32_t) * (g.nadj + 1), s));
        k_node_nbrs<<<blocks_for(N, 128), 128, 0, s>>>(mu, Np, (int32_t *)iptr.p, (int32_t *)inc.p, N, nullptr,
                                                       g.aptr, g.adj, (int32_t *)dbad.p);
    }
    int32_t hb = 0;
    RET(cudaMemcpyAsync(&hb, dbad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    *bad = hb;
    return cudaGetLastError();
}

void free_node_graph(DevGraph &g, cudaStream_t s) {
    if (g.deg) dev_free(g.deg, s);
    if (g.aptr) dev_free(g.aptr, s);
    if (g.adj) dev_free(g.adj, s);
    g = DevGraph{};
}

cudaError_t strategy_order(const int32_t *mu_can, const double *vxy, const int32_t *tri_or, int64_t E, int P,
                           int64_t N, int strategy, const DevGraph &g, const double *edge_t, double x0, double y0,
                           int32_t *elem_perm, int32_t *order, int64_t *n_levels, cudaStream_t s) {
    const int Np = (P + 1) * (P + 2) / 2;
    Tmp key(s), key2(s), ids(s), ids2(s), rank(s), pos(s), par(s), cand(s), cnt(s), best(s), scr(s);
    RET(key.alloc(sizeof(uint64_t) * (N > E ? N : E)));
    RET(key2.alloc(sizeof(uint64_t) * (N > E ? N : E)));
    RET(ids.alloc(sizeof(int32_t) * (N > E ? N : E)));
    RET(ids2.alloc(sizeof(int32_t) * (N > E ? N : E)));
    RET(rank.alloc(sizeof(int32_t) * N));
    RET(pos.alloc(sizeof(int32_t) * N));
    RET(par.alloc(sizeof(int32_t) * N));
    RET(cand.alloc(sizeof(int32_t) * N));
    RET(cnt.alloc(sizeof(int32_t)));
    RET(best.alloc(sizeof(int32_t)));
    // node key: degree (Conn.) or squared distance to (x0, y0) (Dist.); rank = position in (key, id) order
    if (strategy == 0) {
        k_key_degree<<<blocks_for(N), kThreads, 0, s>>>(g.deg, N, (uint64_t *)key.p);
    } else {
        RET(cudaMemcpyToSymbolAsync(c_edge_t, edge_t, sizeof(double) * (P - 1), 0, cudaMemcpyHostToDevice, s));
        k_key_dist<<<blocks_for(E), kThreads, 0, s>>>(vxy, tri_or, mu_can, E, P, x0, y0, (uint64_t *)key.p);
    }
    k_iota<<<blocks_for(N), kThreads, 0, s>>>((int32_t *)ids.p, N);
    RET(sort_pairs_u64((uint64_t *)key.p, (int32_t *)ids.p, (uint64_t *)key2.p, (int32_t *)ids2.p, N, 64, s));
    const int32_t *sorted_ids = (const int32_t *)ids2.p;
    k_scatter_rank<<<blocks_for(N), kThreads, 0, s>>>(sorted_ids, N, (int32_t *)rank.p);
    k_fill_i32<<<blocks_for(N), kThreads, 0, s>>>((int32_t *)pos.p, N, -1);
    k_fill_i32<<<blocks_for(N), kThreads, 0, s>>>((int32_t *)par.p, N, INT_MAX);
    // one sort workspace for every level (largest case: N keys)
    int nbits = 1;
    while (nbits < 31 && ((int64_t)1 << nbits) < N) nbits++;
    size_t sbytes = 0;
    RET(cub::DeviceRadixSort::SortPairs(nullptr, sbytes, (uint64_t *)key.p, (uint64_t *)key2.p, (int32_t *)cand.p,
                                        (int32_t *)ids.p, (int)N, 0, 32 + nbits, s));
    RET(scr.alloc(sbytes));
    int64_t a = 0, b = 0, levels = 0;
    while (b < N) {
        if (a == b) {  // (re)start at the smallest-key unvisited node
            k_fill_i32<<<1, 32, 0, s>>>((int32_t *)best.p, 1, INT_MAX);
            k_min_unvisited<<<blocks_for(N), kThreads, 0, s>>>((int32_t *)pos.p, (int32_t *)rank.p, N,
                                                               (int32_t *)best.p);
            k_bfs_start<<<1, 1, 0, s>>>(sorted_ids, (int32_t *)best.p, (int32_t)b, (int32_t *)pos.p, order);
            b++;
        }
        RET(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t), s));
        k_bfs_expand<<<blocks_for(b - a, 128), 128, 0, s>>>(order, (int32_t)a, (int32_t)b, g.aptr, g.adj,
                                                            (int32_t *)pos.p, (int32_t *)par.p, (int32_t *)cand.p,
                                                            (int32_t *)cnt.p);
        int32_t c = 0;
        RET(cudaMemcpyAsync(&c, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        RET(cudaStreamSynchronize(s));
        a = b;
        levels++;
        if (c == 0) continue;
        k_bfs_keys<<<blocks_for(c), kThreads, 0, s>>>((int32_t *)cand.p, (int32_t *)cnt.p, (int32_t *)par.p,
                                                      (int32_t *)rank.p, (uint64_t *)key.p);
        RET(cub::DeviceRadixSort::SortPairs(scr.p, sbytes, (uint64_t *)key.p, (uint64_t *)key2.p, (int32_t *)cand.p,
                                            (int32_t *)ids.p, c, 0, 32 + nbits, s));
        k_bfs_assign<<<blocks_for(c), kThreads, 0, s>>>((int32_t *)ids.p, (int32_t *)cnt.p, (int32_t)b,
                                                        (int32_t *)pos.p, order);
        b += c;
    }
    *n_levels = levels;
    // element list (key = first visited node, then element id)
    k_elem_first_pos<<<blocks_for(E), kThreads, 0, s>>>(mu_can, E, Np, (int32_t *)pos.p, (uint64_t *)key.p,
                                                        (int32_t *)ids.p);
    RET(sort_pairs_u64((uint64_t *)key.p, (int32_t *)ids.p, (uint64_t *)key2.p, elem_perm, E, 64, s));
    return cudaGetLastError();
}

cudaError_t launch_find_i32(const int32_t *a, int64_t n, int32_t v, int32_t *first, cudaStream_t s) {
    k_fill_i32<<<1, 32, 0, s>>>(first, 1, INT_MAX);
    k_find_i32<<<blocks_for(n), kThreads, 0, s>>>(a, n, v, first);
    return cudaGetLastError();
}

cudaError_t relabel_from_perm(const int32_t *mu, int64_t n, const int32_t *node_perm, int64_t N, int32_t *mu_out,
                              cudaStream_t s) {
    Tmp label(s);
    RET(label.alloc(sizeof(int32_t) * N));
    k_label_from_perm<<<blocks_for(N), kThreads, 0, s>>>(node_perm, N, (int32_t *)label.p);
    k_relabel<<<blocks_for(n), kThreads, 0, s>>>(mu, (int32_t *)label.p, n, mu_out);
    return cudaGetLastError();
}

}  // namespace sem
