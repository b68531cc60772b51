// partition_gpu.cu -- the multi-GPU partition of partition.cpp on the GPU
// (product path).  Rank r owns the global elements
// [floor(rE/G), floor((r+1)E/G)) of the Hilbert order; its local nodes are the
// nodes those elements touch, in ascending global id; a local node is remote
// (an interface node) if another rank touches it and owned (for I/O) if no
// lower rank does.  The per-node rank masks, the local numbering and the local
// connectivity are built with one atomic pass and scans; only the interface
// nodes' masks (a few tens of thousands) come back to the host, where the
// neighbour lists and the rank-ordered summation lists are derived exactly as
// in partition.cpp (tests/test_gpu_multirank.py checks both agree).
#include <cub/cub.cuh>

#include "kernels.h"

namespace sem {

namespace {

constexpr int kT = 256;

inline unsigned nb(int64_t n) {
    int64_t b = (n + kT - 1) / kT;
    return (unsigned)(b < 1 ? 1 : b);
}

#define RET(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)

__host__ __device__ inline int64_t range_start(int q, int64_t E, int G) { return (int64_t)q * E / G; }

__global__ void k_rank_masks(const int32_t *__restrict__ mu, int64_t E, int Np, int G, uint32_t *mask) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= E * Np) return;
    const int64_t e = i / Np;
    int q = (int)(e * G / E);  // owner: start(q) <= e < start(q+1)
    while (q + 1 < G && range_start(q + 1, E, G) <= e) q++;
    while (q > 0 && range_start(q, E, G) > e) q--;
    atomicOr(&mask[mu[i]], 1u << q);
}

__global__ void k_flag_bit(const uint32_t *__restrict__ mask, int64_t n, uint32_t bit, int32_t *flag) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < n) flag[g] = (mask[g] & bit) ? 1 : 0;
}

__global__ void k_local_maps(const uint32_t *__restrict__ mask, const int32_t *__restrict__ g2l, int64_t N,
                             uint32_t me, int32_t *loc2glob, uint8_t *remote, uint8_t *owned, int32_t *rflag,
                             uint32_t *lmask) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= N || !(mask[g] & me)) return;
    const int32_t l = g2l[g];
    const uint32_t m = mask[g];
    loc2glob[l] = (int32_t)g;
    remote[l] = (m & ~me) ? 1 : 0;
    owned[l] = (m & (me - 1)) ? 0 : 1;
    rflag[l] = (m & ~me) ? 1 : 0;
    lmask[l] = m;
}

__global__ void k_mu_local(const int32_t *__restrict__ mu, int64_t k0, int64_t n, const int32_t *__restrict__ g2l,
                           int32_t *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = g2l[mu[k0 + k]];
}

__global__ void k_if_masks(const int32_t *__restrict__ rflag, const int32_t *__restrict__ ridx,
                           const uint32_t *__restrict__ lmask, int64_t NL, uint32_t *ifmask) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l < NL && rflag[l]) ifmask[ridx[l]] = lmask[l];
}

template <typename T>
cudaError_t excl_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    RET(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    void *t = nullptr;
    RET(dev_malloc(&t, bytes ? bytes : 16, s));
    cudaError_t e = cub::DeviceScan::ExclusiveSum(t, bytes, in, out, n, s);
    dev_free(t, s);
    return e;
}

// I/O maps: loc_can[l] = node_perm[loc2glob[l]]; owned subset compacted
__global__ void k_loc_can(const int32_t *__restrict__ loc2glob, const int32_t *__restrict__ node_perm, int64_t NL,
                          int32_t *loc_can) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l < NL) loc_can[l] = node_perm[loc2glob[l]];
}

__global__ void k_owned_flag(const uint8_t *__restrict__ owned, int64_t NL, int32_t *f) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l <= NL) f[l] = (l < NL && owned[l]) ? 1 : 0;
}

__global__ void k_owned_lists(const int32_t *__restrict__ f, const int32_t *__restrict__ idx, int64_t NL,
                              const int32_t *__restrict__ loc_int, const int32_t *__restrict__ loc_can,
                              const int32_t *__restrict__ loc2glob, int32_t *own_int, int32_t *own_can,
                              int32_t *own_ft) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= NL || !f[l]) return;
    const int32_t j = idx[l];
    own_int[j] = loc_int[l];
    own_can[j] = loc_can[l];
    own_ft[j] = loc2glob[l];
}

}  // namespace

cudaError_t build_partition_gpu(const int32_t *d_mu, int64_t E, int Np, int64_t N, int rank, int world,
                                const DeviceAlloc &dalloc, DevPartition &P, std::string &err, cudaStream_t s) {
    P = DevPartition();
    if (world < 2 || world > 32 || rank < 0 || rank >= world) {
        err = "build_partition_gpu: world size must be in [2, 32]";
        return cudaSuccess;
    }
    P.e0 = range_start(rank, E, world);
    P.e1 = range_start(rank + 1, E, world);
    if (P.e1 <= P.e0) {
        err = "build_partition: rank " + std::to_string(rank) + " has no elements";
        return cudaSuccess;
    }
    const uint32_t me = 1u << rank;
    uint32_t *mask = nullptr;
    int32_t *flag = nullptr, *g2l = nullptr;
    RET(dev_malloc((void **)&mask, 4 * (N + 1), s));
    RET(dev_malloc((void **)&flag, 4 * (N + 1), s));
    RET(dev_malloc((void **)&g2l, 4 * (N + 1), s));
    struct F { cudaStream_t s; void *a, *b, *c; ~F() { dev_free(a, s); dev_free(b, s); dev_free(c, s); } }
    fr{s, mask, flag, g2l};
    RET(cudaMemsetAsync(mask, 0, 4 * (N + 1), s));
    RET(cudaMemsetAsync(flag, 0, 4 * (N + 1), s));
    k_rank_masks<<<nb(E * Np), kT, 0, s>>>(d_mu, E, Np, world, mask);
    k_flag_bit<<<nb(N), kT, 0, s>>>(mask, N, me, flag);
    RET(excl_scan(flag, g2l, N + 1, s));
    int32_t nl32 = 0;
    RET(cudaMemcpyAsync(&nl32, g2l + N, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    P.NL = nl32;
    const int64_t NL = P.NL, El = P.e1 - P.e0;
    RET(dalloc((void **)&P.loc2glob, 4 * (size_t)(NL + 1)));
    RET(dalloc((void **)&P.remote, (size_t)NL + 16));
    RET(dalloc((void **)&P.owned, (size_t)NL + 16));
    RET(dalloc((void **)&P.mu_local, 4 * (size_t)(El * Np + 1)));
    int32_t *rflag = nullptr, *ridx = nullptr;
    uint32_t *lmask = nullptr;
    RET(dev_malloc((void **)&rflag, 4 * (NL + 1), s));
    RET(dev_malloc((void **)&ridx, 4 * (NL + 1), s));
    RET(dev_malloc((void **)&lmask, 4 * (NL + 1), s));
    F fr2{s, rflag, ridx, lmask};
    RET(cudaMemsetAsync(rflag, 0, 4 * (NL + 1), s));
    k_local_maps<<<nb(N), kT, 0, s>>>(mask, g2l, N, me, P.loc2glob, P.remote, P.owned, rflag, lmask);
    k_mu_local<<<nb(El * Np), kT, 0, s>>>(d_mu, P.e0 * Np, El * Np, g2l, P.mu_local);
    RET(excl_scan(rflag, ridx, NL + 1, s));
    int32_t nif32 = 0;
    RET(cudaMemcpyAsync(&nif32, ridx + NL, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    const int64_t nif = nif32;
    P.n_if = nif;
    std::vector<uint32_t> ifm((size_t)nif + 1);
    if (nif > 0) {
        uint32_t *d_ifm = nullptr;
        RET(dev_malloc((void **)&d_ifm, 4 * (nif + 1), s));
        k_if_masks<<<nb(NL), kT, 0, s>>>(rflag, ridx, lmask, NL, d_ifm);
        RET(cudaMemcpyAsync(ifm.data(), d_ifm, 4 * nif, cudaMemcpyDeviceToHost, s));
        dev_free(d_ifm, s);
        RET(cudaStreamSynchronize(s));
    }
    // neighbours, per-neighbour send lists, rank-ordered summation lists (as partition.cpp)
    uint32_t nbr_mask = 0;
    for (int64_t i = 0; i < nif; i++) nbr_mask |= ifm[i];
    nbr_mask &= ~me;
    for (int q = 0; q < world; q++)
        if (nbr_mask & (1u << q)) P.nbr.push_back(q);
    const int nn = (int)P.nbr.size();
    P.nbr_off.assign(nn + 1, 0);
    std::vector<std::vector<int32_t>> pos_in(nn, std::vector<int32_t>(nif, -1));
    for (int k = 0; k < nn; k++) {
        const uint32_t bit = 1u << P.nbr[k];
        int32_t cnt = 0;
        for (int64_t i = 0; i < nif; i++)
            if (ifm[i] & bit) {
                pos_in[k][i] = P.nbr_off[k] + cnt;
                P.send_if.push_back((int32_t)i);
                cnt++;
            }
        P.nbr_off[k + 1] = P.nbr_off[k] + cnt;
    }
    P.sum_start.assign(nif + 1, 0);
    for (int64_t i = 0; i < nif; i++) {
        for (int q = 0; q < world; q++) {
            if (!(ifm[i] & (1u << q))) continue;
            if (q == rank) {
                P.sum_src.push_back((int32_t)i);
            } else {
                const int k = (int)(std::lower_bound(P.nbr.begin(), P.nbr.end(), q) - P.nbr.begin());
                P.sum_src.push_back((int32_t)(nif + pos_in[k][i]));
            }
        }
        P.sum_start[i + 1] = (int32_t)P.sum_src.size();
    }
    return cudaGetLastError();
}

cudaError_t partition_io_maps(const DevPartition &P, const int32_t *d_node_perm, const int32_t *d_loc_int,
                              const DeviceAlloc &dalloc, int32_t **loc_can, int32_t **own_int, int32_t **own_can,
                              int32_t **own_ft, int64_t *n_own, cudaStream_t s) {
    const int64_t NL = P.NL;
    RET(dalloc((void **)loc_can, 4 * (size_t)(NL + 1)));
    k_loc_can<<<nb(NL), kT, 0, s>>>(P.loc2glob, d_node_perm, NL, *loc_can);
    int32_t *f = nullptr, *idx = nullptr;
    RET(dev_malloc((void **)&f, 4 * (NL + 1), s));
    RET(dev_malloc((void **)&idx, 4 * (NL + 1), s));
    k_owned_flag<<<nb(NL + 1), kT, 0, s>>>(P.owned, NL, f);
    RET(excl_scan(f, idx, NL + 1, s));
    int32_t no = 0;
    RET(cudaMemcpyAsync(&no, idx + NL, 4, cudaMemcpyDeviceToHost, s));
    RET(cudaStreamSynchronize(s));
    *n_own = no;
    RET(dalloc((void **)own_int, 4 * (size_t)(no + 1)));
    RET(dalloc((void **)own_can, 4 * (size_t)(no + 1)));
    RET(dalloc((void **)own_ft, 4 * (size_t)(no + 1)));
    k_owned_lists<<<nb(NL), kT, 0, s>>>(f, idx, NL, d_loc_int, *loc_can, P.loc2glob, *own_int, *own_can, *own_ft);
    dev_free(f, s);
    dev_free(idx, s);
    return cudaGetLastError();
}

}  // namespace sem
