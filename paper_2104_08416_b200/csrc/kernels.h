// kernels.h -- host launchers of the sm_100a kernels (product path).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "sem_internal.h"

namespace sem {

// Device memory of every call goes through the calling context's sem_allocator hook (sem.h), or
// cudaMallocAsync / cudaFreeAsync without one.  The hook is installed per thread for the
// duration of an API call (api.cu: AllocScope).
cudaError_t dev_malloc_raw(void **p, size_t bytes, cudaStream_t s);
cudaError_t dev_free(void *p, cudaStream_t s);
template <typename T>
inline cudaError_t dev_malloc(T **p, size_t bytes, cudaStream_t s) {
    return dev_malloc_raw(reinterpret_cast<void **>(p), bytes, s);
}

// ----------------------------- reorder.cu ---------------------------------
// Vertex bounding box {xmin, ymin, xmax, ymax} -> out4 (device).
cudaError_t launch_bbox(const double *vxy, int64_t nv, double *out4, cudaStream_t s);
// Orientation fix (det < 0 -> swap v1,v2); bad[0] = min element with det == 0, bad[1] = min
// element with a vertex id outside [0, nv) (both INT_MAX when none).
cudaError_t launch_orient(const double *vxy, const int32_t *tri, int64_t E, int64_t nv, int32_t *tri_or,
                          int32_t *bad, cudaStream_t s);
// K1: generalized-Hilbert key of every element's centroid cell.
cudaError_t launch_hilbert_keys(const double *vxy, const int32_t *tri, int64_t E, double xm0,
                                double xm1, double ws, double hs, int32_t wb, int32_t hb,
                                uint32_t *keys, cudaStream_t s);
cudaError_t launch_random_keys(int64_t E, uint64_t seed, uint64_t *keys, cudaStream_t s);
cudaError_t launch_iota(int32_t *a, int64_t n, cudaStream_t s);
cudaError_t launch_fill_i32(int32_t *a, int64_t n, int32_t v, cudaStream_t s);
// K2: stable radix sort of (key, id) pairs -> perm (CUB onesweep).
cudaError_t sort_pairs_u32(const uint32_t *keys, const int32_t *vals, uint32_t *keys_out,
                           int32_t *vals_out, int64_t n, int end_bit, cudaStream_t s);
cudaError_t sort_pairs_u64(const uint64_t *keys, const int32_t *vals, uint64_t *keys_out,
                           int32_t *vals_out, int64_t n, int end_bit, cudaStream_t s);
// K4: canonical SEM node numbering (reading R13).  Returns n_edges via host ptr.
cudaError_t canonical_nodes(const int32_t *tri_or, int64_t nv, int64_t E, int P,
                            int32_t *mu_can, int64_t *n_edges, int64_t *n_unused,
                            int32_t *first_unused, cudaStream_t s);
// K3: rows of src [E][w] permuted: dst[k] = src[perm[k]].
cudaError_t launch_permute_rows(const int32_t *src, const int32_t *perm, int64_t E, int w,
                                int32_t *dst, cudaStream_t s);
// K5: first-touch renumbering.  node_perm[new] = old;
// mu_out = relabelled mu.  Returns number of labels via host ptr.
// deg != nullptr: PAPER.md:318 step 2 as well (each element's group sorted by
// (degree, old id); reading R12, SEM_NODES_FIRST_TOUCH_DEGREE).
cudaError_t first_touch(const int32_t *mu, int64_t E, int Np, int64_t N, int32_t *node_perm,
                        int32_t *mu_out, int64_t *n_labels, cudaStream_t s, const int32_t *deg = nullptr);

// Node graph (nodes connected iff they share an element): degree [N] and,
// with want_adj, the CSR of ascending distinct neighbours.  Device buffers
// come from the device-memory facade (dev_malloc); release with free_node_graph.  *bad is
// kept for the ABI of this helper but never set (nodes with many neighbours take a slower path).
struct DevGraph {
    int32_t *deg = nullptr;
    int64_t *aptr = nullptr;
    int32_t *adj = nullptr;
    int64_t nadj = 0;
};
cudaError_t build_node_graph(const int32_t *mu, int64_t E, int Np, int64_t N, bool want_adj, DevGraph &g,
                             int *bad, cudaStream_t s);
void free_node_graph(DevGraph &g, cudaStream_t s);
// Conn. (strategy 0, key = degree) / Dist. (strategy 1, key = squared distance
// to (x0, y0)) traversal of reading R20 on the canonical connectivity mu_can
// (input element order): order [N] = visit order (new -> canonical),
// elem_perm [E] = element list (new -> input).  edge_t [P-1]: reference edge
// node positions.  Level-synchronous: parent = smallest frontier position,
// each level sorted by (parent, key rank) = the sequential queue order.
cudaError_t strategy_order(const int32_t *mu_can, const double *vxy, const int32_t *tri_or, int64_t E, int P,
                           int64_t N, int strategy, const DevGraph &g, const double *edge_t, double x0, double y0,
                           int32_t *elem_perm, int32_t *order, int64_t *n_levels, cudaStream_t s);
// *first = smallest i < n with a[i] == v (INT_MAX if none)
cudaError_t launch_find_i32(const int32_t *a, int64_t n, int32_t v, int32_t *first, cudaStream_t s);
// label_of[node_perm[i]] = i, then mu_out = label_of[mu]
cudaError_t relabel_from_perm(const int32_t *mu, int64_t n, const int32_t *node_perm, int64_t N, int32_t *mu_out,
                              cudaStream_t s);

// ------------------------------- step.cu -----------------------------------
struct DevChunks {  // device view of ChunkMeta
    int B, Np;
    int64_t E, N, nchunks, N_int, N_sh, N_tot, n_slots;
    int64_t N_if;              // interface nodes: the last N_if of the shared range
    int max_local, max_win, max_count, max_nsh;
    const int32_t *cmeta;      // [nchunks][8]
    const uint16_t *lidx;      // [nchunks][Np][B] chunk-local node of (p, t)
    const uint16_t *lpos;      // [nchunks][Np*B] entry-buffer (JDS) position of entry p*B + t
    const uint16_t *jds;       // [nchunks][2 kJdsW] jagged-diagonal starts (interior, shared segment)
    const int32_t *sh_pstart;  // [N_sh+1] node-major slots of shared node s
    const int32_t *shl_node;   // per chunk (block at cmeta[2]): shared index of each local shared node
    const int32_t *shl_slot;   // per chunk: the slot it writes
    const uint16_t *shl_cr;    // per chunk: (slots of the node << 8) | rank of this chunk among them
    const int32_t *own0;       // [nchunks+1] shared indices owned by chunk c: [own0[c], own0[c+1])
};

// ------------------------------ chunks_gpu.cu --------------------------------
// The chunk builder of chunks.cpp on the GPU, same arrays bit for bit.  mu: device
// [E][Np]; forced: device [N] flags of rank-interface nodes or nullptr.  Persistent
// arrays come from `dalloc` (owned by the caller); `err` is set (and cudaSuccess
// returned) for mesh errors.  Fills the scalars and lists of m (no host arrays),
// the device view d, the node -> internal id map and the chunk lists.
using DeviceAlloc = std::function<cudaError_t(void **, size_t)>;
cudaError_t build_chunks_gpu(const int32_t *d_mu, int64_t E, int Np, int64_t N, int B, const uint8_t *d_forced,
                             const DeviceAlloc &dalloc, ChunkMeta &m, DevChunks &d, int32_t **d_int_of,
                             int32_t **d_bnd, int32_t **d_intc, std::string &err, cudaStream_t s);

// ----------------------------- partition_gpu.cu ------------------------------
// partition.cpp on the GPU for world >= 2: device loc2glob / mu_local / remote /
// owned (persistent, from dalloc), host neighbour and summation lists.
struct DevPartition {
    int64_t e0 = 0, e1 = 0, NL = 0, n_if = 0;
    int32_t *loc2glob = nullptr, *mu_local = nullptr;
    uint8_t *remote = nullptr, *owned = nullptr;
    std::vector<int32_t> nbr, nbr_off, send_if, sum_start, sum_src;
};
cudaError_t build_partition_gpu(const int32_t *d_mu, int64_t E, int Np, int64_t N, int rank, int world,
                                const DeviceAlloc &dalloc, DevPartition &P, std::string &err, cudaStream_t s);
// loc_can[l] = node_perm[loc2glob[l]]; the owned subset of (loc_int, loc_can, loc2glob)
cudaError_t partition_io_maps(const DevPartition &P, const int32_t *d_node_perm, const int32_t *d_loc_int,
                              const DeviceAlloc &dalloc, int32_t **loc_can, int32_t **own_int, int32_t **own_can,
                              int32_t **own_ft, int64_t *n_own, cudaStream_t s);

cudaError_t upload_ref_tables(const RefTables &T, cudaStream_t s);
// K6: per element (new order) G = c^2 detJ J^-1 J^-T and detJ.
cudaError_t launch_geometry(const double *vxy, const int32_t *tri_or_in, const int32_t *perm,
                            const double *c_in, int64_t E, int64_t Epad, double *Grr,
                            double *Gss, double *Grs, double *detJ, int32_t *bad,
                            cudaStream_t s);
// Lumped mass, assembled with the chunk machinery; writes dt2M = numer / Mbar
// (numer = dt^2 for the leapfrog, h/2 for Heun; 0 in the alignment holes).
// Uses `slot` as scratch.
cudaError_t assemble_mass(const DevChunks &ch, const double *detJ, double numer, double *slot,
                          double *dt2M, cudaStream_t s);

struct StepParams {
    const double *Grr, *Gss, *Grs;
    const double *dt2M;
    const double *U;   // U^n
    double *Uprev;     // U^{n-1} in, U^{n+1} out
    double *slot;      // node-major partial sums of shared nodes (K7 writes, K8 reads)
    int32_t *cnt;      // [N_sh] arrival counters: K7 finalises a shared node when its last
                       // chunk arrives (nullptr: K8 does it)
    int32_t src;       // internal node id of the source (-1 none)
    double amp, f0, t0, dt;
    int64_t n;         // step index of U
    const int64_t *n_dev;  // if set: the step index lives in device memory (CUDA-graph step loop)
    int32_t k8_rev;        // K8 walks the shared nodes from the last block down (the slots K7's
                           // last chunks wrote are the ones still in L2)
};
// persistent K7 grid: resident CTAs per SM x SMs; reserve_sms SMs' worth of CTA slots are left free
// (for the exchange kernels on the comm stream while the interior chunks run)
int k7_grid(const DevChunks &ch, bool fused, int reserve_sms = 0);
// K7's shared memory for these chunks fits one CTA on the current device
bool k7_fits(const DevChunks &ch, bool fused);
// resident K7 CTAs per SM for chunks of B elements with these per-chunk maxima (shared-memory stages)
int k7_ctas_per_sm(int np, int B, int max_local, int max_win, int max_nsh, bool fused, int max_count = 0);
// device step counter of the graph-captured step loop: += 1, = v
// pdl: programmatic dependent launch (the graph-captured step loop, SEM_PDL): the kernel may
// start while its predecessor drains and waits in griddepcontrol.wait before any data access
cudaError_t launch_step_inc(int64_t *n, cudaStream_t s, bool pdl = false);
cudaError_t launch_step_set(int64_t *n, int64_t v, cudaStream_t s);
// overlap probe: `ctas` small CTAs holding their SM slots for `us` microseconds (stand-in for NCCL)
cudaError_t launch_comm_standin(double us, int ctas, cudaStream_t s);
// K7 over all chunks (list == nullptr) or over the chunk ids list[0..nlist).
cudaError_t launch_k7(const DevChunks &ch, const StepParams &p, int grid, cudaStream_t s,
                      const int32_t *list = nullptr, int64_t nlist = 0, bool pdl = false);
cudaError_t launch_k8(const DevChunks &ch, const StepParams &p, cudaStream_t s, bool pdl = false);
// Multi-GPU interface: local partials (+ pack per neighbour), then the
// rank-ordered sum and update (step) or dt^2/M (mass).
cudaError_t launch_if_partial(const DevChunks &ch, const double *slot, double *xbuf, const int32_t *send_if,
                              int64_t n_send, double *sendbuf, cudaStream_t s);
cudaError_t launch_k8_if(const DevChunks &ch, const StepParams &p, const double *xbuf, const int32_t *sum_start,
                         const int32_t *sum_src, cudaStream_t s);
cudaError_t launch_mass_if(const DevChunks &ch, const double *xbuf, const int32_t *sum_start, const int32_t *sum_src,
                           double numer, double *dt2M, cudaStream_t s);
// ------------------------------- heun.cu -----------------------------------
// The paper's Heun predictor-corrector on (U, V) (NEXT-1).
struct HeunParams {
    const double *geo[5];  // per element (new order, padded): F00, F01, F10, F11 (F = c^2 J^-1), sd = detJ/c^2
    const double *hM;      // (h/2) / M-bar per internal node
    double *U;             // U^n in, U^{n+1} out (in place)
    double *W;             // W^{n-1} in (lagged modes), W^n = U^n + (h/2) Udot1 out
    double *V;             // [nchunks][2 Np][B] element velocities (component k*Np + p)
    double *slot;          // double2 per slot: (R(V), K U) partials of shared nodes
    int32_t src;
    double amp, f0, t0, h;
    int64_t n;             // step index of U
};
bool heun_supported(int np, int B);
cudaError_t upload_heun_tables(const RefTables &T, cudaStream_t s);
cudaError_t launch_geometry_heun(const double *vxy, const int32_t *tri_or, const int32_t *perm, const double *c_in,
                                 int64_t E, int64_t Epad, double *const geo[5], double *detJ, int32_t *bad,
                                 cudaStream_t s);
// mode 0: step (V current), 1: step with the lagged V update, 2: V update only
cudaError_t launch_heun(const DevChunks &ch, const HeunParams &p, int mode, cudaStream_t s,
                        const int32_t *list = nullptr, int64_t nlist = 0);
// multi-GPU Heun: interface (R(V), K U) partials of this rank (+ per-neighbour pack, double2), then
// the rank-ordered sums and the U, W update of the interface nodes
cudaError_t launch_heun_if_partial(const DevChunks &ch, const double *slot, double *xbuf, const int32_t *send_if,
                                   int64_t n_send, double *sendbuf, cudaStream_t s);
cudaError_t launch_heun_if(const DevChunks &ch, const HeunParams &p, const double *xbuf, const int32_t *sum_start,
                           const int32_t *sum_src, cudaStream_t s);
cudaError_t launch_heun_fix(const DevChunks &ch, const HeunParams &p, cudaStream_t s);
// V (chunk layout) <-> host layout [E][Np][2] in input element order; in == nullptr -> zeros
cudaError_t launch_v_out(const double *V, const int32_t *perm, int64_t E, int np, int B, double *out, cudaStream_t s);
cudaError_t launch_v_in(const double *in, const int32_t *perm, int64_t E, int np, int B, double *V, cudaStream_t s);

// NEXT-4 ablation scatters: element k in [e0, e1) of mu [.][Np] (internal node
// ids; G read at eidx[k], or k if eidx == nullptr) adds K^e u into KU with fp64
// atomics (atomic) or plain read-modify-write (one colour of a global colouring).
cudaError_t launch_abl_elem(int np, bool atomic, const int32_t *mu, const int32_t *eidx, int64_t e0, int64_t e1,
                            const StepParams &p, double *KU, cudaStream_t s);
// U^{n+1} = 2U^n - U^{n-1} + dt2M (f - KU) over n internal nodes, KU := 0.
cudaError_t launch_abl_update(int64_t n, const StepParams &p, double *KU, cudaStream_t s);

// out[omap ? omap[i] : i] = in[imap ? imap[i] : i], i < n
cudaError_t launch_permute_f64(const double *in, const int32_t *imap, const int32_t *omap, int64_t n,
                               double *out, cudaStream_t s);
cudaError_t launch_nonfinite(const double *a, int64_t n, int32_t *flag, cudaStream_t s);
// *first = min(*first, smallest i < n with !(a[i] > 0) or a[i] not finite)
cudaError_t launch_check_positive(const double *a, int64_t n, int32_t *first, cudaStream_t s);

}  // namespace sem
