// api.cu -- the C ABI of libsem.so (include/sem.h).  Orchestrates the kernels
// of reorder.cu / step.cu, the multi-GPU interface exchange (NCCL, loaded with
// dlopen, or an in-process loopback for one-GPU testing), and owns all device
// memory of a context.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "kernels.h"
#include "sem.h"
#include "sem_internal.h"

using namespace sem;

namespace {
int g_const_P = 0;  // degree whose tables currently sit in __constant__ memory

// Elements per chunk (one CTA iteration of K7): 512 at P3 (one CTA of 17 warps per SM; half the
// shared nodes of 256: C4 step 0.3862 -> 0.3792 ms, C3 0.1926 -> 0.1906 ms), 256 at P2 (C5/4 0.445
// at 256 against 0.569 ms at 512), 128 for Heun; SEM_CHUNK=128|192|256|512 selects the other
// compiled variants (design experiments, chunk size).  A mesh whose largest
// chunks of 512 would not fit one CTA's shared memory is rebuilt with 256 (sem_mesh_reorder).
int chunk_elems(int P, bool heun) {
    const char *v = getenv("SEM_CHUNK");
    if (heun && (P == 5 || P == 7)) {  // Heun's wide kernel: SEM_CHUNK=32|64|128 (A/B)
        const int b = v ? atoi(v) : (P == 5 ? 128 : 64);
        return (b == 32 || b == 64 || (P == 5 && b == 128)) ? b : (P == 5 ? 128 : 64);
    }
    if (P == 4 || P == 5) return 128;  // shared-memory budget of the stage at 15 / 21 nodes per element
    if (P == 6 || P == 7) return 64;   // ... and at 28 / 36
    // Heun (integrator selected before sem_mesh_reorder): 128 runs 2 CTAs per SM
    const int b = v ? atoi(v) : (heun ? 128 : P == 3 ? 512 : 256);
    return (b == 128 || b == 192 || b == 512) ? b : 256;
}

// ---- NCCL through dlopen (no link-time dependency; torch's copy is reused) ----
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

// Which libnccl.so.2 is loaded matters beyond this library: the dynamic linker
// matches a later DT_NEEDED "libnccl.so.2" (libtorch_cuda's) by soname against the
// objects already mapped, whatever RTLD_LOCAL/GLOBAL said.  Loading the system copy
// (2.27) before torch therefore breaks `import torch` (it needs the 2.28 of its
// wheel).  Resolution order, none of which can shadow torch's copy:
//   1. a libnccl.so.2 already mapped in the process (RTLD_NOLOAD): torch's, if imported;
//   2. SEM_NCCL_LIB, an absolute path -- the binding (sem.py) sets it to the nvidia-nccl
//      wheel's library, the file torch itself loads;
//   3. only then the default search path (plain C callers without torch).
NcclApi &nccl() {
    static NcclApi api;
    static std::mutex mu;
    static bool tried = false;
    std::lock_guard<std::mutex> lock(mu);
    if (tried) return api;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char *env = getenv("SEM_NCCL_LIB");
    if (!h && env && *env) {
        h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            api.err = std::string("cannot load SEM_NCCL_LIB=") + env + ": " + dlerror();
            return api;
        }
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return api;
    }
#define SYM(field, name)                                                  \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));    \
    if (!api.field) { api.err = std::string("missing NCCL symbol ") + name; return api; }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = true;
    return api;
}
}  // namespace

// ---- device memory: the context's sem_allocator hook, or the stream-ordered pool ----
namespace {
thread_local const sem_allocator *t_alloc = nullptr;  // the hook of the API call running on this thread
}
cudaError_t sem::dev_malloc_raw(void **p, size_t bytes, cudaStream_t s) {
    if (!t_alloc) return cudaMallocAsync(p, bytes, s);
    *p = t_alloc->alloc(bytes, (void *)s, t_alloc->user);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
}
cudaError_t sem::dev_free(void *p, cudaStream_t s) {
    if (!p) return cudaSuccess;
    if (!t_alloc) return cudaFreeAsync(p, s);
    t_alloc->free(p, (void *)s, t_alloc->user);
    return cudaSuccess;
}

// Device arrays that live as long as a mesh or its operators: stream-ordered pool
// allocations on the context's stream (the pool keeps freed memory mapped, so a
// later sem_mesh_reorder does not pay cudaMalloc's page mapping again).
struct AllocList {
    cudaStream_t s = nullptr;
    std::vector<void *> p;
    size_t size() const { return p.size(); }
    void push_back(void *q) { p.push_back(q); }
    void release_from(size_t n) {  // free the entries [n, size)
        for (size_t i = n; i < p.size(); i++) dev_free(p[i], s);
        p.resize(n);
    }
};

struct sem_ctx {
    int device = 0, rank = 0, world = 1;
    sem_allocator alloc{};     // device-memory hook (sem.h); has_alloc = false: cudaMallocAsync
    bool has_alloc = false;
    bool loopback = false;  // world > 1 without NCCL: only the sem_group_* calls may step it
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    bool dead = false;

    // mesh
    bool have_mesh = false, have_ops = false;
    int P = 0, Np = 0;
    int64_t nv = 0, E = 0, N = 0;  // E, N: this rank's elements / nodes
    int64_t E_glob = 0, N_glob = 0, e0 = 0;
    int32_t grid[2] = {0, 0};
    RefTables T;
    AllocList mesh_allocs, ops_allocs;
    double *d_vxy = nullptr;
    int32_t *d_tri_or = nullptr;  // oriented triangles, INPUT order
    int32_t *d_perm = nullptr;    // new -> input (global order)
    // local node l: internal id, canonical id, reordered (first-touch) id; "own" = I/O owner subset
    int32_t *d_loc_int = nullptr, *d_loc_can = nullptr, *d_loc_ft = nullptr;
    int32_t *d_own_int = nullptr, *d_own_can = nullptr, *d_own_ft = nullptr;
    int64_t n_own = 0;
    std::vector<int32_t> src_lookup;  // local node -> canonical id (source lookup)
    std::vector<int32_t> src_int_of;  // local node -> internal id
    DevChunks dch{};
    ChunkMeta meta_info;  // counts only
    int k7_grid = 0;
    int k7_grid_ovl = 0;  // interior chunks while an interface exchange is in flight (SEM_COMM_SMS)
    // one-GPU overlap probe (SEM_OVERLAP_PROBE_US): one rank, a chunk list split like the
    // boundary / interior lists, a stand-in comm kernel between them
    int32_t *d_probe_list = nullptr;
    cudaEvent_t pev[4] = {nullptr, nullptr, nullptr, nullptr};
    double probe_acc[4] = {0, 0, 0, 0};
    int64_t probe_n = 0;
    // interface exchange
    int64_t n_if = 0, n_send = 0;
    std::vector<int32_t> nbr, nbr_off;
    int32_t *d_send_if = nullptr, *d_sum_start = nullptr, *d_sum_src = nullptr;
    double *d_xbuf = nullptr, *d_sendbuf = nullptr;  // xbuf = [own partials | received]

    // operators / state
    double *d_Grr = nullptr, *d_Gss = nullptr, *d_Grs = nullptr, *d_dt2M = nullptr;
    double *d_U[2] = {nullptr, nullptr};
    double *d_slot = nullptr;
    int32_t *d_cnt = nullptr;  // shared-node arrival counters (K8 fused into K7, SEM_FUSE_K8=1)
    cudaGraphExec_t graph_exec[6][2] = {};  // captured step loops of 32, 16, .., 1 steps per U parity
    // kernel timing inside the graph: the same step loop with event-record nodes around K7 and
    // K8 of every step (gev[3 j .. 3 j + 2] = before K7, after K7, after K8 of step j)
    cudaGraphExec_t graph_exec_t[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> gev;
    int64_t *d_nstep = nullptr;                          // its device step counter
    bool fuse_k8 = false;      // measured slower: off by default
    int cur = 0;
    // Heun (NEXT-1): U = d_U[0], hM = (h/2)/M-bar in d_dt2M, double2 slots in d_slot
    int integrator = SEM_INTEGRATOR_LEAPFROG;
    int ops_integrator = SEM_INTEGRATOR_LEAPFROG;  // integrator the built operators belong to
    double *d_geo[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    double *d_W = nullptr, *d_V = nullptr;
    bool v_lag = false;  // V holds V^{n-1}; V^n = V + h Vdot(W)
    // NEXT-4 ablation scatters (world 1, leapfrog): selected before sem_mesh_reorder
    int scatter = SEM_SCATTER_CHUNK;       // requested
    int mesh_scatter = SEM_SCATTER_CHUNK;  // what the current mesh was prepared for
    int32_t *d_mu_abl = nullptr, *d_eidx_abl = nullptr;  // internal-id rows (colour order for COLOR)
    std::vector<int64_t> color_off;                      // COLOR: element ranges per colour
    double *d_KU = nullptr;
    int32_t src_int = -1;
    double amp = 0, f0 = 1, t0 = 0, dt = 0;
    int64_t step = 0;
    cudaEvent_t xev = nullptr;  // loopback: phase-1 done on this rank
    cudaStream_t comm_stream = nullptr;           // NCCL exchange, overlapped with interior chunks
    cudaStream_t io_stream = nullptr;             // sem_mesh_reorder's output copies, overlapped with the chunk builder
    cudaEvent_t io_ev = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_exchanged = nullptr;
    int32_t *d_bnd = nullptr, *d_intc = nullptr;  // boundary / interior chunk lists
    int64_t n_bnd = 0, n_intc = 0;

    // timing
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev7, ev8, pool;
    double t7 = 0, t8 = 0;
    int64_t n7 = 0, n8 = 0;
    double prep_reorder_ms = 0, prep_build_ms = 0;
    int64_t strategy_levels = 0;  // BFS levels of the last Conn./Dist. ordering
};

namespace {

sem_status fail(sem_ctx *c, sem_status s, const std::string &msg) {
    c->err = msg;
    return s;
}

sem_status cuda_fail(sem_ctx *c, cudaError_t e, const char *where) {
    c->dead = true;
    c->err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return SEM_E_CUDA;
}

// Installs a context's device-memory hook on this thread for the duration of an API call.
struct AllocScope {
    const sem_allocator *prev;
    explicit AllocScope(const sem_ctx *c) : prev(t_alloc) { t_alloc = (c && c->has_alloc) ? &c->alloc : nullptr; }
    ~AllocScope() { t_alloc = prev; }
};

#define CK(call)                                                        \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call);        \
    } while (0)

#define ST(call)                        \
    do {                                \
        sem_status _s = (call);         \
        if (_s != SEM_OK) return _s;    \
    } while (0)

// Temporaries of one call: stream-ordered pool allocations, freed in stream
// order when the call returns (no device-wide synchronisation of cudaFree).
struct TmpList {
    cudaStream_t s;
    std::vector<void *> p;
    ~TmpList() {
        for (void *q : p) dev_free(q, s);
    }
};

template <typename T>
cudaError_t dalloc(TmpList &t, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = dev_malloc(&q, sizeof(T) * (count ? count : 1), t.s);
    if (e != cudaSuccess) return e;
    t.p.push_back(q);
    *p = (T *)q;
    return cudaSuccess;
}

template <typename T>
cudaError_t dalloc(AllocList &list, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = dev_malloc(&q, sizeof(T) * (count ? count : 1), list.s);
    if (e != cudaSuccess) return e;
    list.push_back(q);
    *p = (T *)q;
    return cudaSuccess;
}

void free_list(AllocList &l) {
    if (l.size()) cudaDeviceSynchronize();  // as cudaFree did: no stream (main or comm) still uses them
    l.release_from(0);
}

void destroy_graphs(sem_ctx *ctx);

void reset_ops(sem_ctx *ctx) {
    destroy_graphs(ctx);
    ctx->d_nstep = nullptr;
    free_list(ctx->ops_allocs);
    ctx->d_Grr = ctx->d_Gss = ctx->d_Grs = ctx->d_dt2M = nullptr;
    ctx->d_U[0] = ctx->d_U[1] = nullptr;
    ctx->d_slot = nullptr;
    ctx->d_cnt = nullptr;
    for (auto &g : ctx->d_geo) g = nullptr;
    ctx->d_W = ctx->d_V = nullptr;
    ctx->v_lag = false;
    ctx->d_KU = nullptr;
    ctx->have_ops = false;
    ctx->step = 0;
    ctx->cur = 0;
}

void reset_mesh(sem_ctx *ctx) {
    reset_ops(ctx);
    free_list(ctx->mesh_allocs);
    ctx->have_mesh = false;
    ctx->src_lookup.clear();
    ctx->src_int_of.clear();
    ctx->dch = DevChunks{};
    ctx->d_probe_list = nullptr;
    ctx->d_mu_abl = ctx->d_eidx_abl = nullptr;
    ctx->color_off.clear();
    ctx->mesh_scatter = SEM_SCATTER_CHUNK;
    ctx->n_if = ctx->n_send = 0;
    ctx->nbr.clear();
    ctx->nbr_off.clear();
}

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

struct PhaseTrace {  // SEM_TRACE=1: wall time of each preparation phase on stderr
    bool on = getenv("SEM_TRACE") != nullptr;
    double t = now_ms();
    void mark(cudaStream_t s, const char *what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const double n = now_ms();
        fprintf(stderr, "[sem mesh_reorder] %-30s %8.1f ms\n", what, n - t);
        t = n;
    }
};

template <typename T>
cudaError_t upload(AllocList &list, T **dst, const std::vector<T> &src, cudaStream_t s) {
    cudaError_t e = dalloc(list, dst, src.size());
    if (e != cudaSuccess) return e;
    if (src.empty()) return cudaSuccess;
    return cudaMemcpyAsync(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, s);
}

// NEXT-4 ablation scatters: rows of mu in internal ids; COLOR: greedy global
// element colouring in element order (smallest colour absent from every node's
// elements), elements grouped by colour, ascending within a colour.
sem_status prepare_ablation(sem_ctx *ctx, const std::vector<int32_t> &mu_h, int64_t E, int Np, int64_t N,
                            int degree, bool one, const ChunkMeta &m, cudaStream_t s) {
    if (!one) return fail(ctx, SEM_E_UNSUPPORTED, "ablation scatters run with world_size 1");
    if (degree > 3) return fail(ctx, SEM_E_UNSUPPORTED, "ablation scatters are built for P = 2, 3");
    std::vector<int32_t> rows((size_t)E * Np), eidx, color;
    int ncol = 1;
    if (ctx->scatter == SEM_SCATTER_COLOR) {
        std::vector<uint64_t> used((size_t)N, 0);
        color.assign((size_t)E, 0);
        for (int64_t e = 0; e < E; e++) {
            uint64_t mask = 0;
            for (int p = 0; p < Np; p++) mask |= used[mu_h[e * Np + p]];
            if (~mask == 0) return fail(ctx, SEM_E_MESH, "global colouring needs more than 64 colours");
            const int c = __builtin_ctzll(~mask);
            color[e] = c;
            if (c + 1 > ncol) ncol = c + 1;
            for (int p = 0; p < Np; p++) used[mu_h[e * Np + p]] |= (uint64_t)1 << c;
        }
    }
    ctx->color_off.assign((size_t)ncol + 1, 0);
    if (ctx->scatter == SEM_SCATTER_COLOR) {
        for (int64_t e = 0; e < E; e++) ctx->color_off[color[e] + 1]++;
        for (int c = 0; c < ncol; c++) ctx->color_off[c + 1] += ctx->color_off[c];
        std::vector<int64_t> fillc(ctx->color_off.begin(), ctx->color_off.end() - 1);
        eidx.resize((size_t)E);
        for (int64_t e = 0; e < E; e++) eidx[fillc[color[e]]++] = (int32_t)e;
    } else {
        ctx->color_off[1] = E;
    }
    for (int64_t k = 0; k < E; k++) {
        const int64_t e = eidx.empty() ? k : eidx[k];
        for (int p = 0; p < Np; p++) rows[k * Np + p] = m.int_of[mu_h[e * Np + p]];
    }
    CK(upload(ctx->mesh_allocs, &ctx->d_mu_abl, rows, s));
    if (!eidx.empty()) CK(upload(ctx->mesh_allocs, &ctx->d_eidx_abl, eidx, s));
    ctx->mesh_scatter = ctx->scatter;
    return SEM_OK;
}

// Host-built chunk metadata (chunks.cpp) -> device arrays and the device view.
cudaError_t upload_chunks(AllocList &L, const ChunkMeta &m, DevChunks &d, cudaStream_t s) {
    d.B = m.B; d.Np = m.Np; d.E = m.E; d.N = m.N; d.nchunks = m.nchunks;
    d.N_int = m.N_int; d.N_sh = m.N_sh; d.N_tot = m.N_tot; d.n_slots = m.n_slots; d.N_if = m.N_if;
    d.max_local = m.max_local; d.max_win = m.max_win; d.max_count = m.max_count; d.max_nsh = m.max_nsh;
    int32_t *p_cmeta, *p_pstart, *p_shn, *p_shs, *p_own0;
    uint16_t *p_lpos, *p_jds, *p_lidx, *p_shcr;
    cudaError_t e;
    if ((e = upload(L, &p_cmeta, m.cmeta, s)) || (e = upload(L, &p_lidx, m.lidx, s)) ||
        (e = upload(L, &p_lpos, m.lpos, s)) || (e = upload(L, &p_jds, m.jds, s)) ||
        (e = upload(L, &p_pstart, m.sh_pstart, s)) || (e = upload(L, &p_shn, m.shl_node, s)) ||
        (e = upload(L, &p_shs, m.shl_slot, s)) || (e = upload(L, &p_shcr, m.shl_cr, s)) ||
        (e = upload(L, &p_own0, m.own0, s)))
        return e;
    d.cmeta = p_cmeta; d.lidx = p_lidx; d.lpos = p_lpos; d.jds = p_jds; d.sh_pstart = p_pstart;
    d.shl_node = p_shn; d.shl_slot = p_shs; d.shl_cr = p_shcr; d.own0 = p_own0;
    return cudaSuccess;
}

// SEM_CHUNK_CHECK=1: the GPU chunk builder's arrays against the host builder's.
template <typename T>
bool same_dev(const std::vector<T> &h, const T *dptr, size_t n, cudaStream_t s) {
    if (h.size() < n) return false;
    std::vector<T> g(n);
    if (n && cudaMemcpyAsync(g.data(), dptr, sizeof(T) * n, cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
    cudaStreamSynchronize(s);
    return n == 0 || std::memcmp(g.data(), h.data(), sizeof(T) * n) == 0;
}

std::string compare_chunks(const ChunkMeta &h, const ChunkMeta &m, const DevChunks &d, const int32_t *d_int_of,
                           cudaStream_t s) {
    if (h.nchunks != m.nchunks || h.N_int != m.N_int || h.N_sh != m.N_sh || h.N_if != m.N_if ||
        h.n_slots != m.n_slots || h.max_local != m.max_local || h.max_win != m.max_win ||
        h.max_count != m.max_count || h.max_nsh != m.max_nsh)
        return "scalars";
    if (h.bnd_chunks != m.bnd_chunks || h.int_chunks != m.int_chunks) return "chunk lists";
    if (!same_dev(h.cmeta, d.cmeta, h.cmeta.size(), s)) return "cmeta";
    if (!same_dev(h.lidx, d.lidx, h.lidx.size(), s)) return "lidx";
    if (!same_dev(h.lpos, d.lpos, h.lpos.size(), s)) return "lpos";
    if (!same_dev(h.jds, d.jds, h.jds.size(), s)) return "jds";
    if (!same_dev(h.sh_pstart, d.sh_pstart, h.sh_pstart.size(), s)) return "sh_pstart";
    if (!same_dev(h.shl_node, d.shl_node, h.shl_node.size(), s)) return "shl_node";
    if (!same_dev(h.shl_slot, d.shl_slot, h.shl_slot.size(), s)) return "shl_slot";
    if (!same_dev(h.shl_cr, d.shl_cr, h.shl_cr.size(), s)) return "shl_cr";
    if (!same_dev(h.own0, d.own0, h.own0.size(), s)) return "own0";
    if (!same_dev(h.int_of, d_int_of, h.int_of.size(), s)) return "int_of";
    return "";
}

sem_status ensure_tables(sem_ctx *ctx) {
    if (g_const_P != ctx->P) {
        CK(upload_ref_tables(ctx->T, ctx->stream));
        CK(upload_heun_tables(ctx->T, ctx->stream));
        g_const_P = ctx->P;
    }
    return SEM_OK;
}

sem_status record(sem_ctx *ctx, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &list, bool start) {
    if (start) {
        std::pair<cudaEvent_t, cudaEvent_t> ev;
        if (!ctx->pool.empty()) { ev = ctx->pool.back(); ctx->pool.pop_back(); }
        else {
            CK(cudaEventCreate(&ev.first));
            CK(cudaEventCreate(&ev.second));
        }
        list.push_back(ev);
        CK(cudaEventRecord(ev.first, ctx->stream));
    } else {
        CK(cudaEventRecord(list.back().second, ctx->stream));
    }
    return SEM_OK;
}

sem_status drain_events(sem_ctx *ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto *lst : {&ctx->ev7, &ctx->ev8}) {
        for (auto &ev : *lst) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ev.first, ev.second));
            if (lst == &ctx->ev7) { ctx->t7 += ms; ctx->n7++; }
            else { ctx->t8 += ms; ctx->n8++; }
            ctx->pool.push_back(ev);
        }
        lst->clear();
    }
    return SEM_OK;
}

sem_status check_usable(sem_ctx *ctx) {
    if (!ctx) return SEM_E_ARG;
    if (ctx->dead) return fail(ctx, SEM_E_CUDA, "context unusable after a CUDA error: " + ctx->err);
    return SEM_OK;
}

// ---- interface exchange ------------------------------------------------------------
// NCCL: grouped send/recv of the packed partials with every neighbour rank.
// w = fp64 values per interface node (1: K U or the mass; 2: Heun's (R(V), K U)).
sem_status exchange_nccl(sem_ctx *ctx, cudaStream_t st, int w = 1) {
    if (ctx->nbr.empty()) return SEM_OK;
    NcclApi &N = nccl();
    ncclResult_t r = N.GroupStart();
    for (size_t k = 0; r == ncclSuccess && k < ctx->nbr.size(); k++) {
        const size_t off = ctx->nbr_off[k], cnt = ctx->nbr_off[k + 1] - off;
        r = N.Send(ctx->d_sendbuf + w * off, w * cnt, ncclFloat64, ctx->nbr[k], ctx->comm, st);
        if (r == ncclSuccess)
            r = N.Recv(ctx->d_xbuf + w * (ctx->n_if + off), w * cnt, ncclFloat64, ctx->nbr[k], ctx->comm, st);
    }
    ncclResult_t r2 = N.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(ctx, SEM_E_NCCL, std::string("NCCL exchange failed: ") +
                                         N.GetErrorString(r != ncclSuccess ? r : r2));
    return SEM_OK;
}

// Loopback: contexts of one process; rank r copies what rank q packed for it.
sem_status exchange_loopback(sem_ctx **ctxs, int n, int w = 1) {
    for (int r = 0; r < n; r++) {
        sem_ctx *ctx = ctxs[r];
        CK(cudaSetDevice(ctx->device));
        CK(cudaEventRecord(ctx->xev, ctx->stream));
    }
    for (int r = 0; r < n; r++) {
        sem_ctx *ctx = ctxs[r];
        CK(cudaSetDevice(ctx->device));
        for (size_t k = 0; k < ctx->nbr.size(); k++) {
            const int q = ctx->nbr[k];
            sem_ctx *src = nullptr;
            for (int j = 0; j < n; j++)
                if (ctxs[j]->rank == q) src = ctxs[j];
            if (!src) return fail(ctx, SEM_E_ARG, "loopback group lacks rank " + std::to_string(q));
            size_t kq = 0;
            while (kq < src->nbr.size() && src->nbr[kq] != ctx->rank) kq++;
            if (kq == src->nbr.size()) return fail(ctx, SEM_E_MESH, "asymmetric neighbour lists");
            const size_t cnt = ctx->nbr_off[k + 1] - ctx->nbr_off[k];
            if ((size_t)(src->nbr_off[kq + 1] - src->nbr_off[kq]) != cnt)
                return fail(ctx, SEM_E_MESH, "interface sizes differ between ranks");
            CK(cudaStreamWaitEvent(ctx->stream, src->xev, 0));
            CK(cudaMemcpyAsync(ctx->d_xbuf + w * (ctx->n_if + ctx->nbr_off[k]), src->d_sendbuf + w * src->nbr_off[kq],
                               w * cnt * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        }
    }
    // a rank's send buffer must not be overwritten before its neighbours copied it
    for (int r = 0; r < n; r++) {
        sem_ctx *ctx = ctxs[r];
        CK(cudaSetDevice(ctx->device));
        CK(cudaEventRecord(ctx->xev, ctx->stream));
    }
    for (int r = 0; r < n; r++) {
        sem_ctx *ctx = ctxs[r];
        CK(cudaSetDevice(ctx->device));
        for (size_t k = 0; k < ctx->nbr.size(); k++)
            for (int j = 0; j < n; j++)
                if (ctxs[j]->rank == ctx->nbr[k]) CK(cudaStreamWaitEvent(ctx->stream, ctxs[j]->xev, 0));
    }
    return SEM_OK;
}

// K8 takes the shared nodes in descending order, starting with the slots K7's last chunks wrote
// (still in L2): C4 K8 0.0275 -> 0.0270 ms, C3 step 0.1861 -> 0.1854 ms with two nodes per
// thread (profiles/r2s4_k8_ab.md); SEM_K8_REV=0 takes them ascending (A/B)
bool k8_rev() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("SEM_K8_REV"); v = e && e[0] == '0' ? 0 : 1; }
    return v == 1;
}

StepParams step_params(sem_ctx *ctx) {
    StepParams p;
    p.Grr = ctx->d_Grr; p.Gss = ctx->d_Gss; p.Grs = ctx->d_Grs; p.dt2M = ctx->d_dt2M;
    p.slot = ctx->d_slot;
    p.cnt = ctx->d_cnt;
    p.src = ctx->src_int; p.amp = ctx->amp; p.f0 = ctx->f0; p.t0 = ctx->t0; p.dt = ctx->dt;
    p.U = ctx->d_U[ctx->cur];
    p.Uprev = ctx->d_U[1 - ctx->cur];
    p.n = ctx->step;
    p.n_dev = nullptr;
    p.k8_rev = k8_rev() ? 1 : 0;
    return p;
}

// ---- CUDA-graph step loop (one rank, leapfrog, chunk scatter) --------------------------
// kGraphSteps consecutive steps (K7, K8, counter += 1 each; an even count, so the
// U / U^{n-1} ping-pong returns to the same parity) are captured once per parity
// and replayed; the step index comes from a device counter.  Removes the
// per-launch host overhead that dominates small meshes.  The remainder of a call
// (n mod 32 steps) replays the graphs of 16, 8, 4, 2 and 1 steps (an odd one flips
// the parity); sem_step_n(0) captures all twelve.  Kernel timing mode: 32-step graphs
// with event nodes, the remainder launched step by step.  SEM_GRAPH=0 disables.
constexpr int kGraphSteps = 32;
constexpr int kNGraph = 6;  // graph sizes kGraphSteps >> si

// SEM_COMM_SMS: SMs left to the exchange kernels (NCCL send/recv on the comm stream) while the
// interior chunks run; SEM_OVERLAP_PROBE_US: one-rank overlap probe (stand-in comm kernel)
int comm_sms() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("SEM_COMM_SMS"); v = e ? atoi(e) : 2; if (v < 0) v = 0; }
    return v;
}
double probe_us() {
    static double v = -1;
    if (v < 0) { const char *e = getenv("SEM_OVERLAP_PROBE_US"); v = e ? atof(e) : 0.0; if (!(v > 0)) v = 0.0; }
    return v;
}

bool graph_ok(sem_ctx *ctx) {
    static const bool env_off = getenv("SEM_GRAPH") && atoi(getenv("SEM_GRAPH")) == 0;
    return !env_off && ctx->world == 1 && ctx->stream != nullptr && !(probe_us() > 0) &&
           ctx->ops_integrator == SEM_INTEGRATOR_LEAPFROG && ctx->mesh_scatter == SEM_SCATTER_CHUNK &&
           ctx->d_cnt == nullptr;
}

void destroy_graphs(sem_ctx *ctx) {
    for (int si = 0; si < kNGraph; si++)
        for (int i = 0; i < 2; i++)
            if (ctx->graph_exec[si][i]) { cudaGraphExecDestroy(ctx->graph_exec[si][i]); ctx->graph_exec[si][i] = nullptr; }
    for (int i = 0; i < 2; i++)
        if (ctx->graph_exec_t[i]) { cudaGraphExecDestroy(ctx->graph_exec_t[i]); ctx->graph_exec_t[i] = nullptr; }
}

// the step loop graph of kGraphSteps >> si steps starting at U parity par (timing mode: si = 0
// with the event nodes), captured on first use
sem_status graph_steps(sem_ctx *ctx, int64_t reps, int si = 0, int par = -1) {
    CK(cudaSetDevice(ctx->device));
    ST(ensure_tables(ctx));
    cudaStream_t s = ctx->stream;
    const bool timed = ctx->timing;
    if (timed) si = 0;
    if (par < 0) par = ctx->cur;
    const int nsteps = kGraphSteps >> si;
    cudaGraphExec_t &ex = timed ? ctx->graph_exec_t[par] : ctx->graph_exec[si][par];
    if (timed && ctx->gev.empty()) {
        ctx->gev.resize(3 * kGraphSteps);
        for (auto &e : ctx->gev) CK(cudaEventCreate(&e));
    }
    if (!ex) {
        if (!ctx->d_nstep) CK(dalloc(ctx->ops_allocs, &ctx->d_nstep, 1));
        // one ordinary step's worth of attribute setting happens outside the capture
        (void)k7_grid(ctx->dch, false);
        cudaGraph_t g = nullptr;
        const char *pv = getenv("SEM_PDL");
        // programmatic dependent launch between the steps' kernels: opt-in (SEM_PDL=1), measured
        // 4 % slower on C4
        const bool pdl = pv && pv[0] == '1';
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = cudaSuccess;
        for (int k = 0; k < nsteps && e == cudaSuccess; k++) {
            StepParams p = step_params(ctx);
            p.U = ctx->d_U[(par + k) & 1];
            p.Uprev = ctx->d_U[1 - ((par + k) & 1)];
            p.n_dev = ctx->d_nstep;
            if (timed) e = cudaEventRecordWithFlags(ctx->gev[3 * k], s, cudaEventRecordExternal);
            if (e == cudaSuccess) e = launch_k7(ctx->dch, p, ctx->k7_grid, s, nullptr, 0, pdl);
            if (e == cudaSuccess && timed) e = cudaEventRecordWithFlags(ctx->gev[3 * k + 1], s, cudaEventRecordExternal);
            if (e == cudaSuccess) e = launch_k8(ctx->dch, p, s, pdl);
            if (e == cudaSuccess && timed) e = cudaEventRecordWithFlags(ctx->gev[3 * k + 2], s, cudaEventRecordExternal);
            if (e == cudaSuccess) e = launch_step_inc(ctx->d_nstep, s, pdl);
        }
        cudaError_t e2 = cudaStreamEndCapture(s, &g);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "graph capture");
        if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
    }
    if (reps == 0) return SEM_OK;
    if (par != ctx->cur) return fail(ctx, SEM_E_STATE, "graph replay at the other U parity");
    CK(launch_step_set(ctx->d_nstep, ctx->step, s));
    for (int64_t r = 0; r < reps; r++) {
        CK(cudaGraphLaunch(ex, s));
        if (timed) {  // read this replay's per-step kernel times before the next replay re-records them
            ST(drain_events(ctx));
            const bool k8 = ctx->dch.N_sh - ctx->dch.N_if > 0;
            for (int j = 0; j < kGraphSteps; j++) {
                float a = 0, b = 0;
                CK(cudaEventElapsedTime(&a, ctx->gev[3 * j], ctx->gev[3 * j + 1]));
                CK(cudaEventElapsedTime(&b, ctx->gev[3 * j + 1], ctx->gev[3 * j + 2]));
                ctx->t7 += a;
                ctx->n7++;
                if (k8) { ctx->t8 += b; ctx->n8++; }
            }
        }
    }
    ctx->step += reps * nsteps;
    if (nsteps & 1) ctx->cur ^= (int)(reps & 1);
    return SEM_OK;
}

// Step phase 1: stiffness + update of everything local; pack interface partials.
// With NCCL (use_nccl) the exchange is issued on the comm stream right after
// the boundary chunks are done and overlaps the interior chunks.
// One rank, probe mode: chunks [0, n/8) stand in for the boundary chunks, the rest for the
// interior ones; between them a stand-in comm kernel runs on the comm stream exactly where the
// NCCL exchange would.  Events: before the "boundary" K7, around the "interior" K7, and at the
// end of the stand-in (both streams, one device): the time the main stream waits for it is
// the exposed exchange time.
sem_status step_phase1_probe(sem_ctx *ctx) {
    const DevChunks &d = ctx->dch;
    if (!ctx->d_probe_list) {
        CK(dalloc(ctx->mesh_allocs, &ctx->d_probe_list, d.nchunks));
        CK(launch_iota(ctx->d_probe_list, d.nchunks, ctx->stream));
        if (!ctx->comm_stream) CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        for (auto &e : ctx->pev) CK(cudaEventCreate(&e));
    }
    const StepParams p = step_params(ctx);
    const int64_t nb = d.nchunks / 8;
    CK(cudaEventRecord(ctx->pev[0], ctx->stream));
    CK(launch_k7(d, p, ctx->k7_grid, ctx->stream, ctx->d_probe_list, nb));
    CK(cudaEventRecord(ctx->ev_packed, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
    CK(launch_comm_standin(probe_us(), 4, ctx->comm_stream));
    CK(cudaEventRecord(ctx->pev[3], ctx->comm_stream));
    CK(cudaEventRecord(ctx->pev[1], ctx->stream));
    CK(launch_k7(d, p, ctx->k7_grid_ovl, ctx->stream, ctx->d_probe_list + nb, d.nchunks - nb));
    CK(launch_k8(d, p, ctx->stream));
    CK(cudaEventRecord(ctx->pev[2], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->pev[3], 0));
    CK(cudaStreamSynchronize(ctx->stream));
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, ctx->pev[0], ctx->pev[1]));  // boundary part
    CK(cudaEventElapsedTime(&b, ctx->pev[1], ctx->pev[2]));  // interior part + K8
    CK(cudaEventElapsedTime(&c, ctx->pev[1], ctx->pev[3]));  // stand-in done, from the interior start
    ctx->probe_acc[0] += a;
    ctx->probe_acc[1] += b;
    ctx->probe_acc[2] += c;
    ctx->probe_acc[3] += c > b ? c - b : 0.0;  // exposed: the main stream waits for the exchange
    if (++ctx->probe_n % 200 == 0)
        fprintf(stderr, "[overlap probe] comm SMs reserved %d, stand-in %.1f us on 4 CTAs: boundary K7 %.4f ms, "
                        "interior K7+K8 %.4f ms, stand-in done %.4f ms after the interior start, exposed %.4f ms "
                        "(averages over %lld steps)\n",
                comm_sms(), probe_us(), ctx->probe_acc[0] / ctx->probe_n, ctx->probe_acc[1] / ctx->probe_n,
                ctx->probe_acc[2] / ctx->probe_n, ctx->probe_acc[3] / ctx->probe_n, (long long)ctx->probe_n);
    return SEM_OK;
}

sem_status step_phase1(sem_ctx *ctx, bool use_nccl) {
    CK(cudaSetDevice(ctx->device));
    ST(ensure_tables(ctx));
    if (ctx->world == 1 && probe_us() > 0 && ctx->dch.nchunks >= 16 && !ctx->timing) return step_phase1_probe(ctx);
    const StepParams p = step_params(ctx);
    if (ctx->timing) ST(record(ctx, ctx->ev7, true));
    if (ctx->n_if == 0) {
        CK(launch_k7(ctx->dch, p, ctx->k7_grid, ctx->stream));
    } else {
        CK(launch_k7(ctx->dch, p, ctx->k7_grid, ctx->stream, ctx->d_bnd, ctx->n_bnd));
        CK(launch_if_partial(ctx->dch, ctx->d_slot, ctx->d_xbuf, ctx->d_send_if, ctx->n_send, ctx->d_sendbuf,
                             ctx->stream));
        if (use_nccl) {
            CK(cudaEventRecord(ctx->ev_packed, ctx->stream));
            CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
            ST(exchange_nccl(ctx, ctx->comm_stream));
            CK(cudaEventRecord(ctx->ev_exchanged, ctx->comm_stream));
        }
        // interior chunks: with an exchange in flight, SEM_COMM_SMS SMs stay free for its kernels
        CK(launch_k7(ctx->dch, p, use_nccl ? ctx->k7_grid_ovl : ctx->k7_grid, ctx->stream, ctx->d_intc, ctx->n_intc));
    }
    if (ctx->timing) ST(record(ctx, ctx->ev7, false));
    const bool k8 = p.cnt == nullptr;  // fused: K7 finalised the rank-local shared nodes
    if (ctx->timing && (k8 || ctx->n_if > 0)) ST(record(ctx, ctx->ev8, true));
    if (k8) CK(launch_k8(ctx->dch, p, ctx->stream));
    if (use_nccl && ctx->n_if > 0) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_exchanged, 0));
    if (ctx->timing && ctx->n_if == 0 && k8) ST(record(ctx, ctx->ev8, false));
    return SEM_OK;
}

HeunParams heun_params(sem_ctx *ctx) {
    HeunParams p;
    for (int g = 0; g < 5; g++) p.geo[g] = ctx->d_geo[g];
    p.hM = ctx->d_dt2M;
    p.U = ctx->d_U[0];
    p.W = ctx->d_W;
    p.V = ctx->d_V;
    p.slot = ctx->d_slot;
    p.src = ctx->src_int; p.amp = ctx->amp; p.f0 = ctx->f0; p.t0 = ctx->t0; p.h = ctx->dt;
    p.n = ctx->step;
    return p;
}

// One Heun step (heun.cu), phase 1: element pass with the lagged V update
// (boundary chunks first when there are rank-interface nodes, their (R(V), K U)
// partials packed and exchanged on the comm stream while the interior chunks
// run), then the rank-local shared-node fix-up.
sem_status heun_phase1(sem_ctx *ctx, bool use_nccl) {
    CK(cudaSetDevice(ctx->device));
    ST(ensure_tables(ctx));
    const HeunParams p = heun_params(ctx);
    const int mode = ctx->v_lag ? 1 : 0;
    if (ctx->timing) ST(record(ctx, ctx->ev7, true));
    if (ctx->n_if == 0) {
        CK(launch_heun(ctx->dch, p, mode, ctx->stream));
    } else {
        CK(launch_heun(ctx->dch, p, mode, ctx->stream, ctx->d_bnd, ctx->n_bnd));
        CK(launch_heun_if_partial(ctx->dch, ctx->d_slot, ctx->d_xbuf, ctx->d_send_if, ctx->n_send, ctx->d_sendbuf,
                                  ctx->stream));
        if (use_nccl) {
            CK(cudaEventRecord(ctx->ev_packed, ctx->stream));
            CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
            ST(exchange_nccl(ctx, ctx->comm_stream, 2));
            CK(cudaEventRecord(ctx->ev_exchanged, ctx->comm_stream));
        }
        CK(launch_heun(ctx->dch, p, mode, ctx->stream, ctx->d_intc, ctx->n_intc));
    }
    if (ctx->timing) ST(record(ctx, ctx->ev7, false));
    if (ctx->timing) ST(record(ctx, ctx->ev8, true));
    CK(launch_heun_fix(ctx->dch, p, ctx->stream));
    if (use_nccl && ctx->n_if > 0) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_exchanged, 0));
    if (ctx->timing && ctx->n_if == 0) ST(record(ctx, ctx->ev8, false));
    return SEM_OK;
}

// Heun phase 2: rank-ordered interface sums + update; advance the step.
sem_status heun_phase2(sem_ctx *ctx) {
    CK(cudaSetDevice(ctx->device));
    if (ctx->n_if > 0) {
        CK(launch_heun_if(ctx->dch, heun_params(ctx), ctx->d_xbuf, ctx->d_sum_start, ctx->d_sum_src, ctx->stream));
        if (ctx->timing) ST(record(ctx, ctx->ev8, false));
    }
    ctx->v_lag = true;  // V now lags W by one update
    ctx->step++;
    if (ctx->timing && ctx->ev7.size() >= 4096) ST(drain_events(ctx));
    return SEM_OK;
}

// NEXT-4 ablation step: atomic or global-colour scatter of K U, then the update.
sem_status ablation_step(sem_ctx *ctx) {
    CK(cudaSetDevice(ctx->device));
    ST(ensure_tables(ctx));
    const StepParams p = step_params(ctx);
    const bool atomic = ctx->mesh_scatter == SEM_SCATTER_ATOMIC;
    if (ctx->timing) ST(record(ctx, ctx->ev7, true));
    for (size_t c = 0; c + 1 < ctx->color_off.size(); c++)
        CK(launch_abl_elem(ctx->Np, atomic, ctx->d_mu_abl, ctx->d_eidx_abl, ctx->color_off[c], ctx->color_off[c + 1],
                           p, ctx->d_KU, ctx->stream));
    if (ctx->timing) ST(record(ctx, ctx->ev7, false));
    if (ctx->timing) ST(record(ctx, ctx->ev8, true));
    CK(launch_abl_update(ctx->dch.N_tot, p, ctx->d_KU, ctx->stream));
    if (ctx->timing) ST(record(ctx, ctx->ev8, false));
    ctx->cur = 1 - ctx->cur;
    ctx->step++;
    if (ctx->timing && ctx->ev7.size() >= 4096) ST(drain_events(ctx));
    return SEM_OK;
}

// Apply a pending lagged V update (before V is read or overwritten in part).
sem_status heun_finalize(sem_ctx *ctx) {
    if (!ctx->v_lag) return SEM_OK;
    CK(cudaSetDevice(ctx->device));
    ST(ensure_tables(ctx));
    CK(launch_heun(ctx->dch, heun_params(ctx), 2, ctx->stream));
    ctx->v_lag = false;
    return SEM_OK;
}

// Step phase 2: rank-ordered interface sums + update; advance the step.
sem_status step_phase2(sem_ctx *ctx) {
    CK(cudaSetDevice(ctx->device));
    if (ctx->n_if > 0) {
        const StepParams p = step_params(ctx);
        CK(launch_k8_if(ctx->dch, p, ctx->d_xbuf, ctx->d_sum_start, ctx->d_sum_src, ctx->stream));
        if (ctx->timing) ST(record(ctx, ctx->ev8, false));
    }
    ctx->cur = 1 - ctx->cur;
    ctx->step++;
    if (ctx->timing && ctx->ev7.size() >= 4096) ST(drain_events(ctx));
    return SEM_OK;
}

sem_status build_phase1(sem_ctx *ctx, const double *c_elem_host, int64_t src_vertex, double f0, double t0,
                        double amplitude, double dt) {
    if (!ctx->have_mesh) return fail(ctx, SEM_E_STATE, "sem_build_operators before sem_mesh_reorder");
    if (!c_elem_host) return fail(ctx, SEM_E_ARG, "c_elem is NULL");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(ctx, SEM_E_ARG, "dt must be > 0");
    if (!(f0 > 0.0) && src_vertex >= 0) return fail(ctx, SEM_E_ARG, "f0 must be > 0");
    if (src_vertex < -1 || src_vertex >= ctx->nv)
        return fail(ctx, SEM_E_ARG, "source vertex " + std::to_string(src_vertex) + " out of range");
    if (ctx->integrator == SEM_INTEGRATOR_HEUN) {
        if (ctx->mesh_scatter != SEM_SCATTER_CHUNK)
            return fail(ctx, SEM_E_UNSUPPORTED, "the ablation scatters run the leapfrog only");
        if (ctx->T.consistent)
            return fail(ctx, SEM_E_UNSUPPORTED, "Heun needs the nodal quadrature (P = 2, 3, 5; reading R21b)");
        if (!heun_supported(ctx->Np, ctx->dch.B))
            return fail(ctx, SEM_E_UNSUPPORTED, "Heun kernels are built for chunks of 128 or 256 elements");
    }
    CK(cudaSetDevice(ctx->device));
    reset_ops(ctx);
    ctx->prep_build_ms = -now_ms();
    cudaStream_t s = ctx->stream;
    const DevChunks &d = ctx->dch;
    const int64_t Epad = d.nchunks * d.B;
    auto &L = ctx->ops_allocs;
    TmpList tmp{ctx->stream, {}};
    double *d_c = nullptr, *d_detJ = nullptr;
    int32_t *d_bad = nullptr;
    CK(dalloc(tmp, &d_c, ctx->E_glob));
    CK(dalloc(tmp, &d_detJ, Epad));
    CK(dalloc(tmp, &d_bad, 1));
    CK(cudaMemcpyAsync(d_c, c_elem_host, sizeof(double) * ctx->E_glob, cudaMemcpyHostToDevice, s));
    {  // every wave speed positive and finite (on the device: a host loop over E cost ~8 ms at C4)
        int32_t *d_badc = nullptr, badc = INT_MAX;
        CK(dalloc(tmp, &d_badc, 1));
        CK(launch_fill_i32(d_badc, 1, INT_MAX, s));
        CK(launch_check_positive(d_c, ctx->E_glob, d_badc, s));
        CK(cudaMemcpyAsync(&badc, d_badc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (badc != INT_MAX) return fail(ctx, SEM_E_ARG, "element " + std::to_string(badc) + " has wave speed c <= 0");
    }
    const bool heun = ctx->integrator == SEM_INTEGRATOR_HEUN;
    const int64_t Nt = d.N_tot + 2;
    CK(dalloc(L, &ctx->d_dt2M, Nt));
    CK(dalloc(L, &ctx->d_U[0], Nt));
    CK(launch_fill_i32(d_bad, 1, INT_MAX, s));
    if (!heun) {
        CK(dalloc(L, &ctx->d_Grr, Epad));
        CK(dalloc(L, &ctx->d_Gss, Epad));
        CK(dalloc(L, &ctx->d_Grs, Epad));
        CK(dalloc(L, &ctx->d_U[1], Nt));
        CK(dalloc(L, &ctx->d_slot, d.n_slots + 2));
        ctx->fuse_k8 = getenv("SEM_FUSE_K8") != nullptr;
        if (ctx->fuse_k8) {
            CK(dalloc(L, &ctx->d_cnt, d.N_sh + 1));
            CK(cudaMemsetAsync(ctx->d_cnt, 0, sizeof(int32_t) * (d.N_sh + 1), s));
        }
        CK(launch_geometry(ctx->d_vxy, ctx->d_tri_or, ctx->d_perm + ctx->e0, d_c, ctx->E, Epad, ctx->d_Grr,
                           ctx->d_Gss, ctx->d_Grs, d_detJ, d_bad, s));
        if (ctx->mesh_scatter != SEM_SCATTER_CHUNK) {
            CK(dalloc(L, &ctx->d_KU, Nt));
            CK(cudaMemsetAsync(ctx->d_KU, 0, sizeof(double) * Nt, s));
        }
    } else {
        for (auto &g : ctx->d_geo) CK(dalloc(L, &g, Epad));
        CK(dalloc(L, &ctx->d_W, Nt));
        CK(dalloc(L, &ctx->d_V, Epad * 2 * ctx->Np));
        CK(dalloc(L, &ctx->d_slot, 2 * d.n_slots + 4));
        CK(launch_geometry_heun(ctx->d_vxy, ctx->d_tri_or, ctx->d_perm + ctx->e0, d_c, ctx->E, Epad, ctx->d_geo,
                                d_detJ, d_bad, s));
        CK(cudaMemsetAsync(ctx->d_W, 0, sizeof(double) * Nt, s));
        CK(cudaMemsetAsync(ctx->d_V, 0, sizeof(double) * Epad * 2 * ctx->Np, s));
        ctx->v_lag = false;
    }
    ctx->ops_integrator = ctx->integrator;
    g_const_P = 0;
    ST(ensure_tables(ctx));
    // lumped mass -> dt^2 / M-bar (leapfrog) or (h/2) / M-bar (Heun)
    CK(assemble_mass(d, d_detJ, heun ? 0.5 * dt : dt * dt, ctx->d_slot, ctx->d_dt2M, s));
    CK(launch_if_partial(d, ctx->d_slot, ctx->d_xbuf, ctx->d_send_if, ctx->n_send, ctx->d_sendbuf, s));
    CK(cudaMemsetAsync(ctx->d_U[0], 0, sizeof(double) * Nt, s));
    if (!heun) CK(cudaMemsetAsync(ctx->d_U[1], 0, sizeof(double) * Nt, s));
    int32_t bad = 0;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad != INT_MAX) return fail(ctx, SEM_E_MESH, "element " + std::to_string(bad) + " has detJ <= 0");
    ctx->src_int = -1;
    if (src_vertex >= 0 && ctx->src_lookup.empty()) {  // one rank: search the device map
        int32_t *d_l = nullptr;
        CK(dalloc(tmp, &d_l, 1));
        CK(launch_find_i32(ctx->d_loc_can, ctx->N, (int32_t)src_vertex, d_l, s));
        int32_t l = INT_MAX;
        CK(cudaMemcpyAsync(&l, d_l, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (l != INT_MAX) {
            CK(cudaMemcpyAsync(&ctx->src_int, ctx->d_loc_int + l, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    if (src_vertex >= 0)  // several ranks: host maps (vertex node: canonical id == input vertex id, R13)
        for (size_t l = 0; l < ctx->src_lookup.size(); l++)
            if (ctx->src_lookup[l] == (int32_t)src_vertex) { ctx->src_int = ctx->src_int_of[l]; break; }
    ctx->amp = amplitude;
    ctx->f0 = f0;
    ctx->t0 = t0;
    ctx->dt = dt;
    ctx->prep_build_ms += now_ms();
    return SEM_OK;
}

sem_status build_phase2(sem_ctx *ctx) {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const double t = now_ms();
    const double numer = ctx->ops_integrator == SEM_INTEGRATOR_HEUN ? 0.5 * ctx->dt : ctx->dt * ctx->dt;
    CK(launch_mass_if(ctx->dch, ctx->d_xbuf, ctx->d_sum_start, ctx->d_sum_src, numer, ctx->d_dt2M, s));
    CK(cudaStreamSynchronize(s));
    ctx->step = 0;
    ctx->cur = 0;
    ctx->have_ops = true;
    ctx->prep_build_ms += now_ms() - t;
    return SEM_OK;
}

}  // namespace

extern "C" {

const char *sem_version(void) { return "sem-hilbert-b200 0.2 (sm_100a)"; }

sem_status sem_nccl_unique_id(void *out128) {
    if (!out128) return SEM_E_ARG;
    NcclApi &N = nccl();
    if (!N.ok) return SEM_E_NCCL;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return SEM_E_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return SEM_OK;
}

sem_status sem_create(sem_ctx **out, int device, int rank, int world_size,
                      const void *nccl_unique_id, void *cuda_stream, const sem_allocator *alloc) {
    if (!out) return SEM_E_ARG;
    *out = nullptr;
    if (world_size < 1 || world_size > 32 || rank < 0 || rank >= world_size || device < 0) return SEM_E_ARG;
    if (alloc && (!alloc->alloc || !alloc->free)) return SEM_E_ARG;
    sem_ctx *ctx = new (std::nothrow) sem_ctx();
    if (!ctx) return SEM_E_OOM;
    *out = ctx;
    if (alloc) {
        ctx->alloc = *alloc;
        ctx->has_alloc = true;
    }
    ctx->device = device;
    ctx->rank = rank;
    ctx->world = world_size;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device >= ndev) {
        ctx->dead = true;
        ctx->err = "no CUDA device available (libsem has no CPU fallback)";
        return SEM_E_CUDA;
    }
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess || prop.major != 10) {
        ctx->dead = true;
        ctx->err = "device is not sm_100 (B200); this library is built for sm_100a only";
        return SEM_E_CUDA;
    }
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    {
        // The preparation's temporaries come from the device's default stream-ordered
        // pool.  Keep up to 16 GB of freed pool memory mapped between calls instead of
        // releasing it at every synchronisation (the default), so a later
        // sem_mesh_reorder does not re-map it (SEM_POOL_KEEP_GB overrides; 0 = default).
        cudaMemPool_t pool;
        const char *kv = getenv("SEM_POOL_KEEP_GB");
        const uint64_t keep = (uint64_t)(kv ? atof(kv) : 16.0) * (1ull << 30);
        if (keep > 0 && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t cur = 0;
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur);
            if (cur < keep) cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, (void *)&keep);
        }
    }
    if (cuda_stream) ctx->stream = (cudaStream_t)cuda_stream;
    else {
        if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(ctx, e, "cudaStreamCreate");
        ctx->own_stream = true;
    }
    ctx->mesh_allocs.s = ctx->ops_allocs.s = ctx->stream;
    if ((e = cudaEventCreateWithFlags(&ctx->xev, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_exchanged, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(ctx, e, "cudaEventCreate");
    if (world_size > 1 && (e = cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(ctx, e, "cudaStreamCreate(comm)");
    if (world_size > 1) {
        if (!nccl_unique_id) {
            ctx->loopback = true;  // in-process partitions: step only through sem_group_*
        } else {
            NcclApi &N = nccl();
            if (!N.ok) return fail(ctx, SEM_E_NCCL, N.err);
            ncclUniqueId id;
            std::memcpy(&id, nccl_unique_id, sizeof(id));
            ncclResult_t r = N.CommInitRank(&ctx->comm, world_size, id, rank);
            if (r != ncclSuccess) return fail(ctx, SEM_E_NCCL, std::string("ncclCommInitRank: ") + N.GetErrorString(r));
        }
    }
    return SEM_OK;
}

void sem_free(sem_ctx *ctx) {
    AllocScope scope_(ctx);
    if (!ctx) return;
    if (!ctx->dead) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
    }
    reset_mesh(ctx);
    for (auto *lst : {&ctx->ev7, &ctx->ev8, &ctx->pool})
        for (auto &ev : *lst) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
    for (cudaEvent_t e : ctx->gev) cudaEventDestroy(e);
    if (ctx->xev) cudaEventDestroy(ctx->xev);
    if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
    if (ctx->ev_exchanged) cudaEventDestroy(ctx->ev_exchanged);
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    if (ctx->io_stream) cudaStreamDestroy(ctx->io_stream);
    if (ctx->io_ev) cudaEventDestroy(ctx->io_ev);
    for (auto &e : ctx->pev)
        if (e) cudaEventDestroy(e);
    if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *sem_last_error(const sem_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sem_status sem_mesh_reorder(sem_ctx *ctx, const double *vxy_host, int64_t n_vertices,
                            const int32_t *tri_host, int64_t n_elements, int degree,
                            int elem_order, int node_order, uint64_t seed,
                            uint32_t *hilbert_key_out, int32_t *elem_perm_out,
                            int32_t *node_perm_out, int64_t *n_nodes_out,
                            int32_t grid_wh_out[2]) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!degree_supported(degree))
        return fail(ctx, SEM_E_UNSUPPORTED, "unsupported degree " + std::to_string(degree) + " (2 to 7)");
    if (elem_order < 0 || elem_order > SEM_ORDER_DIST)
        return fail(ctx, SEM_E_UNSUPPORTED, "unknown element ordering " + std::to_string(elem_order));
    if (node_order < SEM_NODES_FIRST_TOUCH || node_order > SEM_NODES_VISIT)
        return fail(ctx, SEM_E_UNSUPPORTED, "unknown node ordering " + std::to_string(node_order));
    const bool strategy = elem_order == SEM_ORDER_CONN || elem_order == SEM_ORDER_DIST;
    if (node_order == SEM_NODES_VISIT && !strategy)
        return fail(ctx, SEM_E_UNSUPPORTED, "SEM_NODES_VISIT needs SEM_ORDER_CONN or SEM_ORDER_DIST");
    if (!vxy_host || !tri_host || n_vertices < 3 || n_elements < 1)
        return fail(ctx, SEM_E_ARG, "empty or missing mesh arrays");
    const int Np = (degree + 1) * (degree + 2) / 2;
    if (n_elements * Np >= (int64_t)INT_MAX || n_vertices >= INT_MAX)
        return fail(ctx, SEM_E_ARG, "mesh too large for 32-bit indices");
    if (n_elements < ctx->world) return fail(ctx, SEM_E_ARG, "fewer elements than ranks");
    try {
        CK(cudaSetDevice(ctx->device));
        reset_mesh(ctx);
        const double t_start = now_ms();
        cudaStream_t s = ctx->stream;
        PhaseTrace tr;
        ctx->P = degree;
        ctx->Np = Np;
        ctx->nv = n_vertices;
        ctx->E_glob = n_elements;
        if (!build_ref_tables(degree, ctx->T)) return fail(ctx, SEM_E_UNSUPPORTED, "reference tables");
        const int64_t E = n_elements, nv = n_vertices;
        TmpList tmp{ctx->stream, {}};  // freed (stream-ordered) at the end of this call

        CK(dalloc(ctx->mesh_allocs, &ctx->d_vxy, 2 * nv));
        CK(cudaMemcpyAsync(ctx->d_vxy, vxy_host, sizeof(double) * 2 * nv, cudaMemcpyHostToDevice, s));
        int32_t *d_tri = nullptr, *d_bad = nullptr;
        CK(dalloc(tmp, &d_tri, 3 * E));
        CK(dalloc(tmp, &d_bad, 2));  // zero-area element, vertex id out of range (checked on the GPU)
        CK(cudaMemcpyAsync(d_tri, tri_host, sizeof(int32_t) * 3 * E, cudaMemcpyHostToDevice, s));
        CK(dalloc(ctx->mesh_allocs, &ctx->d_tri_or, 3 * E));
        CK(launch_fill_i32(d_bad, 2, INT_MAX, s));
        CK(launch_orient(ctx->d_vxy, d_tri, E, nv, ctx->d_tri_or, d_bad, s));
        int32_t bad[2] = {0, 0};
        CK(cudaMemcpyAsync(bad, d_bad, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (bad[1] != INT_MAX)
            return fail(ctx, SEM_E_MESH, "element " + std::to_string(bad[1]) + " has a vertex id out of range");
        if (bad[0] != INT_MAX) return fail(ctx, SEM_E_MESH, "element " + std::to_string(bad[0]) + " has zero area");
        tr.mark(s, "H2D + orientation");

        // ---- canonical SEM nodes (reading R13) ----
        int32_t *d_mu_can = nullptr, *d_node_perm = nullptr;
        CK(dalloc(tmp, &d_mu_can, E * Np));
        int64_t nedges = 0, nunused = 0;
        int32_t first_unused = 0;
        CK(canonical_nodes(ctx->d_tri_or, nv, E, degree, d_mu_can, &nedges, &nunused, &first_unused, s));
        if (nunused)
            return fail(ctx, SEM_E_MESH, "vertex " + std::to_string(first_unused) + " is not used by any element");
        const int nI = (degree - 1) * (degree - 2) / 2;
        const int64_t N = nv + nedges * (degree - 1) + E * nI;
        if (N >= INT_MAX) return fail(ctx, SEM_E_ARG, "too many nodes for 32-bit indices");
        ctx->N_glob = N;
        CK(dalloc(tmp, &d_node_perm, N));
        tr.mark(s, "canonical nodes");
        // node graph: degrees for FIRST_TOUCH_DEGREE and the Conn. key, adjacency for Conn./Dist.
        DevGraph graph;
        struct GraphGuard { DevGraph &g; cudaStream_t s; ~GraphGuard() { free_node_graph(g, s); } } gguard{graph, s};
        if (strategy || node_order == SEM_NODES_FIRST_TOUCH_DEGREE) {
            int bad_graph = 0;
            CK(build_node_graph(d_mu_can, E, Np, N, strategy, graph, &bad_graph, s));
            if (bad_graph) return fail(ctx, SEM_E_MESH, "a node's elements hold more than 384 node entries");
            tr.mark(s, "node graph");
        }

        // ---- element order (list L) ----
        CK(dalloc(ctx->mesh_allocs, &ctx->d_perm, E));
        int32_t *d_ids = nullptr;
        CK(dalloc(tmp, &d_ids, E));
        CK(launch_iota(d_ids, E, s));
        ctx->grid[0] = ctx->grid[1] = 0;
        if (elem_order == SEM_ORDER_INPUT) {
            CK(cudaMemcpyAsync(ctx->d_perm, d_ids, sizeof(int32_t) * E, cudaMemcpyDeviceToDevice, s));
            if (hilbert_key_out) std::memset(hilbert_key_out, 0, sizeof(uint32_t) * E);
        } else if (elem_order == SEM_ORDER_HILBERT) {
            double *d_bb = nullptr;
            CK(dalloc(tmp, &d_bb, 4));
            CK(launch_bbox(ctx->d_vxy, nv, d_bb, s));
            double bb[4];
            CK(cudaMemcpyAsync(bb, d_bb, sizeof(bb), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            // PAPER.md:301 step 2 with reading R9 (same operation order as written)
            const double wm = bb[2] - bb[0], hm = bb[3] - bb[1];
            if (!(wm > 0.0) || !(hm > 0.0)) return fail(ctx, SEM_E_MESH, "mesh has zero width or height");
            const double r = wm / hm;
            const double sq = std::sqrt((double)E);
            const double wbd = std::ceil(sq), hbd = std::ceil(sq / r);
            const int64_t wb = wbd < 1.0 ? 1 : (int64_t)wbd, hb = hbd < 1.0 ? 1 : (int64_t)hbd;
            if (wb * hb > (int64_t)0xFFFFFFFFLL || wb > INT_MAX / 4 || hb > INT_MAX / 4)
                return fail(ctx, SEM_E_ARG, "SFC grid too large");
            const double ws = (double)wb / wm, hs = (double)hb / hm;
            ctx->grid[0] = (int32_t)wb;
            ctx->grid[1] = (int32_t)hb;
            uint32_t *d_keys = nullptr, *d_keys2 = nullptr;
            CK(dalloc(tmp, &d_keys, E));
            CK(dalloc(tmp, &d_keys2, E));
            CK(launch_hilbert_keys(ctx->d_vxy, d_tri, E, bb[0], bb[1], ws, hs, (int32_t)wb,
                                   (int32_t)hb, d_keys, s));
            int bits = 1;
            while (bits < 32 && ((int64_t)1 << bits) < wb * hb) bits++;
            CK(sort_pairs_u32(d_keys, d_ids, d_keys2, ctx->d_perm, E, bits, s));
            if (hilbert_key_out)
                CK(cudaMemcpyAsync(hilbert_key_out, d_keys, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost, s));
        } else if (elem_order == SEM_ORDER_RANDOM) {
            uint64_t *d_k = nullptr, *d_k2 = nullptr;
            CK(dalloc(tmp, &d_k, E));
            CK(dalloc(tmp, &d_k2, E));
            CK(launch_random_keys(E, seed, d_k, s));
            CK(sort_pairs_u64(d_k, d_ids, d_k2, ctx->d_perm, E, 64, s));
            if (hilbert_key_out) std::memset(hilbert_key_out, 0, sizeof(uint32_t) * E);
        } else {  // Conn. / Dist. (reading R20)
            double x0 = 0.0, y0 = 0.0;
            if (elem_order == SEM_ORDER_DIST) {
                double *d_bb = nullptr;
                CK(dalloc(tmp, &d_bb, 4));
                CK(launch_bbox(ctx->d_vxy, nv, d_bb, s));
                double bb[4];
                CK(cudaMemcpyAsync(bb, d_bb, sizeof(bb), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                x0 = bb[0];
                y0 = bb[1];
            }
            double edge_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int i = 1; i < degree; i++) edge_t[i - 1] = ctx->T.node[i][0];  // lattice row j = 0
            int64_t levels = 0;
            CK(strategy_order(d_mu_can, ctx->d_vxy, ctx->d_tri_or, E, degree, N,
                              elem_order == SEM_ORDER_CONN ? 0 : 1, graph, edge_t, x0, y0, ctx->d_perm,
                              d_node_perm, &levels, s));
            ctx->strategy_levels = levels;
            if (hilbert_key_out) std::memset(hilbert_key_out, 0, sizeof(uint32_t) * E);
        }

        tr.mark(s, "element order");
        // ---- relabel ----
        int32_t *d_mu_new = nullptr, *d_mu_ft = nullptr;
        CK(dalloc(tmp, &d_mu_new, E * Np));
        CK(launch_permute_rows(d_mu_can, ctx->d_perm, E, Np, d_mu_new, s));
        if (node_order == SEM_NODES_FIRST_TOUCH || node_order == SEM_NODES_FIRST_TOUCH_DEGREE) {
            CK(dalloc(tmp, &d_mu_ft, E * Np));
            int64_t nl = 0;
            CK(first_touch(d_mu_new, E, Np, N, d_node_perm, d_mu_ft, &nl, s,
                           node_order == SEM_NODES_FIRST_TOUCH_DEGREE ? graph.deg : nullptr));
            if (nl != N) return fail(ctx, SEM_E_MESH, "first-touch labelled " + std::to_string(nl) +
                                                          " of " + std::to_string(N) + " nodes");
        } else if (node_order == SEM_NODES_VISIT) {  // the strategy's node list (d_node_perm = visit order)
            CK(dalloc(tmp, &d_mu_ft, E * Np));
            CK(relabel_from_perm(d_mu_new, E * Np, d_node_perm, N, d_mu_ft, s));
        } else {
            CK(launch_iota(d_node_perm, N, s));
            d_mu_ft = d_mu_new;
        }

        tr.mark(s, "node numbering");
        // ---- host outputs ----
        const bool one = ctx->world == 1;  // fast path: every node local, identity maps
        // partition and chunk metadata built on the GPU (partition_gpu.cu, chunks_gpu.cu)
        // unless a host-side consumer (the ablation scatters) needs mu
        const bool gpu_chunks = ctx->scatter == SEM_SCATTER_CHUNK && getenv("SEM_HOST_CHUNKS") == nullptr;
        const bool check_chunks = gpu_chunks && getenv("SEM_CHUNK_CHECK") != nullptr;
        std::vector<int32_t> node_perm, mu_h;
        if (!one && !gpu_chunks) {  // the host partition and the rank maps need it
            node_perm.resize(N);
            CK(cudaMemcpyAsync(node_perm.data(), d_node_perm, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, s));
        }
        // the caller's permutations go out on a side stream while the chunk builder runs (pinned
        // destinations overlap; pageable ones are staged by the copy call); every return below
        // waits for them first (io_sync, destroyed before the temporaries)
        struct IoSync {
            cudaStream_t st = nullptr;
            ~IoSync() {
                if (st) cudaStreamSynchronize(st);
            }
        } io_sync;
        if (node_perm_out || elem_perm_out) {
            if (!ctx->io_stream) CK(cudaStreamCreateWithFlags(&ctx->io_stream, cudaStreamNonBlocking));
            if (!ctx->io_ev) CK(cudaEventCreateWithFlags(&ctx->io_ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->io_ev, s));
            CK(cudaStreamWaitEvent(ctx->io_stream, ctx->io_ev, 0));
            io_sync.st = ctx->io_stream;
            if (node_perm_out)
                CK(cudaMemcpyAsync(node_perm_out, d_node_perm, sizeof(int32_t) * N, cudaMemcpyDeviceToHost,
                                   ctx->io_stream));
            if (elem_perm_out)
                CK(cudaMemcpyAsync(elem_perm_out, ctx->d_perm, sizeof(int32_t) * E, cudaMemcpyDeviceToHost,
                                   ctx->io_stream));
        }
        if (!gpu_chunks || check_chunks) {
            mu_h.resize((size_t)E * Np);
            CK(cudaMemcpyAsync(mu_h.data(), d_mu_ft, sizeof(int32_t) * E * Np, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        if (n_nodes_out) *n_nodes_out = N;
        if (grid_wh_out) { grid_wh_out[0] = ctx->grid[0]; grid_wh_out[1] = ctx->grid[1]; }

        tr.mark(s, "D2H outputs");
        // ---- this rank's part: contiguous range of the global order ----
        Partition part;
        DevPartition dpart;
        std::string err;
        auto &L = ctx->mesh_allocs;
        const DeviceAlloc da = [&L](void **p, size_t bytes) { return dalloc(L, (char **)p, bytes); };
        if (!one && gpu_chunks) {
            CK(build_partition_gpu(d_mu_ft, E, Np, N, ctx->rank, ctx->world, da, dpart, err, s));
            if (!err.empty()) return fail(ctx, SEM_E_MESH, err);
            ctx->e0 = dpart.e0;
            ctx->E = dpart.e1 - dpart.e0;
            ctx->N = dpart.NL;
            part.nbr = dpart.nbr;
            part.nbr_off = dpart.nbr_off;
            part.send_if = dpart.send_if;
            part.sum_start = dpart.sum_start;
            part.sum_src = dpart.sum_src;
            if (check_chunks) {  // the host partition must agree
                if (!build_partition(mu_h.data(), E, Np, N, ctx->rank, ctx->world, part, err))
                    return fail(ctx, SEM_E_MESH, err);
                std::string diff;
                if (part.e0 != dpart.e0 || part.e1 != dpart.e1 || (int64_t)part.loc2glob.size() != dpart.NL ||
                    (int64_t)part.if_local.size() != dpart.n_if)
                    diff = "sizes";
                else if (!same_dev(part.loc2glob, dpart.loc2glob, part.loc2glob.size(), s)) diff = "loc2glob";
                else if (!same_dev(part.mu_local, dpart.mu_local, part.mu_local.size(), s)) diff = "mu_local";
                else if (!same_dev(part.remote, dpart.remote, part.remote.size(), s)) diff = "remote";
                else if (!same_dev(part.owned, dpart.owned, part.owned.size(), s)) diff = "owned";
                else if (part.nbr != dpart.nbr || part.nbr_off != dpart.nbr_off || part.send_if != dpart.send_if ||
                         part.sum_start != dpart.sum_start || part.sum_src != dpart.sum_src)
                    diff = "exchange lists";
                if (!diff.empty()) return fail(ctx, SEM_E_MESH, "GPU partition differs from the host's: " + diff);
            }
        } else if (!one) {
            if (!build_partition(mu_h.data(), E, Np, N, ctx->rank, ctx->world, part, err))
                return fail(ctx, SEM_E_MESH, err);
            std::vector<int32_t>().swap(mu_h);
            ctx->e0 = part.e0;
            ctx->E = part.e1 - part.e0;
            ctx->N = (int64_t)part.loc2glob.size();
        } else {
            part.nbr_off.assign(1, 0);
            part.sum_start.assign(1, 0);
            ctx->e0 = 0;
            ctx->E = E;
            ctx->N = N;
        }
        tr.mark(s, "partition");

        // ---- chunk metadata for the step kernel ----
        int B_chunk = chunk_elems(degree, ctx->integrator == SEM_INTEGRATOR_HEUN);
        ChunkMeta m;
        DevChunks &d = ctx->dch;
        const size_t mark = L.size();  // the chunk arrays start here (fallback rebuild)
        // chunks of 512 whose largest members overflow one CTA's shared memory: rebuild with 256
        const auto too_big = [&](const ChunkMeta &mm) {
            if (B_chunk != 512 || ctx->integrator == SEM_INTEGRATOR_HEUN) return false;
            DevChunks t{};
            t.Np = Np; t.B = B_chunk;
            t.max_local = mm.max_local; t.max_win = mm.max_win; t.max_count = mm.max_count; t.max_nsh = mm.max_nsh;
            return !k7_fits(t, false);
        };
        for (;;) {  // one pass, or two when chunks of 512 fall back to 256
            if (gpu_chunks) {
                CK(build_chunks_gpu(one ? d_mu_ft : dpart.mu_local, ctx->E, Np, ctx->N, B_chunk,
                                    one ? nullptr : dpart.remote, da, m, d, &ctx->d_loc_int, &ctx->d_bnd,
                                    &ctx->d_intc, err, s));
                if (!err.empty()) return fail(ctx, SEM_E_MESH, err);
                if (too_big(m)) {
                    CK(cudaStreamSynchronize(s));
                    L.release_from(mark);
                    m = ChunkMeta();
                    d = DevChunks{};
                    B_chunk = 256;
                    tr.mark(s, "chunks of 512 do not fit one CTA: rebuilt with 256");
                    continue;
                }
                if (check_chunks) {
                    ChunkMeta h;
                    if (!build_chunks(one ? mu_h.data() : part.mu_local.data(), ctx->E, Np, ctx->N, B_chunk, h,
                                      err, one ? nullptr : part.remote.data()))
                        return fail(ctx, SEM_E_MESH, err);
                    const std::string diff = compare_chunks(h, m, d, ctx->d_loc_int, s);
                    if (!diff.empty())
                        return fail(ctx, SEM_E_MESH, "GPU chunk builder differs from the host's: " + diff);
                }
                std::vector<int32_t>().swap(mu_h);
                tr.mark(s, "chunk builder (GPU)");
            } else {
                if (!build_chunks(one ? mu_h.data() : part.mu_local.data(), ctx->E, Np, ctx->N, B_chunk, m, err,
                                  one ? nullptr : part.remote.data()))
                    return fail(ctx, SEM_E_MESH, err);
                if (too_big(m)) {
                    m = ChunkMeta();
                    B_chunk = 256;
                    continue;
                }
            }
            break;
        }
        if (!gpu_chunks) {
            if (ctx->scatter != SEM_SCATTER_CHUNK) ST(prepare_ablation(ctx, mu_h, E, Np, N, degree, one, m, s));
            std::vector<int32_t>().swap(mu_h);
            tr.mark(s, "chunk builder (host)");
            CK(upload_chunks(L, m, d, s));
        }
        // node maps for I/O (local node l -> internal / canonical / reordered id)
        if (one) {
            // reordered id == local id; the device node_perm (reordered -> canonical) is kept
            if (!gpu_chunks) CK(upload(L, &ctx->d_loc_int, m.int_of, s));
            ctx->d_loc_can = d_node_perm;
            for (auto it = tmp.p.begin(); it != tmp.p.end(); ++it)  // kept: becomes a persistent map
                if (*it == (void *)d_node_perm) { L.push_back(*it); tmp.p.erase(it); break; }
            ctx->d_loc_ft = nullptr;
            ctx->d_own_int = ctx->d_loc_int;
            ctx->d_own_can = ctx->d_loc_can;
            ctx->d_own_ft = nullptr;
            ctx->n_own = N;
            ctx->src_lookup.clear();  // the source vertex is looked up on the device (d_loc_can)
            ctx->src_int_of.clear();
        } else if (gpu_chunks) {  // several ranks, device maps; the source is looked up on the device
            CK(partition_io_maps(dpart, d_node_perm, ctx->d_loc_int, da, &ctx->d_loc_can, &ctx->d_own_int,
                                 &ctx->d_own_can, &ctx->d_own_ft, &ctx->n_own, s));
            ctx->d_loc_ft = dpart.loc2glob;
            ctx->src_lookup.clear();
            ctx->src_int_of.clear();
        } else {
            std::vector<int32_t> loc_int(ctx->N), loc_can(ctx->N), own_int, own_can, own_ft;
            ctx->src_lookup.assign(ctx->N, -1);
            for (int64_t l = 0; l < ctx->N; l++) {
                const int32_t g = part.loc2glob[l];
                loc_int[l] = m.int_of[l];
                loc_can[l] = node_perm[g];
                if (part.owned[l]) {
                    own_int.push_back(m.int_of[l]);
                    own_can.push_back(node_perm[g]);
                    own_ft.push_back(g);
                }
            }
            ctx->n_own = (int64_t)own_int.size();
            CK(upload(L, &ctx->d_loc_int, loc_int, s));
            CK(upload(L, &ctx->d_loc_can, loc_can, s));
            CK(upload(L, &ctx->d_loc_ft, part.loc2glob, s));
            CK(upload(L, &ctx->d_own_int, own_int, s));
            CK(upload(L, &ctx->d_own_can, own_can, s));
            CK(upload(L, &ctx->d_own_ft, own_ft, s));
            ctx->src_lookup.swap(loc_can);
            ctx->src_int_of.swap(loc_int);
        }
        // interface exchange buffers
        ctx->n_if = m.N_if;
        const int64_t nif_part = (!one && gpu_chunks) ? dpart.n_if : (int64_t)part.if_local.size();
        if (nif_part != m.N_if)
            return fail(ctx, SEM_E_MESH, "interface node count mismatch between partition and chunks");
        ctx->n_send = (int64_t)part.send_if.size();
        ctx->nbr = part.nbr;
        ctx->nbr_off = part.nbr_off;
        ctx->n_bnd = (int64_t)m.bnd_chunks.size();
        ctx->n_intc = (int64_t)m.int_chunks.size();
        if (!gpu_chunks) {
            CK(upload(L, &ctx->d_bnd, m.bnd_chunks, s));
            CK(upload(L, &ctx->d_intc, m.int_chunks, s));
        }
        CK(upload(L, &ctx->d_send_if, part.send_if, s));
        CK(upload(L, &ctx->d_sum_start, part.sum_start, s));
        CK(upload(L, &ctx->d_sum_src, part.sum_src, s));
        CK(dalloc(L, &ctx->d_xbuf, 2 * (ctx->n_if + ctx->n_send) + 4));  // room for the Heun double2 payload
        CK(dalloc(L, &ctx->d_sendbuf, 2 * ctx->n_send + 4));
        CK(cudaStreamSynchronize(s));
        tr.mark(s, "uploads + maps");
        ctx->k7_grid = k7_grid(d, false);
        ctx->k7_grid_ovl = k7_grid(d, false, comm_sms());
        tr.mark(s, "k7 occupancy");
        ctx->meta_info = ChunkMeta();
        ChunkMeta &mi = ctx->meta_info;
        mi.B = m.B; mi.Np = m.Np; mi.E = m.E; mi.N = m.N; mi.nchunks = m.nchunks; mi.N_int = m.N_int;
        mi.N_sh = m.N_sh; mi.N_if = m.N_if; mi.N_tot = m.N_tot; mi.n_slots = m.n_slots;
        mi.max_local = m.max_local; mi.max_win = m.max_win; mi.max_colors = m.max_colors;
        ctx->have_mesh = true;
        ctx->prep_reorder_ms = now_ms() - t_start;
        return SEM_OK;
    } catch (const std::bad_alloc &) {
        return fail(ctx, SEM_E_OOM, "host allocation failed in sem_mesh_reorder");
    }
}

sem_status sem_build_operators(sem_ctx *ctx, const double *c_elem_host, int64_t src_vertex,
                               double f0, double t0, double amplitude, double dt) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (ctx->loopback) return fail(ctx, SEM_E_STATE, "loopback partitions are built with sem_group_build_operators");
    try {
        ST(build_phase1(ctx, c_elem_host, src_vertex, f0, t0, amplitude, dt));
        if (ctx->world > 1) ST(exchange_nccl(ctx, ctx->stream));
        return build_phase2(ctx);
    } catch (const std::bad_alloc &) {
        return fail(ctx, SEM_E_OOM, "host allocation failed in sem_build_operators");
    }
}

sem_status sem_step_n(sem_ctx *ctx, int64_t n_steps) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!ctx->have_ops) return fail(ctx, SEM_E_STATE, "sem_step_n before sem_build_operators");
    if (ctx->loopback) return fail(ctx, SEM_E_STATE, "loopback partitions step with sem_group_step_n");
    if (n_steps < 0) return fail(ctx, SEM_E_ARG, "n_steps < 0");
    if (ctx->ops_integrator == SEM_INTEGRATOR_HEUN) {
        for (int64_t k = 0; k < n_steps; k++) {
            ST(heun_phase1(ctx, ctx->world > 1));
            ST(heun_phase2(ctx));
        }
        return SEM_OK;
    }
    if (ctx->mesh_scatter != SEM_SCATTER_CHUNK) {
        for (int64_t k = 0; k < n_steps; k++) ST(ablation_step(ctx));
        return SEM_OK;
    }
    int64_t k = 0;
    if (n_steps == 0 && graph_ok(ctx)) {  // capture only (warm-up): every size, both parities
        if (ctx->timing) return graph_steps(ctx, 0);
        for (int si = 0; si < kNGraph; si++)
            for (int par = 0; par < 2; par++) ST(graph_steps(ctx, 0, si, par));
        return SEM_OK;
    }
    if (graph_ok(ctx) && ctx->timing && n_steps >= kGraphSteps) {
        const int64_t reps = n_steps / kGraphSteps;
        ST(graph_steps(ctx, reps));
        k = reps * kGraphSteps;
    } else if (graph_ok(ctx) && !ctx->timing) {
        for (int si = 0; si < kNGraph; si++) {
            const int64_t sz = kGraphSteps >> si, reps = (n_steps - k) / sz;
            // the remainder graphs only once captured (sem_step_n(0)): a first capture costs more
            // than a few steps' launch gaps save
            if (si > 0 && reps > 0 && !ctx->graph_exec[si][ctx->cur]) break;
            if (reps > 0) {
                ST(graph_steps(ctx, reps, si));
                k += reps * sz;
            }
        }
    }
    for (; k < n_steps; k++) {
        ST(step_phase1(ctx, ctx->world > 1));
        ST(step_phase2(ctx));
    }
    return SEM_OK;
}

sem_status sem_group_build_operators(sem_ctx **ctxs, int n, const double *c_elem_host, int64_t src_vertex,
                                     double f0, double t0, double amplitude, double dt) {
    AllocScope scope_((ctxs && n > 0) ? ctxs[0] : nullptr);
    for (int r = 1; ctxs && r < n; r++)  // one hook for the group (allocated and freed by each member)
        if (!ctxs[r] || ctxs[r]->has_alloc != ctxs[0]->has_alloc ||
            (ctxs[r]->has_alloc && (ctxs[r]->alloc.alloc != ctxs[0]->alloc.alloc ||
                                    ctxs[r]->alloc.free != ctxs[0]->alloc.free ||
                                    ctxs[r]->alloc.user != ctxs[0]->alloc.user)))
            return SEM_E_ARG;
    if (!ctxs || n < 1) return SEM_E_ARG;
    for (int r = 0; r < n; r++) {
        ST(check_usable(ctxs[r]));
        if (!ctxs[r]->loopback && ctxs[r]->world > 1) return fail(ctxs[r], SEM_E_STATE, "not a loopback context");
    }
    try {
        for (int r = 0; r < n; r++) ST(build_phase1(ctxs[r], c_elem_host, src_vertex, f0, t0, amplitude, dt));
        ST(exchange_loopback(ctxs, n));
        for (int r = 0; r < n; r++) ST(build_phase2(ctxs[r]));
        return SEM_OK;
    } catch (const std::bad_alloc &) {
        return SEM_E_OOM;
    }
}

sem_status sem_group_step_n(sem_ctx **ctxs, int n, int64_t n_steps) {
    AllocScope scope_((ctxs && n > 0) ? ctxs[0] : nullptr);
    for (int r = 1; ctxs && r < n; r++)  // one hook for the group (allocated and freed by each member)
        if (!ctxs[r] || ctxs[r]->has_alloc != ctxs[0]->has_alloc ||
            (ctxs[r]->has_alloc && (ctxs[r]->alloc.alloc != ctxs[0]->alloc.alloc ||
                                    ctxs[r]->alloc.free != ctxs[0]->alloc.free ||
                                    ctxs[r]->alloc.user != ctxs[0]->alloc.user)))
            return SEM_E_ARG;
    if (!ctxs || n < 1 || n_steps < 0) return SEM_E_ARG;
    for (int r = 0; r < n; r++) {
        ST(check_usable(ctxs[r]));
        if (!ctxs[r]->have_ops) return fail(ctxs[r], SEM_E_STATE, "sem_group_step_n before build");
        if (ctxs[r]->ops_integrator != ctxs[0]->ops_integrator)
            return fail(ctxs[r], SEM_E_STATE, "loopback group contexts built for different integrators");
        if (ctxs[r]->mesh_scatter != SEM_SCATTER_CHUNK)
            return fail(ctxs[r], SEM_E_UNSUPPORTED, "loopback groups use the chunk scatter");
    }
    const bool heun = ctxs[0]->ops_integrator == SEM_INTEGRATOR_HEUN;
    for (int64_t k = 0; k < n_steps; k++) {
        for (int r = 0; r < n; r++) ST(heun ? heun_phase1(ctxs[r], false) : step_phase1(ctxs[r], false));
        ST(exchange_loopback(ctxs, n, heun ? 2 : 1));
        for (int r = 0; r < n; r++) ST(heun ? heun_phase2(ctxs[r]) : step_phase2(ctxs[r]));
    }
    return SEM_OK;
}

sem_status sem_set_scatter(sem_ctx *ctx, int mode) {
    ST(check_usable(ctx));
    if (mode != SEM_SCATTER_CHUNK && mode != SEM_SCATTER_ATOMIC && mode != SEM_SCATTER_COLOR)
        return fail(ctx, SEM_E_UNSUPPORTED, "unknown scatter mode " + std::to_string(mode));
    ctx->scatter = mode;
    return SEM_OK;
}

sem_status sem_set_integrator(sem_ctx *ctx, int integrator) {
    ST(check_usable(ctx));
    if (integrator != SEM_INTEGRATOR_LEAPFROG && integrator != SEM_INTEGRATOR_HEUN)
        return fail(ctx, SEM_E_UNSUPPORTED, "unknown integrator " + std::to_string(integrator));
    ctx->integrator = integrator;
    return SEM_OK;
}

sem_status sem_read_velocity(sem_ctx *ctx, double *out_host, int64_t *step_out) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!ctx->have_ops || ctx->ops_integrator != SEM_INTEGRATOR_HEUN)
        return fail(ctx, SEM_E_STATE, "sem_read_velocity needs operators built for the Heun integrator");
    if (!out_host) return fail(ctx, SEM_E_ARG, "out is NULL");
    ST(heun_finalize(ctx));
    cudaStream_t s = ctx->stream;
    TmpList tmp{ctx->stream, {}};
    double *d_out = nullptr;
    const int64_t n = ctx->E_glob * ctx->Np * 2;  // this rank fills its own elements only
    CK(dalloc(tmp, &d_out, n));
    if (ctx->world > 1) CK(cudaMemcpyAsync(d_out, out_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CK(launch_v_out(ctx->d_V, ctx->d_perm + ctx->e0, ctx->E, ctx->Np, ctx->dch.B, d_out, s));
    CK(cudaMemcpyAsync(out_host, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> mine;
    if (ctx->world > 1) {
        mine.resize(ctx->E);
        CK(cudaMemcpyAsync(mine.data(), ctx->d_perm + ctx->e0, sizeof(int32_t) * ctx->E, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    if (step_out) *step_out = ctx->step;
    for (int64_t k = 0; k < ctx->E; k++) {
        const int64_t e = mine.empty() ? k : mine[k];
        for (int j = 0; j < 2 * ctx->Np; j++)
            if (!std::isfinite(out_host[e * 2 * ctx->Np + j]))
                return fail(ctx, SEM_E_NONFINITE, "non-finite velocity at step " + std::to_string(ctx->step) +
                                                      " (element " + std::to_string(e) + ")");
    }
    return SEM_OK;
}

sem_status sem_write_velocity(sem_ctx *ctx, const double *v_host) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!ctx->have_ops || ctx->ops_integrator != SEM_INTEGRATOR_HEUN)
        return fail(ctx, SEM_E_STATE, "sem_write_velocity needs operators built for the Heun integrator");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    TmpList tmp{ctx->stream, {}};
    double *d_in = nullptr;
    const int64_t n = ctx->E_glob * ctx->Np * 2;  // global array; each rank takes its elements
    if (v_host) {
        CK(dalloc(tmp, &d_in, n));
        CK(cudaMemcpyAsync(d_in, v_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemsetAsync(ctx->d_V, 0, sizeof(double) * ctx->dch.nchunks * ctx->dch.B * 2 * ctx->Np, s));
    CK(launch_v_in(d_in, ctx->d_perm + ctx->e0, ctx->E, ctx->Np, ctx->dch.B, ctx->d_V, s));
    CK(cudaStreamSynchronize(s));
    ctx->v_lag = false;
    return SEM_OK;
}

sem_status sem_read_field(sem_ctx *ctx, double *out_host, int numbering, int64_t *step_out) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!ctx->have_ops) return fail(ctx, SEM_E_STATE, "sem_read_field before sem_build_operators");
    if (!out_host) return fail(ctx, SEM_E_ARG, "out is NULL");
    if (numbering != SEM_NUMBERING_CANONICAL && numbering != SEM_NUMBERING_INTERNAL)
        return fail(ctx, SEM_E_ARG, "unknown numbering");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    TmpList tmp{ctx->stream, {}};
    double *d_out = nullptr;
    int32_t *d_flag = nullptr;
    const int64_t NG = ctx->N_glob;
    CK(dalloc(tmp, &d_out, NG));
    CK(dalloc(tmp, &d_flag, 1));
    const bool full = ctx->n_own == NG;  // one rank: every global node
    if (!full) CK(cudaMemcpyAsync(d_out, out_host, sizeof(double) * NG, cudaMemcpyHostToDevice, s));
    CK(launch_permute_f64(ctx->d_U[ctx->cur], ctx->d_own_int,
                          numbering == SEM_NUMBERING_CANONICAL ? ctx->d_own_can : ctx->d_own_ft, ctx->n_own,
                          d_out, s));
    CK(launch_fill_i32(d_flag, 1, INT_MAX, s));
    CK(launch_nonfinite(ctx->d_U[ctx->cur], ctx->dch.N_tot, d_flag, s));
    int32_t flag = 0;
    CK(cudaMemcpyAsync(out_host, d_out, sizeof(double) * NG, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&flag, d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (step_out) *step_out = ctx->step;
    if (flag != INT_MAX)
        return fail(ctx, SEM_E_NONFINITE, "non-finite field at step " + std::to_string(ctx->step) +
                                              " (internal node " + std::to_string(flag) + ")");
    return SEM_OK;
}

sem_status sem_write_state(sem_ctx *ctx, const double *u_curr_host, const double *u_prev_host,
                           int numbering) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    if (!ctx->have_ops) return fail(ctx, SEM_E_STATE, "sem_write_state before sem_build_operators");
    if (numbering != SEM_NUMBERING_CANONICAL && numbering != SEM_NUMBERING_INTERNAL)
        return fail(ctx, SEM_E_ARG, "unknown numbering");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    TmpList tmp{ctx->stream, {}};
    double *d_in = nullptr;
    CK(dalloc(tmp, &d_in, ctx->N_glob));
    const int32_t *imap = numbering == SEM_NUMBERING_CANONICAL ? ctx->d_loc_can : ctx->d_loc_ft;
    const double *src[2] = {u_curr_host, u_prev_host};
    double *dst[2] = {ctx->d_U[ctx->cur], ctx->d_U[1 - ctx->cur]};
    const bool heun = ctx->ops_integrator == SEM_INTEGRATOR_HEUN;
    if (heun && u_prev_host) return fail(ctx, SEM_E_ARG, "the Heun state has no U^{n-1} (pass NULL)");
    if (heun) ST(heun_finalize(ctx));  // the pending V update uses the old W
    for (int k = 0; k < (heun ? 1 : 2); k++) {
        CK(cudaMemsetAsync(dst[k], 0, sizeof(double) * (ctx->dch.N_tot + 2), s));
        if (!src[k]) continue;
        CK(cudaMemcpyAsync(d_in, src[k], sizeof(double) * ctx->N_glob, cudaMemcpyHostToDevice, s));
        CK(launch_permute_f64(d_in, imap, ctx->d_loc_int, ctx->N, dst[k], s));
    }
    CK(cudaStreamSynchronize(s));
    return SEM_OK;
}

sem_status sem_set_step(sem_ctx *ctx, int64_t step) {
    AllocScope scope_(ctx);
    if (!ctx) return SEM_E_ARG;
    if (!ctx->have_ops) return fail(ctx, SEM_E_STATE, "sem_set_step before sem_build_operators");
    if (step < 0) return fail(ctx, SEM_E_ARG, "step < 0");
    ctx->step = step;
    return SEM_OK;
}

sem_status sem_sync(sem_ctx *ctx) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    return SEM_OK;
}

sem_status sem_get_info(sem_ctx *ctx, sem_info *o) {
    if (!ctx || !o) return SEM_E_ARG;
    std::memset(o, 0, sizeof(*o));
    if (!ctx->have_mesh) return fail(ctx, SEM_E_STATE, "no mesh");
    const ChunkMeta &m = ctx->meta_info;
    o->n_elements = ctx->E;
    o->n_nodes = ctx->N;
    o->n_nodes_global = ctx->N_glob;
    o->degree = ctx->P;
    o->nodes_per_elem = ctx->Np;
    o->n_chunks = m.nchunks;
    o->chunk_elems = m.B;
    o->max_chunk_nodes = m.max_local;
    o->n_interior_nodes = ctx->N - m.N_sh;
    o->n_shared_nodes = m.N_sh;
    o->n_partial_slots = m.n_slots;
    o->max_colors = m.max_colors;
    o->launches_per_step = 1 + ((m.N_sh - m.N_if) > 0 && !(ctx->have_ops && ctx->d_cnt) ? 1 : 0) +
                           (m.N_if > 0 ? 3 : 0);
    o->step = ctx->step;
    o->bytes_alg_per_step = (double)ctx->E * (4.0 * ctx->Np + 24.0) + 32.0 * (double)ctx->N;
    o->integrator = ctx->have_ops ? ctx->ops_integrator : ctx->integrator;
    o->scatter = ctx->mesh_scatter;
    o->n_global_colors = ctx->mesh_scatter == SEM_SCATTER_COLOR ? (int32_t)ctx->color_off.size() - 1 : 0;
    if (ctx->mesh_scatter != SEM_SCATTER_CHUNK) o->launches_per_step = (int32_t)ctx->color_off.size();
    if (o->integrator == SEM_INTEGRATOR_HEUN) {
        // mu, F (4) + sd, V read + write per element; U r/w, W r/w, (h/2)/M per node
        o->bytes_alg_per_step = (double)ctx->E * (4.0 * ctx->Np + 40.0 + 32.0 * ctx->Np) + 40.0 * (double)ctx->N;
        o->launches_per_step = 1 + ((m.N_sh - m.N_if) > 0 ? 1 : 0);
    }
    o->prep_reorder_ms = ctx->prep_reorder_ms;
    o->prep_build_ms = ctx->prep_build_ms;
    o->n_interface_nodes = m.N_if;
    o->n_neighbors = (int32_t)ctx->nbr.size();
    o->rank = ctx->rank;
    o->world_size = ctx->world;
    o->n_elements_global = ctx->E_glob;
    o->first_element = ctx->e0;
    return SEM_OK;
}

sem_status sem_set_kernel_timing(sem_ctx *ctx, int enable) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    ST(drain_events(ctx));
    ctx->timing = enable != 0;
    ctx->t7 = ctx->t8 = 0;
    ctx->n7 = ctx->n8 = 0;
    return SEM_OK;
}

sem_status sem_kernel_times(sem_ctx *ctx, double *k7_ms, int64_t *k7_launches, double *k8_ms,
                            int64_t *k8_launches) {
    AllocScope scope_(ctx);
    ST(check_usable(ctx));
    ST(drain_events(ctx));
    if (k7_ms) *k7_ms = ctx->t7;
    if (k7_launches) *k7_launches = ctx->n7;
    if (k8_ms) *k8_ms = ctx->t8;
    if (k8_launches) *k8_launches = ctx->n8;
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// Host-only diagnostics (no GPU needed), used by the CPU test-suite.
// ---------------------------------------------------------------------------
sem_status sem_debug_chunk_stats(const int32_t *mu, int64_t E, int Np, int64_t N, int B,
                                 int64_t *stats_out, int32_t *int_of_out, int32_t *cmeta_out,
                                 int32_t *own0_out) {
    if (!mu || !stats_out || E <= 0 || N <= 0) return SEM_E_ARG;
    try {
        ChunkMeta m;
        std::string err;
        if (!build_chunks(mu, E, Np, N, B, m, err)) return SEM_E_MESH;
        int64_t sum_nint = 0, sum_nsh = 0, max_nsh = 0;
        for (int64_t c = 0; c < m.nchunks; c++) {
            sum_nint += m.cmeta[8 * c + 1];
            sum_nsh += m.cmeta[8 * c + 3];
            if (m.cmeta[8 * c + 3] > max_nsh) max_nsh = m.cmeta[8 * c + 3];
        }
        const int64_t st[16] = {m.nchunks, m.N_int, m.N_sh, m.n_slots, m.max_local, m.max_win,
                                m.max_count, m.max_colors, sum_nint, sum_nsh, max_nsh, 0, 0, 0, 0, 0};
        std::memcpy(stats_out, st, sizeof(st));
        if (int_of_out) std::memcpy(int_of_out, m.int_of.data(), sizeof(int32_t) * N);
        if (cmeta_out) std::memcpy(cmeta_out, m.cmeta.data(), sizeof(int32_t) * m.cmeta.size());
        if (own0_out) std::memcpy(own0_out, m.own0.data(), sizeof(int32_t) * m.own0.size());
        return SEM_OK;
    } catch (const std::bad_alloc &) {
        return SEM_E_OOM;
    }
}

sem_status sem_debug_ref_tables(int degree, int32_t *np_out, double *nodes_out, double *wK_out, double *wM_out,
                                double *Dr_out, double *Ds_out) {
    if (!degree_supported(degree)) return SEM_E_UNSUPPORTED;
    RefTables T;
    if (!build_ref_tables(degree, T)) return SEM_E_UNSUPPORTED;
    const int Np = T.Np;
    if (np_out) *np_out = Np;
    for (int p = 0; p < Np; p++) {
        if (nodes_out) { nodes_out[2 * p] = T.node[p][0]; nodes_out[2 * p + 1] = T.node[p][1]; }
        if (wK_out) wK_out[p] = T.wK[p];
        if (wM_out) wM_out[p] = T.wM[p];
        for (int q = 0; q < Np; q++) {
            if (Dr_out) Dr_out[p * Np + q] = T.Dr[p][q];
            if (Ds_out) Ds_out[p * Np + q] = T.Ds[p][q];
        }
    }
    return SEM_OK;
}

sem_status sem_debug_ref_stiffness(int degree, double *Srr_out, double *Sss_out, double *Srs_out) {
    if (!degree_supported(degree)) return SEM_E_UNSUPPORTED;
    RefTables T;
    if (!build_ref_tables(degree, T)) return SEM_E_UNSUPPORTED;
    const int Np = T.Np;
    for (int p = 0; p < Np; p++)
        for (int q = 0; q < Np; q++) {
            if (Srr_out) Srr_out[p * Np + q] = T.Srr[p][q];
            if (Sss_out) Sss_out[p * Np + q] = T.Sss[p][q];
            if (Srs_out) Srs_out[p * Np + q] = T.Srs[p][q];
        }
    return SEM_OK;
}

sem_status sem_debug_partition(const int32_t *mu, int64_t E, int Np, int64_t N, int rank, int world,
                               int64_t *sizes_out, int32_t *loc2glob_out, int32_t *nbr_out, int32_t *nbr_off_out,
                               int32_t *send_glob_out, int32_t *if_glob_out, int32_t *sum_start_out,
                               int32_t *sum_src_out) {
    if (!mu || !sizes_out) return SEM_E_ARG;
    try {
        Partition P;
        std::string err;
        if (!build_partition(mu, E, Np, N, rank, world, P, err)) return SEM_E_ARG;
        const int64_t nif = (int64_t)P.if_local.size();
        sizes_out[0] = P.e0;
        sizes_out[1] = P.e1;
        sizes_out[2] = (int64_t)P.loc2glob.size();
        sizes_out[3] = (int64_t)P.nbr.size();
        sizes_out[4] = (int64_t)P.send_if.size();
        sizes_out[5] = nif;
        sizes_out[6] = (int64_t)P.sum_src.size();
        int64_t nown = 0;
        for (uint8_t o : P.owned) nown += o;
        sizes_out[7] = nown;
        if (loc2glob_out) std::memcpy(loc2glob_out, P.loc2glob.data(), sizeof(int32_t) * P.loc2glob.size());
        if (nbr_out) std::memcpy(nbr_out, P.nbr.data(), sizeof(int32_t) * P.nbr.size());
        if (nbr_off_out) std::memcpy(nbr_off_out, P.nbr_off.data(), sizeof(int32_t) * P.nbr_off.size());
        if (send_glob_out)
            for (size_t k = 0; k < P.send_if.size(); k++) send_glob_out[k] = P.loc2glob[P.if_local[P.send_if[k]]];
        if (if_glob_out)
            for (int64_t i = 0; i < nif; i++) if_glob_out[i] = P.loc2glob[P.if_local[i]];
        if (sum_start_out) std::memcpy(sum_start_out, P.sum_start.data(), sizeof(int32_t) * P.sum_start.size());
        if (sum_src_out) std::memcpy(sum_src_out, P.sum_src.data(), sizeof(int32_t) * P.sum_src.size());
        return SEM_OK;
    } catch (const std::bad_alloc &) {
        return SEM_E_OOM;
    }
}

}  // extern "C"
