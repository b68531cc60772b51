/*
 * sem.h -- C ABI of libsem.so, the B200 (sm_100a) hot path of arxiv 2104.08416:
 * the explicit spectral-element leapfrog step for the 2D acoustic wave equation
 * on unstructured triangles, after the mesh is reordered along a generalized
 * Hilbert curve.
 *
 * Call order (the paper's problem statement, PAPER.md:540 mesh -> SEM nodes,
 * :296-321 reorder, :240-263 operators, :269 explicit stepping):
 *
 *   sem_create -> [sem_set_integrator] [sem_set_scatter] -> sem_mesh_reorder ->
 *   sem_build_operators -> sem_step_n* -> sem_read_field [sem_read_velocity] ->
 *   sem_free
 *
 * Beyond the north_star leapfrog the library also runs the paper's own Heun
 * integrator on (U, V), its other reordering strategies
 * (PAPER.md:548-558), orders 2-7 and the scatter ablations; see DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Pointers named *_host are HOST memory, borrowed for the duration of the
 *    call only; the library copies what it needs.  Outputs are caller-allocated.
 *    Device memory is owned by the context and released by sem_free.
 *  - Index arrays are int32 (E*Np and N must be < 2^31).
 *  - Every call returns a sem_status; on error sem_last_error() holds a message
 *    naming the element, node or step involved.  SEM_E_CUDA is sticky: the
 *    context is unusable afterwards.  No C++ exception crosses the ABI.
 *  - Work is enqueued on the context's CUDA stream; calls that return host
 *    data synchronise that stream.
 *  - A context is not thread-safe; use one per process/GPU.
 *  - There is no CPU fallback: without a usable sm_100 device sem_create fails.
 */
#ifndef SEM_H
#define SEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sem_ctx sem_ctx;

typedef enum {
    SEM_OK = 0,
    SEM_E_ARG = 1,          /* invalid argument (range, NULL, c <= 0, dt <= 0 ...) */
    SEM_E_STATE = 2,        /* call out of order (e.g. step before build)          */
    SEM_E_MESH = 3,         /* degenerate / inconsistent mesh                      */
    SEM_E_UNSUPPORTED = 4,  /* degree not in 2..7, unknown ordering ...             */
    SEM_E_CUDA = 5,         /* CUDA error (sticky)                                 */
    SEM_E_NCCL = 6,         /* NCCL error                                          */
    SEM_E_OOM = 7,          /* device or host allocation failed                    */
    SEM_E_NONFINITE = 8     /* non-finite value in the field (step index in msg)   */
} sem_status;

/* Element orderings (§6.1).  INPUT = the paper's "None"
 * (file order); HILBERT = §4.3 steps 1-4; RANDOM = stable
 * sort of element ids by splitmix64(seed ^ id) (reading R16). */
enum { SEM_ORDER_INPUT = 0, SEM_ORDER_HILBERT = 1, SEM_ORDER_RANDOM = 2,
       /* the paper's other strategies (reading R20):
        * Cuthill-McKee traversal of the SEM node graph from the node with the
        * fewest connections (CONN) or nearest the lower-left corner (DIST); the
        * element list follows the visited nodes */
       SEM_ORDER_CONN = 3, SEM_ORDER_DIST = 4 };

/* Node numberings.  FIRST_TOUCH = PAPER.md:316 step 1 (each node gets the next
 * label the first time an element in the new order touches it);
 * FIRST_TOUCH_DEGREE = PAPER.md:316-318 steps 1 and 2 (each element's newly
 * touched nodes sorted by ascending degree, ties by canonical id; reading
 * R12); CANONICAL = the input numbering of DESIGN.md reading R13 (vertex ids,
 * then edge nodes, then interior nodes); VISIT = the node list of the CONN /
 * DIST traversal (only with those element orders). */
enum { SEM_NODES_FIRST_TOUCH = 0, SEM_NODES_FIRST_TOUCH_DEGREE = 1, SEM_NODES_CANONICAL = 2, SEM_NODES_VISIT = 3 };

/* Numbering of node arrays crossing the ABI (read_field / write_state).
 * CANONICAL = reading R13 input numbering; INTERNAL = the reordered labels
 * chosen by sem_mesh_reorder (node_perm_out maps them to CANONICAL). */
enum { SEM_NUMBERING_CANONICAL = 0, SEM_NUMBERING_INTERNAL = 1 };

/* Time integrators.  LEAPFROG = the north_star step on M U'' = -K U + f
 * (reading R1); HEUN = the paper's own predictor-corrector on the
 * first-order (U, V) system with Algorithms 1-3. */
enum { SEM_INTEGRATOR_LEAPFROG = 0, SEM_INTEGRATOR_HEUN = 1 };

/*
 * Device-memory hook: every device allocation of a context -- its mesh and
 * operator arrays and every temporary of its calls -- goes through alloc / free when a hook
 * is given (e.g. a caching allocator of the caller's framework: sem.py can route it to
 * PyTorch's), else through cudaMallocAsync / cudaFreeAsync.  alloc(bytes, stream, user)
 * returns device memory usable in stream order on `stream` (the context's stream, a
 * cudaStream_t) or NULL on failure (-> SEM_E_CUDA); free(ptr, stream, user) releases it in
 * stream order.  The hook is copied by sem_create and called only from inside that
 * context's calls, on the calling thread.
 */
typedef struct {
    void *(*alloc)(size_t bytes, void *stream, void *user);
    void (*free)(void *ptr, void *stream, void *user);
    void *user;
} sem_allocator;

/*
 * Create a context on CUDA device `device`.
 *  rank, world_size : this process's place in a multi-GPU run (world_size = 1
 *                     for one GPU; at most 32).  Rank r owns the contiguous
 *                     range [floor(rE/G), floor((r+1)E/G)) of the reordered
 *                     elements; nodes touched by several ranks
 *                     are exchanged every step (NCCL send/recv).
 *  nccl_unique_id   : 128-byte ncclUniqueId from rank 0 (sem_nccl_unique_id).
 *                     NULL with world_size > 1 creates an in-process LOOPBACK
 *                     partition: all G contexts live in one process (possibly
 *                     on one GPU) and are built/stepped together with
 *                     sem_group_build_operators / sem_group_step_n.
 *  cuda_stream      : cudaStream_t to enqueue on (e.g. torch's current stream),
 *                     or NULL for a stream owned by the context.
 *  alloc            : device-memory hook (above), or NULL for cudaMallocAsync.
 * Errors: SEM_E_ARG (bad rank/world/device), SEM_E_CUDA (no sm_100 device),
 *         SEM_E_NCCL (libnccl.so.2 not loadable / ncclCommInitRank failed).
 * On error *out may still hold a context carrying the message; free it.
 */
sem_status sem_create(sem_ctx **out, int device, int rank, int world_size,
                      const void *nccl_unique_id, void *cuda_stream, const sem_allocator *alloc);

/* 128-byte NCCL unique id for sem_create (call on rank 0, broadcast the bytes).
 * NCCL is loaded with dlopen("libnccl.so.2").  Errors: SEM_E_ARG, SEM_E_NCCL. */
sem_status sem_nccl_unique_id(void *out128);

/* Release every device buffer and the context.  NULL is a no-op. */
void sem_free(sem_ctx *ctx);

/* Last error message of this context ("" if none).  Owned by the context. */
const char *sem_last_error(const sem_ctx *ctx);

/*
 * Build the SEM mesh and reorder it.
 *
 *  vxy_host   [n_vertices][2] fp64 vertex coordinates.
 *  tri_host   [n_elements][3] int32 vertex ids of linear triangles.  A
 *             clockwise triangle is fixed by swapping its 2nd and 3rd vertex
 *             (the centroid used for the SFC key is taken before the fix).
 *  degree     polynomial order P in 2..7: Np = (P+1)(P+2)/2 local nodes,
 *             placed per DESIGN.md readings R3 / R21 (P2 midpoints; P3
 *             Gauss-Lobatto edge points + centroid; P >= 4 the Blyth-Pozrikidis
 *             Lobatto grid).  P = 4, 6 use the consistent stiffness and the
 *             HRZ-lumped mass (reading R21b; their nodal weights are negative).
 *  elem_order SEM_ORDER_*.  HILBERT follows PAPER.md:299-305: centroids ->
 *             bounding box w_b = ceil(sqrt(E)), h_b = ceil(sqrt(E)/r) of the
 *             vertex extents (r = w_m/h_m) -> generalized Hilbert curve over
 *             w_b x h_b (docs/hilbert.md) -> elements sorted stably by the
 *             curve position of their centroid's sub-rectangle.
 *  node_order SEM_NODES_* (PAPER.md:312-321 first part; reading R12).
 *  seed       used by SEM_ORDER_RANDOM only.
 *
 * Outputs (caller-allocated host memory, any may be NULL):
 *  hilbert_key_out [E]  curve position of each element (INPUT numbering);
 *                       zeros unless elem_order == HILBERT.
 *  elem_perm_out   [E]  elem_perm_out[k] = input id of the element placed k-th.
 *  node_perm_out   [N]  node_perm_out[i] = canonical id of internal node i.
 *                       (N is not known before the call: pass NULL and read
 *                       n_nodes_out, or size it as V + 3E(P-1) + E*nI.)
 *  n_nodes_out          N, the number of global SEM nodes.
 *  grid_wh_out     [2]  (w_b, h_b) for HILBERT, else (0, 0).
 *
 * Errors: SEM_E_UNSUPPORTED (degree, ordering, VISIT without CONN/DIST),
 * SEM_E_MESH ("element e has zero area", "vertex v is not used by any
 * element", a node with more than 64 entries -- elements holding it -- inside one
 * chunk of the step kernel), SEM_E_ARG, SEM_E_CUDA,
 * SEM_E_OOM.
 * Resets any operators/state of an earlier mesh.
 */
sem_status sem_mesh_reorder(sem_ctx *ctx, const double *vxy_host, int64_t n_vertices,
                            const int32_t *tri_host, int64_t n_elements, int degree,
                            int elem_order, int node_order, uint64_t seed,
                            uint32_t *hilbert_key_out, int32_t *elem_perm_out,
                            int32_t *node_perm_out, int64_t *n_nodes_out,
                            int32_t grid_wh_out[2]);

/*
 * Build the per-element operators and the lumped mass (PAPER.md:163-171 element
 * map, :206 inverse Jacobian, :240-250 lumped M-bar), and set the source.
 *
 *  c_elem_host [E] wave speed per element, INPUT element numbering, > 0.
 *              Reading R2: M^(e) = 1, F^(e) = c_e^2 I, B = -I, so
 *              the element stiffness is K^e = sum_ab G_ab S_ab with
 *              G = c^2 detJ J^-1 J^-T (reading R5).
 *  src_vertex  input vertex id (= canonical node id) of the Ricker point source
 *              (Algorithm 3); -1 for no source.
 *  f0, t0, amplitude: source A * r(t), r(t) = (1 - 2 pi^2 f0^2 tau^2)
 *              exp(-pi^2 f0^2 tau^2), tau = t - t0 (reading R7).
 *  dt          time step (> 0), used as dt^2 / M-bar.
 * Resets the state to U^0 = U^-1 = 0 at step 0.
 * Errors: SEM_E_STATE (no mesh), SEM_E_ARG (c <= 0 names the element, dt <= 0,
 * src out of range), SEM_E_CUDA.
 */
sem_status sem_build_operators(sem_ctx *ctx, const double *c_elem_host, int64_t src_vertex,
                               double f0, double t0, double amplitude, double dt);

/*
 * Advance n_steps leapfrog steps (north_star; reading R1):
 *   U^{n+1} = 2 U^n - U^{n-1} + (dt^2 / M-bar) (A r(n dt) e_src - K U^n)
 * where K U^n is the element-by-element stiffness apply with gather and
 * conflict-free scatter (Algorithms 1-2, fused).
 * Enqueued on the context stream; returns without synchronising.  With one
 * rank (leapfrog, chunk scatter, kernel timing off) whole blocks of 32 steps
 * replay a captured CUDA graph (step index in a device counter); the
 * environment variable SEM_GRAPH=0 disables it.  n_steps = 0 advances nothing
 * but captures that graph for the current U parity (a warm-up that keeps the
 * capture out of a later timed call).
 * Errors: SEM_E_STATE (no operators), SEM_E_ARG (n_steps < 0), SEM_E_CUDA.
 */
sem_status sem_step_n(sem_ctx *ctx, int64_t n_steps);

/*
 * Loopback partitions (contexts created with world_size > 1 and no NCCL id):
 * the same builds and steps as sem_build_operators / sem_step_n, run for all n
 * contexts of the group together; the interface exchange is a device-to-device
 * copy ordered with CUDA events.  The kernels are the multi-GPU ones.
 */
sem_status sem_group_build_operators(sem_ctx **ctxs, int n, const double *c_elem_host, int64_t src_vertex,
                                     double f0, double t0, double amplitude, double dt);
sem_status sem_group_step_n(sem_ctx **ctxs, int n, int64_t n_steps);

/*
 * Select the time integrator used by the next sem_build_operators (default
 * LEAPFROG).  With SEM_INTEGRATOR_HEUN (§4.2.1):
 *   predictor  U~ = U + h Udot(V, t_n),  V~ = V + h Vdot(U)
 *   corrector  U+ = U + h/2 (Udot(V, t_n) + Udot(V~, t_n+1)),
 *              V+ = V + h/2 (Vdot(U) + Vdot(U~))
 * with Vdot = Algorithm 1 (F = c^2 I), Udot = M-bar^-1 (R(V) +
 * y(t)) with R = Algorithm 2 (B = -I) and y = Algorithm 3;
 * t_n = n h, the corrector's source at t_{n+1} (reading R18).  The state is
 * (U [N], V [E][Np][2]), zero after sem_build_operators; `dt` is h.  Heun runs
 * at P = 2, 3 (chunks of 128 or 256 elements), P = 5 (chunks of 128) and P = 7
 * (chunks of 64; the paper's order-7 runs), on one rank or
 * several (interface exchange of the (R(V), K U) pairs; loopback groups too).
 * P = 4, 6 have no nodal quadrature (reading R21b): SEM_E_UNSUPPORTED
 * from sem_build_operators.  Selecting HEUN before sem_mesh_reorder also picks
 * its chunk size.
 * Errors: SEM_E_UNSUPPORTED (unknown integrator).
 */
sem_status sem_set_integrator(sem_ctx *ctx, int integrator);

/*
 * Scatter of the element contributions for the leapfrog step (NEXT-4 ablation,
 * SURVEY §8a "rejected as primary").  Takes effect at the next
 * sem_mesh_reorder; world_size 1 and the leapfrog only.
 *  SEM_SCATTER_CHUNK  the product path: chunk-owned CSR reduction in shared
 *                     memory + ordered slots (deterministic, bitwise reproducible);
 *  SEM_SCATTER_ATOMIC one thread per element, fp64 atomicAdd into a global K U
 *                     (addition order not fixed: results vary in the last bits);
 *  SEM_SCATTER_COLOR  the paper's Algorithm 2 scatter: a greedy
 *                     global element colouring in element order, one launch per
 *                     colour with plain read-modify-write (deterministic).
 * Errors: SEM_E_UNSUPPORTED (unknown mode; world_size > 1 or Heun at the
 * next reorder / build).
 */
enum { SEM_SCATTER_CHUNK = 0, SEM_SCATTER_ATOMIC = 1, SEM_SCATTER_COLOR = 2 };
sem_status sem_set_scatter(sem_ctx *ctx, int mode);

/*
 * Heun only: copy V^n to out_host[E][Np][2] (fp64; INPUT element order, local
 * node p in the lattice order of reading R3 after the orientation fix, then the
 * x and y components; E = all elements of the mesh, each rank writing the
 * elements it owns and leaving the others as they were) and return the step
 * index.  Synchronises.
 * Errors: SEM_E_STATE (no Heun operators), SEM_E_ARG, SEM_E_CUDA, SEM_E_NONFINITE.
 */
sem_status sem_read_velocity(sem_ctx *ctx, double *out_host, int64_t *step_out);

/* Heun only: overwrite V from v_host[E][Np][2] (layout of sem_read_velocity);
 * NULL sets V = 0.  U is set with sem_write_state(ctx, U, NULL, numbering). */
sem_status sem_write_velocity(sem_ctx *ctx, const double *v_host);

/*
 * Copy U^n to out_host[N] (fp64, N = global node count) in the requested
 * numbering and return the step index n.  With several ranks only the nodes
 * this rank owns (an interface node belongs to the lowest rank touching it) are
 * written; other entries of out_host are left as they were, so a caller merges
 * ranks by giving each the same array in turn.  Synchronises.
 * Errors: SEM_E_STATE, SEM_E_ARG, SEM_E_CUDA, SEM_E_NONFINITE ("non-finite
 * field at step n").
 */
sem_status sem_read_field(sem_ctx *ctx, double *out_host, int numbering, int64_t *step_out);

/*
 * Test/checkpoint hook: overwrite (U^n, U^{n-1}) from host arrays [N] (global
 * node count) in the given numbering; each rank takes its local nodes.  The
 * step index is left unchanged.  Either pointer may be
 * NULL to set that array to zero.  Errors: SEM_E_STATE, SEM_E_ARG, SEM_E_CUDA.
 */
sem_status sem_write_state(sem_ctx *ctx, const double *u_curr_host, const double *u_prev_host,
                           int numbering);

/* Set the step index n (used with sem_write_state to resume a run). */
sem_status sem_set_step(sem_ctx *ctx, int64_t step);

/* Synchronise the context stream and surface asynchronous errors. */
sem_status sem_sync(sem_ctx *ctx);

/* Descriptive numbers of the built problem (for the bench and tests). */
typedef struct {
    int64_t n_elements;       /* E (this rank) */
    int64_t n_nodes;          /* N (this rank's local nodes) */
    int64_t n_nodes_global;   /* N of the whole mesh */
    int32_t degree;           /* P */
    int32_t nodes_per_elem;   /* Np */
    int64_t n_chunks;         /* CTAs of the step kernel */
    int32_t chunk_elems;      /* elements per chunk */
    int32_t max_chunk_nodes;  /* largest chunk-local node table */
    int64_t n_interior_nodes; /* finalised inside the step kernel */
    int64_t n_shared_nodes;   /* finalised by the fix-up kernel */
    int64_t n_partial_slots;  /* partial sums written per step */
    int32_t max_colors;       /* largest per-chunk colour count */
    int32_t launches_per_step;/* kernels launched per leapfrog step */
    int64_t step;             /* current step index n */
    double bytes_alg_per_step;/* leapfrog: E (4 Np + 24) + 32 N;
                                 Heun: E (4 Np + 40 + 32 Np) + 40 N */
    double prep_reorder_ms;   /* last sem_mesh_reorder wall time */
    double prep_build_ms;     /* last sem_build_operators wall time */
    int64_t n_interface_nodes;/* nodes exchanged with other ranks */
    int32_t n_neighbors;      /* ranks this rank exchanges with */
    int32_t rank, world_size;
    int64_t n_elements_global;
    int64_t first_element;    /* global index of this rank's first element */
    int32_t integrator;       /* SEM_INTEGRATOR_* of the built operators (else the selected one) */
    int32_t scatter;          /* SEM_SCATTER_* the mesh was prepared for */
    int32_t n_global_colors;  /* SEM_SCATTER_COLOR: colours of the global element colouring */
    int32_t reserved0;
} sem_info;

sem_status sem_get_info(sem_ctx *ctx, sem_info *out);

/*
 * Kernel timing: when enabled, CUDA events on the context stream bracket every
 * launch of the stiffness/update kernel (K7) and the fix-up kernel (K8);
 * sem_kernel_times returns their accumulated device milliseconds and launch
 * counts since the last reset.  Synchronises.
 */
sem_status sem_set_kernel_timing(sem_ctx *ctx, int enable);
sem_status sem_kernel_times(sem_ctx *ctx, double *k7_ms, int64_t *k7_launches,
                            double *k8_ms, int64_t *k8_launches);

/*
 * Host-only diagnostic (no GPU, no context): run the chunk builder of the step
 * kernel on a reordered connectivity mu [E][Np] (node ids in [0, N), elements in
 * their final order) with chunks of B elements.  stats_out[16] receives
 * {nchunks, N_int (padded), N_sh, n_slots, max_local, max_win, max_count (most
 *  entries of one node in a chunk), max_colors, sum_nint, sum_nsh, max_nsh, 0, 0, 0, 0, 0};
 * int_of_out [N] (optional) the internal id of every node; cmeta_out
 * [nchunks*8] (optional) the per-chunk descriptors {i0, nint, s0, nsh, end0,
 * ne, nint_al, end1} (end0/end1: ends of the interior / shared jagged-diagonal
 * segments); own0_out [nchunks+1] (optional) the shared indices each chunk owns,
 * [own0[c], own0[c+1]) (owner = the last chunk touching the node; the step kernel
 * finalises them after that chunk).  Errors: SEM_E_ARG, SEM_E_MESH (unused node),
 * SEM_E_OOM.
 */
sem_status sem_debug_chunk_stats(const int32_t *mu, int64_t E, int Np, int64_t N, int B,
                                 int64_t *stats_out, int32_t *int_of_out, int32_t *cmeta_out,
                                 int32_t *own0_out);

/*
 * Host-only diagnostic of the multi-GPU partition (no GPU, no context): rank's
 * part of a reordered connectivity mu [E][Np] (global node ids in [0, N)).
 * sizes_out[8] = {e0, e1, n_local_nodes, n_neighbors, n_send, n_interface,
 * n_sum_src, n_owned}; optional arrays (caller-sized from a first call with
 * NULLs): loc2glob [n_local], nbr [n_neighbors], nbr_off [n_neighbors+1],
 * send_glob [n_send] (global id sent at each position), if_glob [n_interface],
 * sum_start [n_interface+1], sum_src [n_sum_src].  Errors: SEM_E_ARG, SEM_E_OOM.
 */
sem_status sem_debug_partition(const int32_t *mu, int64_t E, int Np, int64_t N, int rank, int world,
                               int64_t *sizes_out, int32_t *loc2glob_out, int32_t *nbr_out, int32_t *nbr_off_out,
                               int32_t *send_glob_out, int32_t *if_glob_out, int32_t *sum_start_out,
                               int32_t *sum_src_out);

/*
 * Host-only diagnostic (no GPU, no context): the reference-triangle tables the
 * library derives for `degree` (refelem.cpp; readings R3, R4, R21): *np_out = Np,
 * nodes_out [Np][2], wK_out / wM_out [Np] (stiffness / mass weights), Dr_out /
 * Ds_out [Np][Np] with Dr[k][p] = dN_p/dr at node k.  Any output may be NULL.
 * Errors: SEM_E_UNSUPPORTED (degree not in 2..7).
 */
sem_status sem_debug_ref_tables(int degree, int32_t *np_out, double *nodes_out, double *wK_out, double *wM_out,
                                double *Dr_out, double *Ds_out);

/*
 * Host-only diagnostic: the element stiffness factors the step kernel uses,
 * K^e = Grr Srr + Gss Sss + Grs Srs, as [Np][Np] each (nodal quadrature
 * D^T W D for P = 2, 3, 5, 7; exact integrals for P = 4, 6, reading R21b).
 * Errors: SEM_E_UNSUPPORTED.
 */
sem_status sem_debug_ref_stiffness(int degree, double *Srr_out, double *Sss_out, double *Srs_out);

/* Library version string. */
const char *sem_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SEM_H */
