// step.cu -- sm_100a kernels of the leapfrog step (product path).
//
//  K6  launch_geometry  G_e = c_e^2 detJ J^-1 J^-T (3 fp64), detJ
//      assemble_mass    M-bar_nu = sum detJ w^M_q, then dt^2 / M-bar
//  K7  launch_k7        persistent, warp-specialised: a producer warp streams
//                       each chunk's contiguous blocks into shared memory with
//                       TMA bulk copies (cp.async.bulk + mbarrier, 2 stages) and
//                       gathers U^n of the chunk's shared nodes (cp.async);
//                       B/32 consumer warps: (E) u_e gathered through the chunk's
//                       local index table, y_e = K^e u_e (one element per thread at
//                       P <= 5, G threads at P6/P7), written to the chunk's
//                       jagged-diagonal entry buffer; each element's own interior
//                       nodes are finalised by its thread; (B) node-centric sums of
//                       the entries in a fixed order fused with the leapfrog update
//                       of the chunk's interior nodes, partial sums of its shared
//                       nodes into their slots  (Alg. 1+2+3)
//  K8  launch_k8        shared nodes: add the slots in ascending chunk order,
//                       same fused update
//
// Element stiffness (readings R2, R5): K^e = Grr*Srr + Gss*Sss + Grs*Srs, with
// S_ab = D_a^T W D_b (+ transpose for rs) from the reference tables: the
// composition of Algorithm 1's gradient and Algorithm 2's
// weighted divergence with F = c^2 I, B = -I; the FK/BK
// precalculation is pushed into the reference
// matrices, as PAPER.md:1568 suggests.
#include <cuda_runtime.h>

#include <vector>

#include "dev_common.cuh"
#include "kernels.h"

namespace sem {

namespace {

constexpr int kThreads = 256;
#ifndef SEM_KSTAGES
#define SEM_KSTAGES 2
#endif
constexpr int kStages = SEM_KSTAGES;  // pipeline depth of K7 (A/B: -DSEM_KSTAGES=3)
// The producer reads the chunk's shared-node ids from a TMA copy in the stage (own
// mbarrier) instead of one dependent global load per cp.async gather (A/B: -DSEM_K7_IDS_TMA=0)
#ifndef SEM_K7_IDS_TMA
#define SEM_K7_IDS_TMA 1
#endif
constexpr bool kIdsTma = SEM_K7_IDS_TMA != 0;
// High orders (P5-P7, G > 1): the element products y = grr (Srr u) + gss (Sss u) + grs (Srs u)
// of a chunk are three dense [Np x Np] x [Np x B] contractions, run on the FP64 tensor cores
// (mma.sync m8n8k4 f64, SASS DMMA) instead of DFMA with one table read per two FMAs
// (A/B: -DSEM_K7_TC=0)
#ifndef SEM_K7_TC
#define SEM_K7_TC 1
#endif
constexpr bool kTcOn = SEM_K7_TC != 0;
__host__ __device__ constexpr bool k7_tc(int np, int g) { return kTcOn && g > 1 && np >= 21; }
__host__ __device__ constexpr int pad_to(int v, int m) { return (v + m - 1) / m * m; }

// D = A B + C for one 8x8x4 fp64 tile (per-thread fragments: A[lane / 4][lane % 4],
// B[lane % 4][lane / 4], C / D[lane / 4][2 (lane % 4) + i], i = 0, 1)
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// S tables packed densely for the current degree ([p * Np + q]): at P3 the three
// tables span 2.4 KB of the constant cache instead of rows strided by kMaxNp
__constant__ double c_Srr[kMaxNp * kMaxNp];
__constant__ double c_Sss[kMaxNp * kMaxNp];
__constant__ double c_Srs[kMaxNp * kMaxNp];
__constant__ double c_wM[kMaxNp];
// (Srr, Sss, Srs, 0) of the canonical mirror pairs (mirror_pair, sem_internal.h), P <= 5
__constant__ double c_mir[4 * kMirMax];

// One-thread-per-element K^e u (P3-P5) with the reflection symmetry of the reference triangle:
// pair (p, q) and its mirror (p', q') share their three factors (Srr_p'q' = Sss_pq,
// Sss_p'q' = Srr_pq, Srs_p'q' = Srs_pq), so each canonical pair reads 3 constants and forms
// grs Srs once for both K^e entries (A/B: -DSEM_K7_MIRROR=0).
#ifndef SEM_K7_MIRROR
#define SEM_K7_MIRROR 1
#endif
#ifndef SEM_K7_REV_TAIL
#define SEM_K7_REV_TAIL 1
#endif
template <int NP, int K>
__device__ __forceinline__ void mirror_products(double (&y)[NP], const double (&u)[NP], double grr, double gss,
                                                double grs) {
    constexpr MirrorTable<NP> T{};
    if constexpr (K < T.n) {
        constexpr int p = T.p[K], q = T.q[K], mp = T.mp[K], mq = T.mq[K];
        const double A = c_mir[4 * K], Bs = c_mir[4 * K + 1], Cs = c_mir[4 * K + 2];
        const double g = grs * Cs;
        const double k1 = fma(grr, A, fma(gss, Bs, g));
        if constexpr (p == q) {
            y[p] = fma(k1, u[p], y[p]);
        } else {
            y[p] = fma(k1, u[q], y[p]);
            y[q] = fma(k1, u[p], y[q]);
        }
        if constexpr (!(mp == p && mq == q)) {
            const double k2 = fma(grr, Bs, fma(gss, A, g));
            if constexpr (mp == mq) {
                y[mp] = fma(k2, u[mp], y[mp]);
            } else {
                y[mp] = fma(k2, u[mq], y[mp]);
                y[mq] = fma(k2, u[mp], y[mq]);
            }
        }
        mirror_products<NP, K + 1>(y, u, grr, gss, grs);
    }
}

// step index of U: from device memory when the step loop runs as a CUDA graph
// (one graph replays many steps; k_step_inc advances the counter), else the
// launch argument
__device__ __forceinline__ int64_t step_index(const StepParams &a) { return a.n_dev ? *a.n_dev : a.n; }

__global__ void k_step_inc(int64_t *n) {
    pdl_trigger();
    pdl_wait();
    *n += 1;
}
__global__ void k_step_set(int64_t *n, int64_t v) { *n = v; }

// One-GPU stand-in for the NCCL send/recv kernels of the interface exchange (overlap probe,
// SEM_OVERLAP_PROBE_US): a few small CTAs that hold their SM slots for `ns` nanoseconds.
__global__ void k_comm_standin(long long ns) {
    extern __shared__ unsigned char standin_smem[];  // the footprint of the kernel it stands in for
    if (threadIdx.x == 0) standin_smem[0] = 0;
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
        __nanosleep(500);
    }
}

inline unsigned blocks_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    return (unsigned)b;
}

// Shared-memory layout of one pipeline stage (all offsets 16-byte aligned).
// Lf = Ls when K8 is fused (slot counters), else 0; Ws = the U^{n-1} / dt^2/M
// window length when the windows travel in the stage (double-buffered with
// it), else 0 (single-buffered windows outside the stages).
struct StageLayout {
    int lidx, lpos, jds, shs, shn, scr, g, meta, u, up, m, size;
    __host__ __device__ StageLayout(int np, int B, int L, int Lp, int Ls, int Lf, int Ws) {
        lidx = 0;
        lpos = np * B * 2;
        jds = lpos + np * B * 2;
        shs = jds + Lp * 2;
        shn = shs + Ls * 4;
        scr = shn + (kIdsTma ? Ls : Lf) * 4;
        g = scr + Lf * 2;
        meta = g + 3 * B * 8;
        u = meta + 32;
        up = u + L * 8;
        m = up + Ws * 8;
        size = (m + Ws * 8 + 127) & ~127;
    }
};

__global__ void k_geometry(const double *__restrict__ vxy, const int32_t *__restrict__ tri,
                           const int32_t *__restrict__ perm, const double *__restrict__ c_in,
                           int64_t E, int64_t Epad, double *__restrict__ Grr,
                           double *__restrict__ Gss, double *__restrict__ Grs,
                           double *__restrict__ detJ, int32_t *bad) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= Epad) return;
    if (k >= E) { Grr[k] = 0.0; Gss[k] = 0.0; Grs[k] = 0.0; detJ[k] = 0.0; return; }
    const int64_t e = perm[k];
    const int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
    const double j00 = vxy[2 * v1] - vxy[2 * v0], j01 = vxy[2 * v2] - vxy[2 * v0];
    const double j10 = vxy[2 * v1 + 1] - vxy[2 * v0 + 1], j11 = vxy[2 * v2 + 1] - vxy[2 * v0 + 1];
    const double det = j00 * j11 - j01 * j10;
    const double c = c_in[e];
    if (!(det > 0.0)) atomicMin(bad, (int32_t)e);
    const double s = c * c / det;  // c^2 detJ / detJ^2
    Grr[k] = s * (j11 * j11 + j01 * j01);
    Gss[k] = s * (j10 * j10 + j00 * j00);
    Grs[k] = -s * (j11 * j10 + j01 * j00);
    detJ[k] = det;
}

// Sum of a local node's element contributions in the jagged-diagonal (JDS)
// entry buffer (chunks.cpp): jo = the node's segment's diagonal starts, end =
// end of that segment, ii = node index in the segment.  Diagonal d holds the
// d-th entry (ascending e = p*B + t) of every node with more than d entries;
// diagonal lengths do not increase with d.  The sum runs over d in order (a
// fixed order), and a warp's lanes read consecutive words of each diagonal.
// W = diagonals walked at most: 32 when no node of the mesh has more entries in a chunk (the
// common case; the 64-diagonal loop measured 4.5 % slower on C4's K7), else kJdsW.
template <int W = kJdsW>
__device__ __forceinline__ double jds_sum(const double *ebuf, const uint16_t *jo, int end, int ii) {
    double y = ebuf[jo[0] + ii];  // every local node has an entry
    for (int d = 1; d < W; d++) {
        const int nd = (d + 1 < kJdsW ? (int)jo[d + 1] : end) - (int)jo[d];
        if (ii >= nd) break;
        y += ebuf[jo[d] + ii];
    }
    return y;
}

// ---- lumped mass with the chunk machinery (one-time, not pipelined) -----------
template <int NP, int B>
__global__ void __launch_bounds__(B) k_mass_chunk(const DevChunks ch, const double *__restrict__ detJ,
                                                         double dt2, double *__restrict__ slot,
                                                         double *__restrict__ dt2M) {
    __shared__ double ybuf[NP * B];
    const int c = blockIdx.x, t = threadIdx.x;
    const int *cm = ch.cmeta + 8 * (int64_t)c;
    const int i0 = cm[0], nint = cm[1], s0 = cm[2], nsh = cm[3], ne = cm[5], ni_al = cm[6];
    const int64_t e = (int64_t)c * B + t;
    if (t < ne) {
        const double dj = detJ[e];
        const uint16_t *lpo = ch.lpos + (int64_t)c * NP * B;
#pragma unroll
        for (int p = 0; p < NP; p++) ybuf[lpo[p * B + t]] = 1.0 * dj * c_wM[p];
    }
    __syncthreads();
    const uint16_t *jd = ch.jds + (int64_t)c * 2 * kJdsW;
    for (int i = t; i < ni_al + nsh; i += B) {
        if (i < nint) dt2M[i0 + i] = dt2 / jds_sum(ybuf, jd, cm[4], i);
        else if (i >= ni_al) slot[ch.shl_slot[s0 + i - ni_al]] = jds_sum(ybuf, jd + kJdsW, cm[7], i - ni_al);
    }
}

__global__ void k_mass_fix(const DevChunks ch, const double *__restrict__ slot, double dt2,
                           double *__restrict__ dt2M) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ch.N_sh - ch.N_if) return;
    double m = 0.0;
    for (int j = ch.sh_pstart[s]; j < ch.sh_pstart[s + 1]; j++) m += slot[j];
    dt2M[ch.N_int + s] = dt2 / m;
}


// Fused K8 (shared nodes finalised by their last chunk): after writing its
// partial into slot `sl`, a chunk counts its arrival on the node's counter with
// an acq_rel atomic (release: the slot write is ordered before it; acquire: the
// last arriver sees every other chunk's slot).  The last arriver sums the
// node's slots in ascending chunk order -- the same order and association as
// k8_fix, so the result does not depend on which chunk finishes -- applies the
// update and resets the counter for the next step.  Rank-interface nodes stay
// with the exchange path.
__device__ __forceinline__ int atomic_add_acq_rel(int32_t *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// The leapfrog update U^{n+1} = 2 U^n - U^{n-1} + (dt^2/M) (f - (K U^n)) (north_star,
// reading R1), spelled with explicit roundings so every kernel that finalises a node
// (K7 element or node phase, K8, the interface and ablation kernels) yields the same bits.
__device__ __forceinline__ double leap_update(double u, double up, double m, double f, double y) {
#ifdef SEM_LEAP_PLAIN
    return 2.0 * u - up + m * (f - y);
#else
    return __fma_rn(m, __dsub_rn(f, y), __dsub_rn(__dmul_rn(2.0, u), up));
#endif
}

__device__ __forceinline__ void finish_shared(const DevChunks &ch, const StepParams &a, int32_t sg, uint16_t cr,
                                              int sl, double u) {
    if (sg >= ch.N_sh - ch.N_if) return;
    const int cnt = cr >> 8, rk = cr & 255;
    if (atomic_add_acq_rel(&a.cnt[sg], 1) != cnt - 1) return;
    const int j0 = sl - rk, j1 = j0 + cnt;
    double part[4];
#pragma unroll
    for (int d = 0; d < 4; d++) part[d] = (j0 + d < j1) ? __ldcg(&a.slot[j0 + d]) : 0.0;
    double y = part[0];
#pragma unroll
    for (int d = 1; d < 4; d++) y += part[d];
    for (int j = j0 + 4; j < j1; j++) y += __ldcg(&a.slot[j]);
    const int64_t id = ch.N_int + sg;
    const double f = (id == a.src) ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
    a.Uprev[id] = leap_update(u, a.Uprev[id], a.dt2M[id], f, y);
    a.cnt[sg] = 0;
}

// ---- K7 ---------------------------------------------------------------------------
// G > 1 (high orders): G consumer threads per element.  Warp w takes elements
// 32 (w / G) + lane and the row block w % G of y = K^e u, computed as
// y_p = grr (Srr u)_p + gss (Sss u)_p + grs (Srs u)_p with the S tables staged in
// shared memory (all lanes of a warp read the same entry: broadcast).
template <int NP, int B, int WM, int G = 1, int JW = 32>
__global__ void __launch_bounds__(B * G + 32, (G > 1 ? 1 : NP > 21 ? 1 : NP > 10 ? 2 : B <= 128 ? 4 : B <= 192 ? 3 : B <= 256 ? 2 : 1))
    k7_step(const DevChunks ch, const StepParams a, int L, int W, int Lp, int Ls,
            const int32_t *__restrict__ list, int64_t nlist) {
    constexpr int C = B * G;  // consumer threads
    constexpr int kNI = lattice_n_interior(NP);  // element-interior nodes per element
    // finalised by the element's thread (P3, P4; at P5 this measured 0.8 % slower, 168 registers)
    constexpr bool kInnerFin = G == 1 && kNI > 0 && NP < 21;
    extern __shared__ __align__(128) unsigned char sm[];
    // WM: U^{n-1} / dt^2/M windows -- 0 read from global in the node phase, 1 single-buffered
    // TMA window (default), 2 inside the double-buffered stages
    constexpr bool WIN2 = WM == 2, WIN1 = WM == 1;
    const StageLayout lay(NP, B, L, Lp, Ls, a.cnt ? Ls : 0, WIN2 ? W : 0);
    double *ebuf = reinterpret_cast<double *>(sm + kStages * lay.size);  // [NP][B] element slots
    double *up_w = ebuf + NP * B;                                       // U^{n-1} window (single buffer)
    double *m_w = up_w + (WIN1 ? W : 0);                                // dt^2/M window (single buffer)
    uint64_t *full = reinterpret_cast<uint64_t *>(m_w + (WIN1 ? W : 0));  // TMA blocks landed
    uint64_t *gath = full + kStages;                                    // shared-node gathers landed
    uint64_t *empty = gath + kStages;                                   // consumers done with stage
    uint64_t *wfull = empty + kStages;                                  // U^{n-1}, dt^2/M windows landed
    uint64_t *wempty = wfull + 1;                                       // ... consumed
    uint64_t *idb = wempty + 1;                                         // shared-node ids landed
    double *S_s = reinterpret_cast<double *>(idb + kStages);            // G > 1: Srr, Sss, Srs [NP][NP]
    const int t = threadIdx.x;
    const int64_t nch = list ? nlist : ch.nchunks;  // chunks this launch walks
    pdl_trigger();  // the next kernel (K8) may be scheduled; it waits for this grid to complete

    constexpr int kNPp = NP + (NP & 1);  // G > 1: S table rows padded to an even length (16-byte pairs)
    constexpr bool kTc = k7_tc(NP, G);
    constexpr int kMP = pad_to(NP, 8), kKP = pad_to(NP, 4);  // tensor-core tiles: rows to 8, columns to 4
    if (kTc) {  // Srr, Sss, Srs as [3][kMP][kKP], zero-padded (the A operands of the tile products)
        for (int i = t; i < 3 * kMP * kKP; i += blockDim.x) {
            const int tb = i / (kMP * kKP), r = (i / kKP) % kMP, q = i % kKP;
            const double *src = tb == 0 ? c_Srr : tb == 1 ? c_Sss : c_Srs;
            S_s[i] = (r < NP && q < NP) ? src[r * NP + q] : 0.0;
        }
    } else if (G > 1) {
        for (int i = t; i < NP * NP; i += blockDim.x) {
            const int p = i / NP, q = i % NP;
            S_s[p * kNPp + q] = c_Srr[i];
            S_s[NP * kNPp + p * kNPp + q] = c_Sss[i];
            S_s[2 * NP * kNPp + p * kNPp + q] = c_Srs[i];
        }
    }
    if (t == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&gath[s], 32);
            mbar_init(&empty[s], 1);
            mbar_init(&idb[s], 1);
        }
        mbar_init(wfull, 1);
        mbar_init(wempty, 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();  // graph step loop: the previous step's K8 / step counter are complete

    if (t >= C) {
        // ===== producer warp =====
        // lane 0 streams the chunk's contiguous blocks with TMA bulk copies; all
        // 32 lanes gather U^n of the chunk's shared nodes with cp.async.
        const int lane = t - C;
        int k = 0;
        for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
            const int64_t c = list ? list[pos] : pos;
            const int s = k % kStages;
            if (k >= kStages && lane == 0) mbar_wait(&empty[s], ((k / kStages) & 1) ^ 1);
            if (lane == 0) chaos_delay(0x10000u * blockIdx.x + 2u * k);
#ifdef SEM_INJECT_RACE
            if (lane == 0 && k >= kStages) __nanosleep(20000);  // a late refill the consumers do not wait for
#endif
            __syncwarp();
            unsigned char *st = sm + s * lay.size;
            const int4 m0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
            const int4 m1 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c + 1];
            const int i0 = m0.x, s0 = m0.z, nsh = m0.w, ni_al = m1.z;
            if (lane == 0) {
                reinterpret_cast<int4 *>(st + lay.meta)[0] = m0;
                reinterpret_cast<int4 *>(st + lay.meta)[1] = m1;
                const int nsh8 = (nsh + 7) & ~7;
                const bool fuse = a.cnt != nullptr;
                const uint32_t bytes = 2 * NP * B * 2 + 2 * kJdsW * 2 + nsh8 * (fuse ? (kIdsTma ? 6 : 10) : 4) +
                                       3 * B * 8 + (uint32_t)ni_al * (WIN2 ? 24 : 8);
                SEM_DCHECK(c >= 0 && c < ch.nchunks, "chunk id in range");
                SEM_DCHECK(ni_al + ((nsh + 1) & ~1) <= L, "local nodes fit the stage's u buffer");
                SEM_DCHECK(nsh8 <= Ls, "shared-node lists fit the stage");
                SEM_DCHECK(!(WIN1 || WIN2) || ni_al <= W, "interior window fits");
                SEM_DCHECK(i0 % 2 == 0 && i0 + ni_al <= ch.N_int + 1, "interior window inside the interior range");
                SEM_DCHECK(lay.meta + 32 <= lay.size && lay.u + L * 8 <= lay.size, "stage layout");
                if (kIdsTma) {  // first: the ids the gathers below wait for
                    mbar_arrive_expect_tx(&idb[s], nsh8 * 4);
                    if (nsh8 > 0) tma_load(st + lay.shn, ch.shl_node + s0, nsh8 * 4, &idb[s]);
                }
                mbar_arrive_expect_tx(&full[s], bytes);
                const int64_t e0 = c * B;
                tma_load(st + lay.lidx, ch.lidx + e0 * NP, NP * B * 2, &full[s]);
                tma_load(st + lay.lpos, ch.lpos + e0 * NP, NP * B * 2, &full[s]);
                tma_load(st + lay.jds, ch.jds + c * 2 * kJdsW, 2 * kJdsW * 2, &full[s]);
                if (nsh8 > 0) {
                    tma_load(st + lay.shs, ch.shl_slot + s0, nsh8 * 4, &full[s]);
                    if (fuse) {
                        if (!kIdsTma) tma_load(st + lay.shn, ch.shl_node + s0, nsh8 * 4, &full[s]);
                        tma_load(st + lay.scr, ch.shl_cr + s0, nsh8 * 2, &full[s]);
                    }
                }
                tma_load(st + lay.g, a.Grr + e0, B * 8, &full[s]);
                tma_load(st + lay.g + B * 8, a.Gss + e0, B * 8, &full[s]);
                tma_load(st + lay.g + 2 * B * 8, a.Grs + e0, B * 8, &full[s]);
                if (ni_al > 0) tma_load(st + lay.u, a.U + i0, ni_al * 8, &full[s]);
                if (WIN2 && ni_al > 0) {
                    tma_load(st + lay.up, a.Uprev + i0, ni_al * 8, &full[s]);
                    tma_load(st + lay.m, a.dt2M + i0, ni_al * 8, &full[s]);
                }
            }
            double *u_sh = reinterpret_cast<double *>(st + lay.u) + ni_al;
            if (kIdsTma) {
                __syncwarp();
                mbar_wait(&idb[s], (k / kStages) & 1);
                const int32_t *ids = reinterpret_cast<const int32_t *>(st + lay.shn);
                for (int j = lane; j < nsh; j += 32) cp_async8(u_sh + j, a.U + ch.N_int + ids[j]);
            } else {
                for (int j = lane; j < nsh; j += 32) cp_async8(u_sh + j, a.U + ch.N_int + ch.shl_node[s0 + j]);
            }
            cp_async_arrive_noinc(&gath[s]);
            // the single U^{n-1} / dt^2/M window buffer: free once the previous
            // chunk's update is done; lands while this chunk's element phase runs
            if (WIN1 && lane == 0) {
                if (k >= 1) mbar_wait(wempty, (k - 1) & 1);
                chaos_delay(0x10000u * blockIdx.x + 2u * k + 1u);
                mbar_arrive_expect_tx(wfull, (uint32_t)ni_al * 16);
                if (ni_al > 0) {
                    tma_load(up_w, a.Uprev + i0, ni_al * 8, wfull);
                    tma_load(m_w, a.dt2M + i0, ni_al * 8, wfull);
                }
            }
        }
        return;
    }

    // ===== consumer warps =====
    // the Ricker source term of this step (Alg. 3), once per thread instead of inline at every
    // finalising site (keeps the cold exp() code out of the element and node loops)
    const double fsrc = a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0);
    int k = 0;
    for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
        const int s = k % kStages;
#ifdef SEM_INJECT_RACE
        // the checked build's own pin (tools/checked_build.sh): consumers read reused stages
        // without waiting for their refill -- the poison and asserts must make this fail
        if (k < kStages)
#endif
        {
            MBAR_WAIT_INLINE(&full[s], (k / kStages) & 1);  // stage blocks (TMA)
            MBAR_WAIT_INLINE(&gath[s], (k / kStages) & 1);  // shared-node U gathers (cp.async)
        }
        // fused K8 reads the shared-node ids the idb copy wrote: wait on it directly rather than
        // through the producer's wait -> cp.async arrive chain (already complete: near free)
        if (kIdsTma && a.cnt) MBAR_WAIT_INLINE(&idb[s], (k / kStages) & 1);
        const unsigned char *st = sm + s * lay.size;
        const int4 m0 = reinterpret_cast<const int4 *>(st + lay.meta)[0];
        const int4 m1 = reinterpret_cast<const int4 *>(st + lay.meta)[1];
        const int i0 = m0.x, nint = m0.y, nsh = m0.w, ne = m1.y, ni_al = m1.z;
        const double *u_s = reinterpret_cast<const double *>(st + lay.u);
        const uint16_t *li_s = reinterpret_cast<const uint16_t *>(st + lay.lidx);
        const uint16_t *lpo = reinterpret_cast<const uint16_t *>(st + lay.lpos);
        const uint16_t *jd = reinterpret_cast<const uint16_t *>(st + lay.jds);
        const int end0 = m1.x, end1 = m1.w;
        const int32_t *shs = reinterpret_cast<const int32_t *>(st + lay.shs);
        const double *g_s = reinterpret_cast<const double *>(st + lay.g);
        if (kChecked) {  // the stage holds this chunk (a stale or foreign stage fails here)
            const int64_t c = list ? list[pos] : pos;
            const int4 r0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
            const int4 r1 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c + 1];
            SEM_DCHECK(r0.x == m0.x && r0.y == m0.y && r0.z == m0.z && r0.w == m0.w && r1.x == m1.x &&
                           r1.y == m1.y && r1.z == m1.z && r1.w == m1.w,
                       "stage meta is this chunk's");
            SEM_DCHECK(ne > 0 && ne <= B && end0 <= end1 && end1 <= NP * B, "chunk shape");
            for (int e = t; e < NP * ne; e += C) {
                const int q = e / ne, te = e % ne, li = li_s[q * B + te];
                SEM_DCHECK(li < nint || (li >= ni_al && li < ni_al + nsh), "local index in range (poisoned?)");
                SEM_DCHECK(lpo[q * B + te] < end1, "entry position in range (poisoned?)");
            }
            for (int j = t; j < nsh; j += C) SEM_DCHECK(shs[j] >= 0 && shs[j] < ch.n_slots, "slot id in range");
        }

        if (kTc) {
            // (E, tensor cores) warp wi takes the element tiles nt = wi, wi + C/32, ... of 8 elements
            // each; per tile the three products over k-steps of 4 nodes, then the G_e combination
            constexpr int MT = kMP / 8, KT = kKP / 4, NT = B / 8;
            const int lane = t & 31;
            for (int nt = t >> 5; nt < NT; nt += C / 32) {
                const int eb = nt * 8 + (lane >> 2);  // element of this lane's B-fragment column
                double acc[MT][3][2];
#pragma unroll
                for (int m = 0; m < MT; m++)
#pragma unroll
                    for (int tb = 0; tb < 3; tb++) acc[m][tb][0] = acc[m][tb][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KT; ks++) {
                    const int q = ks * 4 + (lane & 3);
                    const double b = (q < NP && eb < ne) ? u_s[li_s[q * B + eb]] : 0.0;
#pragma unroll
                    for (int m = 0; m < MT; m++)
#pragma unroll
                        for (int tb = 0; tb < 3; tb++)
                            dmma_8x8x4(acc[m][tb][0], acc[m][tb][1], S_s[(tb * kMP + m * 8 + (lane >> 2)) * kKP + q], b);
                }
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const int e = nt * 8 + 2 * (lane & 3) + i;
                    if (e < ne) {
                        const double grr = g_s[e], gss = g_s[B + e], grs = g_s[2 * B + e];
#pragma unroll
                        for (int m = 0; m < MT; m++) {
                            const int p = m * 8 + (lane >> 2);
                            if (p < NP) ebuf[lpo[p * B + e]] = fma(grr, acc[m][0][i], fma(gss, acc[m][1][i], grs * acc[m][2][i]));
                        }
                    }
                }
            }
        } else if (G > 1) {
            // (E, wide) this thread: element te, rows [p0, p1) of y = K^e u
            constexpr int R = (NP + G - 1) / G;
            const int w = t >> 5, te = ((w / G) << 5) + (t & 31), p0 = (w % G) * R;
            if (te < ne) {
                const double grr = g_s[te], gss = g_s[B + te], grs = g_s[2 * B + te];
                double u[NP];
#pragma unroll
                for (int q = 0; q < NP; q++) u[q] = u_s[li_s[q * B + te]];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const int p = p0 + r;
                    if (p < NP) {
                        const double *srr = S_s + p * kNPp, *sss = srr + NP * kNPp, *srs = sss + NP * kNPp;
                        double arr = 0.0, ass = 0.0, ars = 0.0;
#pragma unroll
                        for (int q = 0; q < NP; q += 2) {  // one 16-byte broadcast read per table and q pair
                            const double2 a2 = *reinterpret_cast<const double2 *>(srr + q);
                            const double2 b2 = *reinterpret_cast<const double2 *>(sss + q);
                            const double2 c2 = *reinterpret_cast<const double2 *>(srs + q);
                            arr = fma(a2.x, u[q], arr);
                            ass = fma(b2.x, u[q], ass);
                            ars = fma(c2.x, u[q], ars);
                            if (q + 1 < NP) {
                                arr = fma(a2.y, u[q + 1], arr);
                                ass = fma(b2.y, u[q + 1], ass);
                                ars = fma(c2.y, u[q + 1], ars);
                            }
                        }
                        ebuf[lpo[p * B + te]] = fma(grr, arr, fma(gss, ass, grs * ars));
                    }
                }
            }
        }
        // (E) y = K^e u, K^e symmetric: each K_pq (p <= q) built once
        double y[NP];
#pragma unroll
        for (int p = 0; p < NP; p++) y[p] = 0.0;
        if (G == 1 && t < ne) {
            const double grr = g_s[t], gss = g_s[B + t], grs = g_s[2 * B + t];
            double u[NP];
#pragma unroll
            for (int p = 0; p < NP; p++) u[p] = u_s[li_s[p * B + t]];
            if constexpr (SEM_K7_MIRROR != 0 && NP >= 10 && NP <= 21) {  // P2: 66 -> 76 registers cost its third CTA per SM (C5/4 0.447 -> 0.546 ms)
                mirror_products<NP, 0>(y, u, grr, gss, grs);
            } else {
#pragma unroll
            for (int p = 0; p < NP; p++) {
#pragma unroll
                for (int q = p; q < NP; q++) {
                    const double kk = fma(grr, c_Srr[p * NP + q], fma(gss, c_Sss[p * NP + q], grs * c_Srs[p * NP + q]));
                    if (q == p) {
                        y[p] = fma(kk, u[p], y[p]);
                    } else {
                        y[p] = fma(kk, u[q], y[p]);
                        y[q] = fma(kk, u[p], y[q]);
                    }
                }
            }
            }
        }
        const double *up_s = WIN2 ? reinterpret_cast<const double *>(st + lay.up) : up_w;
        const double *m_s = WIN2 ? reinterpret_cast<const double *>(st + lay.m) : m_w;
        double *Unew = a.Uprev;
        // Element-interior nodes (lattice interior of the element, e.g. the P3 centroid) have one
        // entry, and the chunk builder places them last in the interior segment: the node phase
        // covers [0, nint - ne * kNI) and each element's thread finalises its own interior nodes
        // after the barrier (with the U^{n-1} / dt^2/M window); their K U is y_e[p] alone.
        const int nint_np = nint - (kInnerFin ? ne * kNI : 0);  // interior nodes left to the node phase
        if (G == 1 && t < ne) {
#pragma unroll
            for (int p = 0; p < NP; p++)
                if (!(kInnerFin && lattice_interior(NP, p))) ebuf[lpo[p * B + t]] = y[p];  // the node's JDS entry
        }
        consumer_sync<C>();
        if (WIN1) MBAR_WAIT_INLINE(wfull, k & 1);  // U^{n-1} / dt^2/M window
        if (kInnerFin && t < ne) {
#pragma unroll
            for (int p = 0; p < NP; p++) {
                if (!lattice_interior(NP, p)) continue;
                const int li = li_s[p * B + t];
                const int id = i0 + li;
                const double up = WM == 0 ? a.Uprev[id] : up_s[li];
                const double m = WM == 0 ? __ldg(a.dt2M + id) : m_s[li];
                Unew[id] = leap_update(u_s[li], up, m, id == a.src ? fsrc : 0.0, y[p]);
            }
        }
        // (B) node-centric gather of K U^n in fixed order + fused update;
        //     shared nodes: this chunk's partial into the node's slot.  Work item w:
        //     interior node w < nint_np, else shared node ni_al + (w - nint_np) (skips
        //     the element-interior nodes and the alignment hole)
        const int nwork = nint_np + nsh;
        // P3: the work items are sorted by entry count (the vertex nodes' six-entry sums first), so
        // the threads that drew them in the first round skip the last, partial round: it is taken
        // in reverse thread order (C4 0.3835 -> 0.3724 ms per step, C3 0.1923 -> 0.1881 ms; at P2
        // and P5 it measured 1-2 % slower; A/B: -DSEM_K7_REV_TAIL=0).
        constexpr bool kRevTail = SEM_K7_REV_TAIL != 0 && NP == 10;
        const int nfull = kRevTail ? nwork / C * C : nwork;
        for (int w0 = 0; w0 < nwork; w0 += C) {
            const int w = w0 + (w0 >= nfull ? C - 1 - t : t);
            if (w >= nwork) continue;
            const int i = w < nint_np ? w : ni_al + (w - nint_np);
            double upg = 0.0, mg = 0.0;
            if (WM == 0 && i < nint) {  // coalesced global loads, issued before the shared-memory sum
                upg = a.Uprev[i0 + i];
                mg = __ldg(a.dt2M + i0 + i);
            }
            const double yi = i < nint ? jds_sum<JW>(ebuf, jd, end0, i) : jds_sum<JW>(ebuf, jd + kJdsW, end1, i - ni_al);
            if (i < nint) {
                const int id = i0 + i;
                Unew[id] = leap_update(u_s[i], WM == 0 ? upg : up_s[i], WM == 0 ? mg : m_s[i], id == a.src ? fsrc : 0.0, yi);
            } else {
                const int j = i - ni_al;
                const int sl = shs[j];
                a.slot[sl] = yi;
                if (a.cnt) finish_shared(ch, a, reinterpret_cast<const int32_t *>(st + lay.shn)[j],
                                         reinterpret_cast<const uint16_t *>(st + lay.scr)[j], sl, u_s[i]);
            }
        }
        consumer_sync<C>();
        if (kChecked) {  // poison everything handed back: only a refill may be read after this
            unsigned char *stw = sm + s * lay.size;
            double *uw = reinterpret_cast<double *>(stw + lay.u);
            double *gw = reinterpret_cast<double *>(stw + lay.g);
            uint16_t *lw = reinterpret_cast<uint16_t *>(stw + lay.lidx);
            for (int i = t; i < ni_al + nsh; i += C) uw[i] = poison_f64();
            for (int i = t; i < 3 * B; i += C) gw[i] = poison_f64();
            for (int i = t; i < 2 * NP * B; i += C) lw[i] = 0xFFFF;  // lidx and lpos
            for (int i = t; i < end1; i += C) ebuf[i] = poison_f64();
            if (WIN1)
                for (int i = t; i < ni_al; i += C) { up_w[i] = poison_f64(); m_w[i] = poison_f64(); }
            consumer_sync<C>();
            if (t == 0) chaos_delay(0x20000u * blockIdx.x + k);
        }
        if (t == 0) {
            mbar_arrive(&empty[s]);
            if (WIN1) mbar_arrive(wempty);
        }
    }
}

// ---- K8: shared-node fix-up --------------------------------------------------
__global__ void k8_fix(const DevChunks ch, const StepParams a) {
    pdl_trigger();
    pdl_wait();
    const int64_t blk = a.k8_rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int64_t s = blk * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ch.N_sh - ch.N_if) return;  // interface nodes: k_if_partial / k8_if
    const int j0 = ch.sh_pstart[s], j1 = ch.sh_pstart[s + 1];
    SEM_DCHECK(j0 >= 0 && j0 < j1 && j1 <= ch.n_slots, "slot run of a shared node");
    const int64_t id = ch.N_int + s;
    const double u = a.U[id], up = a.Uprev[id], m = a.dt2M[id];  // independent of the slots
    double part[4];
#pragma unroll
    for (int d = 0; d < 4; d++) part[d] = (j0 + d < j1) ? a.slot[j0 + d] : 0.0;
    double y = part[0];  // contiguous slots, ascending chunk order
#pragma unroll
    for (int d = 1; d < 4; d++) y += part[d];
    for (int j = j0 + 4; j < j1; j++) y += a.slot[j];
    const double f = (id == a.src) ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
    a.Uprev[id] = leap_update(u, up, m, f, y);
}

// K8 with two consecutive shared nodes per thread (the default): the three slot-run bounds and
// both nodes' U^n / U^{n-1} / dt^2/M loads are issued before any slot is read, so a thread keeps
// twice the independent loads in flight; the same sums in the same order per node as k8_fix
// (identical bits).  C4: K8 0.0307 -> 0.0275 ms (profiles/r2s4_k8_ab.md).
__global__ void k8_fix2(const DevChunks ch, const StepParams a) {
    pdl_trigger();
    pdl_wait();
    const int64_t nsh = ch.N_sh - ch.N_if;
    const int64_t blk = a.k8_rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int64_t s = 2 * (blk * (int64_t)blockDim.x + threadIdx.x);
    if (s >= nsh) return;  // interface nodes: k_if_partial / k8_if
    const bool two = s + 1 < nsh;
    const int j0 = ch.sh_pstart[s], j1 = ch.sh_pstart[s + 1], j2 = two ? ch.sh_pstart[s + 2] : j1;
    SEM_DCHECK(j0 >= 0 && j0 < j1 && (!two || j1 < j2) && j2 <= ch.n_slots, "slot run of a shared node");
    const int64_t id = ch.N_int + s;
    const double u0 = a.U[id], up0 = a.Uprev[id], m0 = a.dt2M[id];
    double u1 = 0.0, up1 = 0.0, m1 = 0.0;
    if (two) { u1 = a.U[id + 1]; up1 = a.Uprev[id + 1]; m1 = a.dt2M[id + 1]; }
    double p0[4], p1[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        p0[d] = (j0 + d < j1) ? a.slot[j0 + d] : 0.0;
        p1[d] = (j1 + d < j2) ? a.slot[j1 + d] : 0.0;
    }
    double y0 = p0[0], y1 = p1[0];  // contiguous slots, ascending chunk order
#pragma unroll
    for (int d = 1; d < 4; d++) { y0 += p0[d]; y1 += p1[d]; }
    for (int j = j0 + 4; j < j1; j++) y0 += a.slot[j];
    for (int j = j1 + 4; j < j2; j++) y1 += a.slot[j];
    const bool hs = id == a.src || id + 1 == a.src;
    const double fs = hs ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
    a.Uprev[id] = leap_update(u0, up0, m0, id == a.src ? fs : 0.0, y0);
    if (two) a.Uprev[id + 1] = leap_update(u1, up1, m1, id + 1 == a.src ? fs : 0.0, y1);
}

// K8 with NPT consecutive shared nodes per thread (SEM_K8_NPT=4, A/B): the k8_fix2 scheme for
// any NPT (same sums, same order per node).
template <int NPT>
__global__ void k8_fixn(const DevChunks ch, const StepParams a) {
    pdl_trigger();
    pdl_wait();
    const int64_t nsh = ch.N_sh - ch.N_if;
    const int64_t blk = a.k8_rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
    const int64_t s = NPT * (blk * (int64_t)blockDim.x + threadIdx.x);
    if (s >= nsh) return;  // interface nodes: k_if_partial / k8_if
    const int nn = nsh - s < NPT ? (int)(nsh - s) : NPT;  // nodes of this thread
    int j[NPT + 1];
    j[0] = ch.sh_pstart[s];
#pragma unroll
    for (int q = 1; q <= NPT; q++) j[q] = q <= nn ? ch.sh_pstart[s + q] : j[q - 1];
    const int64_t id = ch.N_int + s;
    double u[NPT], up[NPT], m[NPT];
#pragma unroll
    for (int q = 0; q < NPT; q++) {
        SEM_DCHECK(q >= nn || (j[q] >= 0 && j[q] < j[q + 1] && j[q + 1] <= ch.n_slots), "slot run of a shared node");
        u[q] = q < nn ? a.U[id + q] : 0.0;
        up[q] = q < nn ? a.Uprev[id + q] : 0.0;
        m[q] = q < nn ? a.dt2M[id + q] : 0.0;
    }
    double y[NPT];
#pragma unroll
    for (int q = 0; q < NPT; q++) {
        double part[4];
#pragma unroll
        for (int d = 0; d < 4; d++) part[d] = (j[q] + d < j[q + 1]) ? a.slot[j[q] + d] : 0.0;
        y[q] = part[0];  // contiguous slots, ascending chunk order
#pragma unroll
        for (int d = 1; d < 4; d++) y[q] += part[d];
    }
#pragma unroll
    for (int q = 0; q < NPT; q++)
        for (int k = j[q] + 4; k < j[q + 1]; k++) y[q] += a.slot[k];
    const bool hs = a.src >= id && a.src < id + nn;
    const double fs = hs ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
#pragma unroll
    for (int q = 0; q < NPT; q++)
        if (q < nn) a.Uprev[id + q] = leap_update(u[q], up[q], m[q], id + q == a.src ? fs : 0.0, y[q]);
}

// ---- multi-GPU interface -----------------------------------------
// This rank's partial of interface node i = its slots summed in chunk order.
__global__ void k_if_partial(const DevChunks ch, const double *__restrict__ slot, double *__restrict__ xbuf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ch.N_if) return;
    const int64_t s = ch.N_sh - ch.N_if + i;
    double y = 0.0;
    for (int j = ch.sh_pstart[s]; j < ch.sh_pstart[s + 1]; j++) y += slot[j];
    xbuf[i] = y;
}

__global__ void k_pack(const double *__restrict__ xbuf, const int32_t *__restrict__ send_if, int64_t n,
                       double *__restrict__ sendbuf) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) sendbuf[k] = xbuf[send_if[k]];
}

// All ranks' partials of interface node i, added in ascending rank order, then
// the fused update (identical bits on every rank holding the node).
__global__ void k8_if(const DevChunks ch, const StepParams a, const double *__restrict__ xbuf,
                      const int32_t *__restrict__ sum_start, const int32_t *__restrict__ sum_src) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ch.N_if) return;
    double y = 0.0;
    for (int j = sum_start[i]; j < sum_start[i + 1]; j++) y += xbuf[sum_src[j]];
    const int64_t s = ch.N_sh - ch.N_if + i;
    const int64_t id = ch.N_int + s;
    const double f = (id == a.src) ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
    a.Uprev[id] = leap_update(a.U[id], a.Uprev[id], a.dt2M[id], f, y);
}

__global__ void k_mass_if(const DevChunks ch, const double *__restrict__ xbuf, const int32_t *__restrict__ sum_start,
                          const int32_t *__restrict__ sum_src, double dt2, double *__restrict__ dt2M) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ch.N_if) return;
    double m = 0.0;
    for (int j = sum_start[i]; j < sum_start[i + 1]; j++) m += xbuf[sum_src[j]];
    dt2M[ch.N_int + ch.N_sh - ch.N_if + i] = dt2 / m;
}

__global__ void k_permute_f64(const double *__restrict__ in, const int32_t *__restrict__ imap,
                              const int32_t *__restrict__ omap, int64_t n, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[omap ? omap[i] : i] = in[imap ? imap[i] : i];
}

__global__ void k_positive(const double *__restrict__ a, int64_t n, int32_t *first) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !(a[i] > 0.0 && isfinite(a[i]))) atomicMin(first, (int32_t)i);
}

__global__ void k_nonfinite(const double *__restrict__ a, int64_t n, int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !isfinite(a[i])) atomicMin(flag, (int32_t)i);
}

// ---- NEXT-4 ablation scatters (the rejected alternatives of SURVEY §8a K7) -----------
// One thread per element: u gathered straight from global U through mu (internal
// numbering), y = K^e u as in K7, then either fp64 atomicAdd into KU (order of
// the additions not fixed) or, for the paper's global element colouring
// (PAPER.md:516), a plain read-modify-write: one launch per colour, elements of
// a colour share no node.
template <int NP, bool ATOMIC>
__global__ void __launch_bounds__(256) k_abl_elem(const int32_t *__restrict__ mu, const int32_t *__restrict__ eidx,
                                                  int64_t e0, int64_t e1, const StepParams a, double *KU) {
    const int64_t k = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= e1) return;
    const int64_t e = eidx ? eidx[k] : k;  // element (product order) for G
    const double grr = a.Grr[e], gss = a.Gss[e], grs = a.Grs[e];
    int32_t g[NP];
    double u[NP], y[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) { g[p] = mu[k * NP + p]; u[p] = a.U[g[p]]; y[p] = 0.0; }
#pragma unroll
    for (int p = 0; p < NP; p++) {
#pragma unroll
        for (int q = p; q < NP; q++) {
            const double kk = fma(grr, c_Srr[p * NP + q], fma(gss, c_Sss[p * NP + q], grs * c_Srs[p * NP + q]));
            if (q == p) {
                y[p] = fma(kk, u[p], y[p]);
            } else {
                y[p] = fma(kk, u[q], y[p]);
                y[q] = fma(kk, u[p], y[q]);
            }
        }
    }
#pragma unroll
    for (int p = 0; p < NP; p++) {
        if (ATOMIC) atomicAdd(&KU[g[p]], y[p]);
        else KU[g[p]] += y[p];
    }
}

// Leapfrog update of every node from the assembled KU; KU reset for the next step.
__global__ void k_abl_update(int64_t n, const StepParams a, double *KU) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double f = (i == a.src) ? a.amp * ricker_dev((double)step_index(a) * a.dt, a.f0, a.t0) : 0.0;
    const double y = KU[i];
    KU[i] = 0.0;
    a.Uprev[i] = leap_update(a.U[i], a.Uprev[i], a.dt2M[i], f, y);
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return raise_max_smem((const void *)kernel, bytes);
}

// U^{n-1} / dt^2/M windows: SEM_K7_WIN=1 single-buffered TMA window (default),
// 2 inside the double-buffered stages, 0 plain global loads in the node phase
int k7_win() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("SEM_K7_WIN"); v = e ? atoi(e) : 1; if (v < 0 || v > 2) v = 1; }
    return v;
}

// consumer threads per element of the K7 instantiation used for np (1, or 4 at P7)
int k7_group(int np) {
    static int g7 = -1, g5 = -1;
    if (g7 < 0) { const char *e = getenv("SEM_K7_G"); g7 = e ? atoi(e) : 4; if (g7 != 1 && g7 != 2 && g7 != 4) g7 = 4; }
    // P5: one thread per element with the symmetric K^e build (B1 0.202 ms per step; the tensor-core
    // path with 2 threads per element: 0.264 ms); SEM_K7_G5=2|4 selects the wide / tensor-core one
    if (g5 < 0) { const char *e = getenv("SEM_K7_G5"); g5 = e ? atoi(e) : 1; if (g5 != 1 && g5 != 2 && g5 != 4) g5 = 1; }
    return (np == 36 || np == 28) ? g7 : np == 21 ? g5 : 1;
}

// window mode of the instantiation: meshes with a node of more than 32 entries in a chunk (wide
// JDS) run the default single-buffered window only
int k7_mode(bool wide) { return wide ? 1 : k7_win(); }
size_t k7_smem_bytes(int np, int B, int L, int W, int Lp, int Ls, bool fuse, bool wide) {
    const int wm = k7_mode(wide);
    const StageLayout lay(np, B, L, Lp, Ls, fuse ? Ls : 0, wm == 2 ? W : 0);
    const int g = k7_group(np);
    const size_t stab = k7_tc(np, g) ? 3 * (size_t)pad_to(np, 8) * pad_to(np, 4) * 8
                        : g > 1    ? 3 * (size_t)np * (np + (np & 1)) * 8
                                   : 0;
    return (size_t)kStages * lay.size + (size_t)np * B * 8 + (wm == 1 ? 2 * (size_t)W * 8 : 0) +
           (4 * kStages + 2) * 8 + stab;
}

using K7Fn = void (*)(const DevChunks, const StepParams, int, int, int, int, const int32_t *, int64_t);
template <int W2, int JW>
K7Fn k7_fn_w(int np, int B) {
    if (np == 15) return k7_step<15, 128, W2, 1, JW>;  // P4 (R21b): chunks of 128
    if (np == 21) {  // P5 (R21): chunks of 128
        const int g = k7_group(21);
        return g == 4 ? k7_step<21, 128, W2, 4, JW> : g == 2 ? k7_step<21, 128, W2, 2, JW> : k7_step<21, 128, W2, 1, JW>;
    }
    if (np == 28) {                              // P6 (R21b): chunks of 64, G threads per element
        const int g = k7_group(28);
        return g == 4 ? k7_step<28, 64, W2, 4, JW> : g == 2 ? k7_step<28, 64, W2, 2, JW> : k7_step<28, 64, W2, 1, JW>;
    }
    if (np == 36) {                              // P7: chunks of 64, G threads per element
        const int g = k7_group(36);
        return g == 4 ? k7_step<36, 64, W2, 4, JW> : g == 2 ? k7_step<36, 64, W2, 2, JW> : k7_step<36, 64, W2, 1, JW>;
    }
    if (np == 6)
        return B == 128   ? k7_step<6, 128, W2, 1, JW>
               : B == 192 ? k7_step<6, 192, W2, 1, JW>
               : B == 512 ? k7_step<6, 512, W2, 1, JW>
                          : k7_step<6, 256, W2, 1, JW>;
    return B == 128   ? k7_step<10, 128, W2, 1, JW>
           : B == 192 ? k7_step<10, 192, W2, 1, JW>
           : B == 512 ? k7_step<10, 512, W2, 1, JW>
                      : k7_step<10, 256, W2, 1, JW>;
}

// wide: a node of the mesh has more than 32 entries in one chunk -> the 64-diagonal JDS walk
K7Fn k7_fn(int np, int B, bool wide) {
    if (wide) return k7_fn_w<1, kJdsW>(np, B);
    const int wm = k7_win();
    return wm == 2 ? k7_fn_w<2, 32>(np, B) : wm == 0 ? k7_fn_w<0, 32>(np, B) : k7_fn_w<1, 32>(np, B);
}

}  // namespace

cudaError_t upload_ref_tables(const RefTables &T, cudaStream_t s) {
    cudaError_t e;
    // pageable source: the copies return once the data is staged, so the packed
    // buffers may go out of scope
    const int n = T.Np;
    std::vector<double> rr(n * n), ss(n * n), rs(n * n);
    for (int p = 0; p < n; p++)
        for (int q = 0; q < n; q++) { rr[p * n + q] = T.Srr[p][q]; ss[p * n + q] = T.Sss[p][q]; rs[p * n + q] = T.Srs[p][q]; }
    if ((e = cudaMemcpyToSymbolAsync(c_Srr, rr.data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Sss, ss.data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Srs, rs.data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if (n <= 21) {  // the canonical mirror pairs of the one-thread K7 (P <= 5)
        static constexpr MirrorTable<6> t6{};
        static constexpr MirrorTable<10> t10{};
        static constexpr MirrorTable<15> t15{};
        static constexpr MirrorTable<21> t21{};
        static_assert(t21.n <= kMirMax, "mirror pairs fit c_mir");
        const int cnt = n == 6 ? t6.n : n == 10 ? t10.n : n == 15 ? t15.n : t21.n;
        const int *tp = n == 6 ? t6.p : n == 10 ? t10.p : n == 15 ? t15.p : t21.p;
        const int *tq = n == 6 ? t6.q : n == 10 ? t10.q : n == 15 ? t15.q : t21.q;
        std::vector<double> mir(4 * kMirMax, 0.0);
        for (int k = 0; k < cnt; k++) {
            const int p = tp[k], q = tq[k];
            mir[4 * k] = T.Srr[p][q];
            mir[4 * k + 1] = T.Sss[p][q];
            mir[4 * k + 2] = T.Srs[p][q];
        }
        if ((e = cudaMemcpyToSymbolAsync(c_mir, mir.data(), sizeof(double) * 4 * kMirMax, 0, cudaMemcpyHostToDevice, s)))
            return e;
        // Host copies above are pageable: the call returns once staged, so `mir` may go out of scope.
    }
    return cudaMemcpyToSymbolAsync(c_wM, T.wM, sizeof(T.wM), 0, cudaMemcpyHostToDevice, s);
}

cudaError_t launch_geometry(const double *vxy, const int32_t *tri_or_in, const int32_t *perm,
                            const double *c_in, int64_t E, int64_t Epad, double *Grr,
                            double *Gss, double *Grs, double *detJ, int32_t *bad,
                            cudaStream_t s) {
    k_geometry<<<blocks_for(Epad), kThreads, 0, s>>>(vxy, tri_or_in, perm, c_in, E, Epad, Grr, Gss,
                                                     Grs, detJ, bad);
    return cudaGetLastError();
}

cudaError_t assemble_mass(const DevChunks &ch, const double *detJ, double numer, double *slot,
                          double *dt2M, cudaStream_t s) {
    const double dt2 = numer;
    cudaError_t e;
    if ((e = cudaMemsetAsync(dt2M, 0, sizeof(double) * (ch.N_tot + 2), s))) return e;
#define MASS(NP_, B_) k_mass_chunk<NP_, B_><<<(unsigned)ch.nchunks, B_, 0, s>>>(ch, detJ, dt2, slot, dt2M)
    if (ch.Np == 15) {
        MASS(15, 128);
    } else if (ch.Np == 21) {
        if (ch.B == 32) MASS(21, 32); else if (ch.B == 64) MASS(21, 64); else MASS(21, 128);
    } else if (ch.Np == 28) {
        MASS(28, 64);
    } else if (ch.Np == 36) {
        if (ch.B == 32) MASS(36, 32); else MASS(36, 64);
    } else if (ch.Np == 6) {
        if (ch.B == 128) MASS(6, 128); else if (ch.B == 192) MASS(6, 192); else if (ch.B == 512) MASS(6, 512); else MASS(6, 256);
    } else {
        if (ch.B == 128) MASS(10, 128); else if (ch.B == 192) MASS(10, 192); else if (ch.B == 512) MASS(10, 512); else MASS(10, 256);
    }
#undef MASS
    if (ch.N_sh - ch.N_if > 0) k_mass_fix<<<blocks_for(ch.N_sh - ch.N_if), kThreads, 0, s>>>(ch, slot, dt2, dt2M);
    return cudaGetLastError();
}

int k7_ctas_per_sm(int np, int B, int max_local, int max_win, int max_nsh, bool fused, int max_count) {
    const bool wide = max_count > 32;
    const size_t smem = k7_smem_bytes(np, B, max_local, max_win, 2 * kJdsW, max_nsh, fused, wide);
    const K7Fn fn = k7_fn(np, B, wide);
    set_smem(fn, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, B * k7_group(np) + 32, smem);
    return occ < 1 ? 1 : occ;
}

bool k7_fits(const DevChunks &ch, bool fused) {
    const bool wide = ch.max_count > 32;
    const size_t smem = k7_smem_bytes(ch.Np, ch.B, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, fused, wide);
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return false;
    // SEM_K7_SMEM_CAP (bytes, tests): a smaller budget than the device's, to exercise the fallback
    const char *cap = getenv("SEM_K7_SMEM_CAP");
    if (cap && atol(cap) > 0 && atol(cap) < optin) optin = (int)atol(cap);
    return smem <= (size_t)optin;
}

int k7_grid(const DevChunks &ch, bool fused, int reserve_sms) {
    const int occ = k7_ctas_per_sm(ch.Np, ch.B, ch.max_local, ch.max_win, ch.max_nsh, fused, ch.max_count);
    const int nsm = current_sm_count();
    if (reserve_sms >= nsm) reserve_sms = nsm - 1;
    int64_t g = (int64_t)occ * (nsm - (reserve_sms > 0 ? reserve_sms : 0));
    if (persistent_grid_cap() > 0 && g > persistent_grid_cap()) g = persistent_grid_cap();
    if (g > ch.nchunks) g = ch.nchunks;
    return (int)g;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*fn)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, bool pdl,
                      Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, args...);
}

cudaError_t launch_k7(const DevChunks &ch, const StepParams &p, int grid, cudaStream_t s,
                      const int32_t *list, int64_t nlist, bool pdl) {
    const int64_t n = list ? nlist : ch.nchunks;
    if (n == 0) return cudaSuccess;
    if (persistent_grid_cap() > 0 && grid > persistent_grid_cap()) grid = (int)persistent_grid_cap();
    if (grid > n) grid = (int)n;
    const bool wide = ch.max_count > 32;
    const size_t smem = k7_smem_bytes(ch.Np, ch.B, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, p.cnt != nullptr, wide);
    const K7Fn fn = k7_fn(ch.Np, ch.B, wide);
    cudaError_t e = set_smem(fn, smem);
    if (e != cudaSuccess) return e;
    return launch_ex(fn, (unsigned)grid, ch.B * k7_group(ch.Np) + 32, smem, s, pdl, ch, p, ch.max_local, ch.max_win,
                     2 * kJdsW, ch.max_nsh, list, nlist);
}

cudaError_t launch_k8(const DevChunks &ch, const StepParams &p, cudaStream_t s, bool pdl) {
    if (ch.N_sh - ch.N_if == 0) return cudaSuccess;
    // threads per K8 block: 128 (C4 K8 0.0403 -> 0.0393 ms against 256; 64: 0.0655, 512: 0.0410,
    // 1024: 0.0533 ms); SEM_K8_THREADS overrides (A/B)
    static const int bt = [] {
        const char *v = getenv("SEM_K8_THREADS");
        const int b = v ? atoi(v) : 128;
        return (b == 64 || b == 128 || b == 256 || b == 512 || b == 1024) ? b : 128;
    }();
    // shared nodes per thread: 2 (C4 step 0.3782 -> 0.3763 ms, C3 0.1875 -> 0.1861 ms against 1;
    // profiles/r2s4_k8_ab.md); SEM_K8_NPT=1|2|4 overrides (A/B)
    static const int npt = [] {
        const char *v = getenv("SEM_K8_NPT");
        const int n = v ? atoi(v) : 2;
        return (n == 1 || n == 2 || n == 4) ? n : 2;
    }();
    const int64_t nsh = ch.N_sh - ch.N_if;
    if (npt == 2) return launch_ex(k8_fix2, blocks_for((nsh + 1) / 2, bt), (unsigned)bt, 0, s, pdl, ch, p);
    if (npt == 4) return launch_ex(k8_fixn<4>, blocks_for((nsh + 3) / 4, bt), (unsigned)bt, 0, s, pdl, ch, p);
    return launch_ex(k8_fix, blocks_for(ch.N_sh - ch.N_if, bt), (unsigned)bt, 0, s, pdl, ch, p);
}

cudaError_t launch_if_partial(const DevChunks &ch, const double *slot, double *xbuf, const int32_t *send_if,
                              int64_t n_send, double *sendbuf, cudaStream_t s) {
    if (ch.N_if == 0) return cudaSuccess;
    k_if_partial<<<blocks_for(ch.N_if), kThreads, 0, s>>>(ch, slot, xbuf);
    if (n_send > 0) k_pack<<<blocks_for(n_send), kThreads, 0, s>>>(xbuf, send_if, n_send, sendbuf);
    return cudaGetLastError();
}

cudaError_t launch_k8_if(const DevChunks &ch, const StepParams &p, const double *xbuf, const int32_t *sum_start,
                         const int32_t *sum_src, cudaStream_t s) {
    if (ch.N_if == 0) return cudaSuccess;
    k8_if<<<blocks_for(ch.N_if), kThreads, 0, s>>>(ch, p, xbuf, sum_start, sum_src);
    return cudaGetLastError();
}

cudaError_t launch_mass_if(const DevChunks &ch, const double *xbuf, const int32_t *sum_start, const int32_t *sum_src,
                           double numer, double *dt2M, cudaStream_t s) {
    if (ch.N_if == 0) return cudaSuccess;
    k_mass_if<<<blocks_for(ch.N_if), kThreads, 0, s>>>(ch, xbuf, sum_start, sum_src, numer, dt2M);
    return cudaGetLastError();
}

cudaError_t launch_abl_elem(int np, bool atomic, const int32_t *mu, const int32_t *eidx, int64_t e0, int64_t e1,
                            const StepParams &p, double *KU, cudaStream_t s) {
    if (e1 <= e0) return cudaSuccess;
    const unsigned nb = blocks_for(e1 - e0);
    if (np == 6) {
        if (atomic) k_abl_elem<6, true><<<nb, kThreads, 0, s>>>(mu, eidx, e0, e1, p, KU);
        else k_abl_elem<6, false><<<nb, kThreads, 0, s>>>(mu, eidx, e0, e1, p, KU);
    } else {
        if (atomic) k_abl_elem<10, true><<<nb, kThreads, 0, s>>>(mu, eidx, e0, e1, p, KU);
        else k_abl_elem<10, false><<<nb, kThreads, 0, s>>>(mu, eidx, e0, e1, p, KU);
    }
    return cudaGetLastError();
}

cudaError_t launch_abl_update(int64_t n, const StepParams &p, double *KU, cudaStream_t s) {
    k_abl_update<<<blocks_for(n), kThreads, 0, s>>>(n, p, KU);
    return cudaGetLastError();
}

cudaError_t launch_step_inc(int64_t *n, cudaStream_t s, bool pdl) {
    return launch_ex(k_step_inc, 1, 1, 0, s, pdl, n);
}

cudaError_t launch_comm_standin(double us, int ctas, cudaStream_t s) {
    static const int kb = [] { const char *e = getenv("SEM_OVERLAP_PROBE_SMEM_KB"); return e ? atoi(e) : 0; }();
    const size_t smem = (size_t)(kb > 0 ? kb : 1) * 1024;
    cudaError_t e = raise_max_smem((const void *)k_comm_standin, smem);
    if (e != cudaSuccess) return e;
    k_comm_standin<<<ctas, 128, smem, s>>>((long long)(us * 1e3));
    return cudaGetLastError();
}

cudaError_t launch_step_set(int64_t *n, int64_t v, cudaStream_t s) {
    k_step_set<<<1, 1, 0, s>>>(n, v);
    return cudaGetLastError();
}

cudaError_t launch_permute_f64(const double *in, const int32_t *imap, const int32_t *omap, int64_t n,
                               double *out, cudaStream_t s) {
    k_permute_f64<<<blocks_for(n), kThreads, 0, s>>>(in, imap, omap, n, out);
    return cudaGetLastError();
}

cudaError_t launch_check_positive(const double *a, int64_t n, int32_t *first, cudaStream_t s) {
    if (n > 0) k_positive<<<blocks_for(n), kThreads, 0, s>>>(a, n, first);
    return cudaGetLastError();
}

cudaError_t launch_nonfinite(const double *a, int64_t n, int32_t *flag, cudaStream_t s) {
    k_nonfinite<<<blocks_for(n), kThreads, 0, s>>>(a, n, flag);
    return cudaGetLastError();
}

}  // namespace sem
