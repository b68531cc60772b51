// heun.cu -- sm_100a kernels of the paper's own integrator (NEXT-1 of SURVEY §8f):
// Heun's predictor-corrector on the first-order velocity-pressure system
// (§4.2.1) with Algorithm 1 (V-dot = F grad U,
// per element and node), Algorithm 2 (R = weighted divergence
// of V, scattered to the global nodes), Algorithm 3 (point
// source).  Acoustic coefficients B = -I, F = c_e^2 I, M = 1
// (reading R2).  Product path; the oracle's orc_heun is the CPU definition.
//
// One Heun step, exactly rearranged (linearity of Algorithms 1 and 2):
//   a   = R(V^n)                       (Algorithm 2 on the stored V)
//   b   = K U^n                        (= -R(Vdot(U^n)): Alg. 2 o Alg. 1)
//   Ud1 = (a + y(t_n)) / M
//   U^{n+1} = U^n + (h/2)/M (2a - h b + y(t_n) + y(t_{n+1}))
//   W^n     = U^n + (h/2) Ud1
//   V^{n+1} = V^n + h Vdot(W^n)        (= V + h/2 (Vdot(U) + Vdot(U + h Ud1)))
// The V update needs W^n at all nodes of an element, i.e. after the step's
// node reduction, so it is LAGGED into the next step's element pass: kernel
// mode LAG first finalises V^n = V^{n-1}+h Vdot(W^{n-1}) from the gathered W,
// then runs the step.  Mode FIN only finalises V (before read-out).  One pass
// over the mesh per Heun step, where the paper runs two RHS evaluations.
//
//  KH7 k_heun<NP,B,MODE>  persistent, warp-specialised like K7 (step.cu): TMA
//                         bulk copies of the chunk's blocks + cp.async gathers of
//                         shared-node U, W; per element (one thread): V lagged
//                         update, r = Alg. 2 element contribution of V, k = K^e u;
//                         (r, k) pairs reduced per node in CSR order, interior
//                         nodes updated in place, shared nodes -> double2 slots
//  KH8 k_heun_fix         shared nodes: slots summed in chunk order, same update
#include <cuda_runtime.h>

#include <map>
#include <vector>

#include "dev_common.cuh"
#include "kernels.h"

namespace sem {

namespace {

constexpr int kStagesH = 2;

// tables packed densely for the current degree: h_Dr[p * Np + q] = dN_q/dr at node p
__constant__ double h_Dr[kMaxNp * kMaxNp];
__constant__ double h_Ds[kMaxNp * kMaxNp];
__constant__ double h_Srr[kMaxNp * kMaxNp];
__constant__ double h_Sss[kMaxNp * kMaxNp];
__constant__ double h_Srs[kMaxNp * kMaxNp];
__constant__ double h_wK[kMaxNp];

// Shared-memory layout of one stage (offsets 16-byte aligned).
// The producer reads the gathers' shared-node ids from a TMA copy in the stage at P >= 5
// (B1 Heun P5 1.102 -> 1.045 ms); at P2/P3 the dependent global loads measured 0.7 % faster.
__host__ __device__ constexpr bool ids_tma(int np) { return np > 10; }
// P5 / P7 with several consumer threads per element: the element products on the FP64 tensor
// cores (A/B: -DSEM_HEUN_TC=0)
#ifndef SEM_HEUN_TC
#define SEM_HEUN_TC 1
#endif
__host__ __device__ constexpr bool heun_tc(int np, int g) { return SEM_HEUN_TC != 0 && g >= 4 && np >= 21; }

// D = A B + C for one 8x8x4 fp64 tile (mma.sync, SASS DMMA); per-lane fragments A[lane / 4][lane % 4],
// B[lane % 4][lane / 4], C / D[lane / 4][2 (lane % 4) + i]
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct HeunLayout {
    int lidx, lpos, jds, shs, shn, g, meta, u, w, size;
    __host__ __device__ HeunLayout(int np, int B, int L, int Lp, int Ls) {
        lidx = 0;
        lpos = np * B * 2;
        jds = lpos + np * B * 2;
        shs = jds + Lp * 2;
        shn = shs + Ls * 4;  // P >= 5: the shared-node ids of the producer's gathers (TMA, own mbarrier)
        g = shn + (ids_tma(np) ? Ls * 4 : 0);
        meta = g + 5 * B * 8;
        u = meta + 32;
        w = u + L * 8;
        size = (w + L * 8 + 127) & ~127;
    }
};

// (R(V), K U) of a local node from the jagged-diagonal entry buffer (see
// jds_sum in step.cu): diagonals in order, a warp's lanes on consecutive pairs
template <int W = kJdsW>  // diagonals walked at most (see jds_sum)
__device__ __forceinline__ double2 jds_sum2(const double2 *ebuf, const uint16_t *jo, int end, int ii) {
    double2 y = ebuf[jo[0] + ii];
    for (int d = 1; d < W; d++) {
        const int nd = (d + 1 < kJdsW ? (int)jo[d + 1] : end) - (int)jo[d];
        if (ii >= nd) break;
        const double2 e = ebuf[jo[d] + ii];
        y.x += e.x;
        y.y += e.y;
    }
    return y;
}

__device__ __forceinline__ double src_term(const HeunParams &a, int64_t id, int64_t n) {
    return (id == a.src) ? a.amp * ricker_dev((double)n * a.h, a.f0, a.t0) : 0.0;
}

// The Heun update of a node from its assembled (R(V), K U) = (r, y) (PAPER.md:269-291,
// reading R19): W = U + hM (r + f^n), U' = U + hM ((2 r - h y) + (f^n + f^{n+1})), spelled
// with explicit roundings so every kernel that finalises a node yields the same bits.
__device__ __forceinline__ void heun_update(double u0, double hm, double r, double y, double yn, double yn1,
                                            double h, double &w_out, double &u_out) {
    w_out = __fma_rn(hm, __dadd_rn(r, yn), u0);
    u_out = __fma_rn(hm, __dadd_rn(__fma_rn(-h, y, __dmul_rn(2.0, r)), __dadd_rn(yn, yn1)), u0);
}

// MODE 0: step with V^n stored (no lag); 1: step with V lagged by one W
// update; 2: finalise V only.
template <int NP, int B, int MODE, int G = 1, bool TC = true>
__global__ void __launch_bounds__(B * G + 32, G > 1 ? 1 : B <= 128 ? 2 : 1)
    k_heun(const DevChunks ch, const HeunParams a, int L, int W, int Lp, int Ls, const int32_t *__restrict__ list,
           int64_t nlist) {
    constexpr int C = B * G;  // consumer threads
    constexpr bool kLag = MODE >= 1, kStep = MODE <= 1, kFin = MODE == 2;
    extern __shared__ __align__(128) unsigned char sm[];
    const HeunLayout lay(NP, B, L, Lp, Ls);
    double2 *ebuf = reinterpret_cast<double2 *>(sm + kStagesH * lay.size);  // [NP*B] (r, k) per entry
    double *m_s = reinterpret_cast<double *>(ebuf + (kStep ? NP * B : 0));  // (h/2)/M window
    uint64_t *full = reinterpret_cast<uint64_t *>(m_s + (kStep ? W : 0));
    uint64_t *gath = full + kStagesH;
    uint64_t *empty = gath + kStagesH;
    uint64_t *wfull = empty + kStagesH;
    uint64_t *wempty = wfull + 1;
    uint64_t *idb = wempty + 1;  // shared-node ids landed
    // G > 1: the five tables in shared memory, rows padded to an even length (16-byte pairs):
    // Dr, Ds, Srr, Sss, Srs at tab + k * NP * kNPp.  Warp-uniform row, broadcast reads.
    constexpr int kNPp = NP + (NP & 1);
    constexpr bool kTcH = TC && heun_tc(NP, G);
    constexpr int kMP = (NP + 7) / 8 * 8, kKP = (NP + 3) / 4 * 4;  // tensor-core tiles: rows to 8, columns to 4
    // table row stride = 4 or 12 mod 16 doubles: a warp's A-fragment reads (8 rows x 4 columns) hit
    // distinct banks per half-warp
    constexpr int kKS = (kKP % 16 == 4 || kKP % 16 == 12) ? kKP : kKP + 4;
    double *tab = reinterpret_cast<double *>(idb + kStagesH);
    if (kTcH) {  // Dr, Ds, Dr^T, Ds^T, Srr, Sss, Srs zero-padded to [kMP][kKP] (A operands)
        for (int i = threadIdx.x; i < 7 * kMP * kKS; i += blockDim.x) {
            const int tb = i / (kMP * kKS), r = (i / kKS) % kMP, q = i % kKS;
            double v = 0.0;
            if (r < NP && q < NP) {
                const double *src[7] = {h_Dr, h_Ds, h_Dr, h_Ds, h_Srr, h_Sss, h_Srs};
                v = (tb == 2 || tb == 3) ? src[tb][q * NP + r] : src[tb][r * NP + q];
            }
            tab[i] = v;
        }
    } else if (G > 1) {
        for (int i = threadIdx.x; i < NP * NP; i += blockDim.x) {
            const int p = i / NP, q = i % NP;
            tab[p * kNPp + q] = h_Dr[i];
            tab[NP * kNPp + p * kNPp + q] = h_Ds[i];
            tab[2 * NP * kNPp + p * kNPp + q] = h_Srr[i];
            tab[3 * NP * kNPp + p * kNPp + q] = h_Sss[i];
            tab[4 * NP * kNPp + p * kNPp + q] = h_Srs[i];
        }
    }
    const int t = threadIdx.x;
    const int64_t nch = list ? nlist : ch.nchunks;  // chunks this launch walks

    if (t == 0) {
        for (int s = 0; s < kStagesH; s++) {
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

    if (t >= C) {
        // ===== producer warp =====
        const int lane = t - C;
        int k = 0;
        for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
            const int64_t c = list ? list[pos] : pos;
            const int s = k % kStagesH;
            if (k >= kStagesH && lane == 0) mbar_wait(&empty[s], ((k / kStagesH) & 1) ^ 1);
            if (lane == 0) chaos_delay(0x10000u * blockIdx.x + 2u * k);
            __syncwarp();
            unsigned char *st = sm + s * lay.size;
            const int4 m0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
            const int4 m1 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c + 1];
            const int i0 = m0.x, s0 = m0.z, nsh = m0.w, ni_al = m1.z;
            if (lane == 0) {
                reinterpret_cast<int4 *>(st + lay.meta)[0] = m0;
                reinterpret_cast<int4 *>(st + lay.meta)[1] = m1;
                const int nsh4 = (nsh + 3) & ~3;
                uint32_t bytes = NP * B * 2 + 5 * B * 8;
                if (kStep) bytes += NP * B * 2 + 2 * kJdsW * 2 + nsh4 * 4 + (uint32_t)ni_al * 8;
                if (kLag) bytes += (uint32_t)ni_al * 8;
                SEM_DCHECK(c >= 0 && c < ch.nchunks, "chunk id in range");
                SEM_DCHECK(ni_al + ((nsh + 1) & ~1) <= L, "local nodes fit the stage's u / w buffers");
                SEM_DCHECK(((nsh + 3) & ~3) <= Ls, "shared-node lists fit the stage");
                SEM_DCHECK(!kStep || ni_al <= W, "(h/2)/M window fits");
                if (ids_tma(NP)) {  // first: the ids the gathers wait for
                    mbar_arrive_expect_tx(&idb[s], nsh4 * 4);
                    if (nsh4 > 0) tma_load(st + lay.shn, ch.shl_node + s0, nsh4 * 4, &idb[s]);
                }
                mbar_arrive_expect_tx(&full[s], bytes);
                const int64_t e0 = c * B;
                tma_load(st + lay.lidx, ch.lidx + e0 * NP, NP * B * 2, &full[s]);
                for (int g = 0; g < 5; g++) tma_load(st + lay.g + g * B * 8, a.geo[g] + e0, B * 8, &full[s]);
                if (kStep) {
                    tma_load(st + lay.lpos, ch.lpos + e0 * NP, NP * B * 2, &full[s]);
                    tma_load(st + lay.jds, ch.jds + c * 2 * kJdsW, 2 * kJdsW * 2, &full[s]);
                    if (nsh4 > 0) tma_load(st + lay.shs, ch.shl_slot + s0, nsh4 * 4, &full[s]);
                    if (ni_al > 0) tma_load(st + lay.u, a.U + i0, ni_al * 8, &full[s]);
                }
                if (kLag && ni_al > 0) tma_load(st + lay.w, a.W + i0, ni_al * 8, &full[s]);
            }
            double *u_sh = reinterpret_cast<double *>(st + lay.u) + ni_al;
            double *w_sh = reinterpret_cast<double *>(st + lay.w) + ni_al;
            const int32_t *ids = ids_tma(NP) ? reinterpret_cast<const int32_t *>(st + lay.shn) : ch.shl_node + s0;
            if (ids_tma(NP)) {
                __syncwarp();
                mbar_wait(&idb[s], (k / kStagesH) & 1);
            }
            for (int j = lane; j < nsh; j += 32) {
                const int64_t g = ch.N_int + ids[j];
                if (kStep) cp_async8(u_sh + j, a.U + g);
                if (kLag) cp_async8(w_sh + j, a.W + g);
            }
            cp_async_arrive_noinc(&gath[s]);
            if (kStep && lane == 0) {
                if (k >= 1) mbar_wait(wempty, (k - 1) & 1);
                chaos_delay(0x10000u * blockIdx.x + 2u * k + 1u);
                mbar_arrive_expect_tx(wfull, (uint32_t)ni_al * 8);
                if (ni_al > 0) tma_load(m_s, a.hM + i0, ni_al * 8, wfull);
            }
        }
        return;
    }

    if constexpr (kTcH) {
        // ===== consumer warps, tensor cores (P5, P7) =====
        // Every per-element product of the step is a dense [Np x Np] x [Np x 8] tile product per
        // warp (warp wi: elements 8 wi .. 8 wi + 7 of the chunk), on mma.sync m8n8k4 f64 (DMMA):
        //   (1) Algorithm 1 on W: (gr, gs) = (Dr, Ds) W, the lagged V update in the epilogue
        //       (V read and written straight from / to global, fragment by fragment), which
        //       also forms Algorithm 2's aux = -detJ w J^-1 V into shared memory;
        //   (2) r = Dr^T ar + Ds^T as (aux from shared memory) and Srr u, Sss u, Srs u;
        //       y = grr Srr u + gss Sss u + grs Srs u in the epilogue.
        // Fragments (per lane): A[lane / 4][lane % 4], B[lane % 4][lane / 4], C[lane / 4][2 (lane % 4) + i].
        constexpr int MT = kMP / 8, KT = kKP / 4;
        static_assert(B / 8 <= C / 32, "one 8-element tile per consumer warp");
        const int lane = t & 31, nt = t >> 5;
        const bool tile = nt < B / 8;
        const int eb = nt * 8 + (lane >> 2);  // this lane's B-fragment element
        const double f_n = src_term(a, a.src, a.n), f_n1 = src_term(a, a.src, a.n + 1);
        double *xs = reinterpret_cast<double *>(ebuf);  // aux [NP][2][B], aliases the entry buffer
        auto At = [&](int tb, int m, int ks) { return tab[(tb * kMP + m * 8 + (lane >> 2)) * kKS + ks * 4 + (lane & 3)]; };
        int k = 0;
        for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
            const int64_t c = list ? list[pos] : pos;
            const int s = k % kStagesH;
            mbar_wait(&full[s], (k / kStagesH) & 1);
            mbar_wait(&gath[s], (k / kStagesH) & 1);
            const unsigned char *st = sm + s * lay.size;
            const int4 m0 = reinterpret_cast<const int4 *>(st + lay.meta)[0];
            const int4 m1 = reinterpret_cast<const int4 *>(st + lay.meta)[1];
            const int i0 = m0.x, nint = m0.y, nsh = m0.w, ne = m1.y, ni_al = m1.z;
            const uint16_t *li_s = reinterpret_cast<const uint16_t *>(st + lay.lidx);
            const double *g_s = reinterpret_cast<const double *>(st + lay.g);
            double *Vc = a.V + (c * 2 * NP) * B;  // this chunk's V, [2 NP][B]
            if (kChecked) {
                const int4 r0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
                SEM_DCHECK(r0.x == m0.x && r0.y == m0.y && r0.z == m0.z && r0.w == m0.w, "stage meta is this chunk's");
            }
            // (1) lagged V update (and aux) per tile
            if (kLag && tile) {
                const double *w_s = reinterpret_cast<const double *>(st + lay.w);
                // this lane's V entries of the epilogue, loaded before the products
                double vv[MT][2][2];
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const int e = nt * 8 + 2 * (lane & 3) + i;
#pragma unroll
                    for (int m = 0; m < MT; m++) {
                        const int p = m * 8 + (lane >> 2);
                        const bool ok = e < ne && p < NP;
                        vv[m][i][0] = ok ? Vc[p * B + e] : 0.0;
                        vv[m][i][1] = ok ? Vc[(NP + p) * B + e] : 0.0;
                    }
                }
                double gr[MT][2], gs[MT][2];
#pragma unroll
                for (int m = 0; m < MT; m++) gr[m][0] = gr[m][1] = gs[m][0] = gs[m][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KT; ks++) {
                    const int q = ks * 4 + (lane & 3);
                    const double b = (q < NP && eb < ne) ? w_s[li_s[q * B + eb]] : 0.0;
#pragma unroll
                    for (int m = 0; m < MT; m++) {
                        dmma_8x8x4(gr[m][0], gr[m][1], At(0, m, ks), b);
                        dmma_8x8x4(gs[m][0], gs[m][1], At(1, m, ks), b);
                    }
                }
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const int e = nt * 8 + 2 * (lane & 3) + i;
                    if (e < ne) {
                        const double F00 = g_s[e], F01 = g_s[B + e], F10 = g_s[2 * B + e], F11 = g_s[3 * B + e];
                        const double sd = g_s[4 * B + e];
                        const double hF00 = a.h * F00, hF01 = a.h * F01, hF10 = a.h * F10, hF11 = a.h * F11;
#pragma unroll
                        for (int m = 0; m < MT; m++) {
                            const int p = m * 8 + (lane >> 2);
                            if (p < NP) {
                                double v0 = vv[m][i][0], v1 = vv[m][i][1];
                                v0 = fma(hF00, gr[m][i], fma(hF10, gs[m][i], v0));
                                v1 = fma(hF01, gr[m][i], fma(hF11, gs[m][i], v1));
                                Vc[p * B + e] = v0;
                                Vc[(NP + p) * B + e] = v1;
                                if (kStep) {
                                    const double sw = -sd * h_wK[p];
                                    xs[(2 * p) * B + e] = sw * fma(F00, v0, F01 * v1);
                                    xs[(2 * p + 1) * B + e] = sw * fma(F10, v0, F11 * v1);
                                }
                            }
                        }
                    }
                }
            }
            if (kStep) {
                if (!kLag) {  // V as stored: aux straight from it
                    for (int idx = t; idx < NP * ne; idx += C) {
                        const int p = idx / ne, e = idx % ne;
                        const double F00 = g_s[e], F01 = g_s[B + e], F10 = g_s[2 * B + e], F11 = g_s[3 * B + e];
                        const double sw = -g_s[4 * B + e] * h_wK[p];
                        const double v0 = Vc[p * B + e], v1 = Vc[(NP + p) * B + e];
                        xs[(2 * p) * B + e] = sw * fma(F00, v0, F01 * v1);
                        xs[(2 * p + 1) * B + e] = sw * fma(F10, v0, F11 * v1);
                    }
                }
                consumer_sync<C>();
                // (2) r = Dr^T ar + Ds^T as; Srr u, Sss u, Srs u
                const double *u_s = reinterpret_cast<const double *>(st + lay.u);
                double rr[MT][2], yr[MT][2], ys[MT][2], yx[MT][2];
#pragma unroll
                for (int m = 0; m < MT; m++)
                    rr[m][0] = rr[m][1] = yr[m][0] = yr[m][1] = ys[m][0] = ys[m][1] = yx[m][0] = yx[m][1] = 0.0;
                if (tile) {
#pragma unroll
                    for (int ks = 0; ks < KT; ks++) {
                        const int q = ks * 4 + (lane & 3);
                        const bool ok = q < NP && eb < ne;
                        const double bar = ok ? xs[(2 * q) * B + eb] : 0.0;
                        const double bas = ok ? xs[(2 * q + 1) * B + eb] : 0.0;
                        const double bu = ok ? u_s[li_s[q * B + eb]] : 0.0;
#pragma unroll
                        for (int m = 0; m < MT; m++) {
                            dmma_8x8x4(rr[m][0], rr[m][1], At(2, m, ks), bar);
                            dmma_8x8x4(rr[m][0], rr[m][1], At(3, m, ks), bas);
                            dmma_8x8x4(yr[m][0], yr[m][1], At(4, m, ks), bu);
                            dmma_8x8x4(ys[m][0], ys[m][1], At(5, m, ks), bu);
                            dmma_8x8x4(yx[m][0], yx[m][1], At(6, m, ks), bu);
                        }
                    }
                }
                consumer_sync<C>();  // every aux read before the entries overwrite it
                const uint16_t *lpo = reinterpret_cast<const uint16_t *>(st + lay.lpos);
                if (tile) {
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        const int e = nt * 8 + 2 * (lane & 3) + i;
                        if (e < ne) {
                            const double F00 = g_s[e], F01 = g_s[B + e], F10 = g_s[2 * B + e], F11 = g_s[3 * B + e];
                            const double sd = g_s[4 * B + e];
                            const double grr = sd * fma(F00, F00, F01 * F01);
                            const double gss = sd * fma(F10, F10, F11 * F11);
                            const double grs = sd * fma(F00, F10, F01 * F11);
#pragma unroll
                            for (int m = 0; m < MT; m++) {
                                const int p = m * 8 + (lane >> 2);
                                if (p < NP)
                                    ebuf[lpo[p * B + e]] =
                                        make_double2(rr[m][i], fma(grr, yr[m][i], fma(gss, ys[m][i], grs * yx[m][i])));
                            }
                        }
                    }
                }
                consumer_sync<C>();
                mbar_wait(wfull, k & 1);
                // (4) node-centric reduction in fixed (JDS diagonal) order + fused Heun update
                const uint16_t *jd = reinterpret_cast<const uint16_t *>(st + lay.jds);
                const int32_t *shs = reinterpret_cast<const int32_t *>(st + lay.shs);
                const int nwork = nint + nsh;
                for (int wk = t; wk < nwork; wk += C) {
                    const int i = wk < nint ? wk : ni_al + (wk - nint);  // skips the alignment hole
                    const double2 ab = ch.max_count <= 32
                                           ? (i < nint ? jds_sum2<32>(ebuf, jd, m1.x, i) : jds_sum2<32>(ebuf, jd + kJdsW, m1.w, i - ni_al))
                                           : (i < nint ? jds_sum2(ebuf, jd, m1.x, i) : jds_sum2(ebuf, jd + kJdsW, m1.w, i - ni_al));
                    if (i < nint) {
                        const int64_t id = i0 + i;
                        const bool src = id == a.src;
                        heun_update(u_s[i], m_s[i], ab.x, ab.y, src ? f_n : 0.0, src ? f_n1 : 0.0, a.h, a.W[id],
                                    a.U[id]);
                    } else {
                        reinterpret_cast<double2 *>(a.slot)[shs[i - ni_al]] = ab;
                    }
                }
            }
            consumer_sync<C>();
            if (kChecked) {
                unsigned char *stw = sm + s * lay.size;
                double *uw = reinterpret_cast<double *>(stw + lay.u);
                double *ww = reinterpret_cast<double *>(stw + lay.w);
                for (int i = t; i < ni_al + nsh; i += C) { uw[i] = poison_f64(); ww[i] = poison_f64(); }
                if (kStep) for (int i = t; i < ni_al; i += C) m_s[i] = poison_f64();
                consumer_sync<C>();
            }
            if (t == 0) {
                mbar_arrive(&empty[s]);
                if (kStep) mbar_arrive(wempty);
            }
        }
        return;
    }
    if constexpr (G > 1 && !kTcH) {
        // ===== consumer warps, G threads per element (high orders: P5 optionally, P7) =====
        // Warp wi takes elements 32 (wi / G) + lane and the row block rb = wi % G (rows
        // p = rb R + r) of every per-element product: the lagged V update (Algorithm 1) on its
        // rows of V, its rows of Algorithm 2's aux = -detJ w J^-1 V handed to the element's
        // other threads through shared memory (the entry buffer, before it holds entries), and
        // its rows of r = D^T aux and y = K^e u (three products with the S tables, then
        // combined with G_e).  The node phase is the G = 1 one with C threads.
        constexpr int R = (NP + G - 1) / G;
        const int wi = t >> 5, te = ((wi / G) << 5) + (t & 31), rb = wi % G;
        const double f_n = src_term(a, a.src, a.n), f_n1 = src_term(a, a.src, a.n + 1);
        double *xs = reinterpret_cast<double *>(ebuf);  // aux scratch [NP][2][B], aliases the entry buffer
        int k = 0;
        for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
            const int64_t c = list ? list[pos] : pos;
            const int s = k % kStagesH;
            double *vg = a.V + (c * 2 * NP) * B + te;  // this element's V, layout [chunk][2 NP][B]
            double v[2 * R];
#pragma unroll
            for (int r = 0; r < R; r++) {
                const int p = rb * R + r;
                v[r] = p < NP ? vg[p * B] : 0.0;
                v[R + r] = p < NP ? vg[(NP + p) * B] : 0.0;
            }
            mbar_wait(&full[s], (k / kStagesH) & 1);
            mbar_wait(&gath[s], (k / kStagesH) & 1);
            const unsigned char *st = sm + s * lay.size;
            const int4 m0 = reinterpret_cast<const int4 *>(st + lay.meta)[0];
            const int4 m1 = reinterpret_cast<const int4 *>(st + lay.meta)[1];
            const int i0 = m0.x, nint = m0.y, nsh = m0.w, ne = m1.y, ni_al = m1.z;
            const uint16_t *li_s = reinterpret_cast<const uint16_t *>(st + lay.lidx);
            const double *g_s = reinterpret_cast<const double *>(st + lay.g);
            const bool act = te < ne;
            const double F00 = g_s[te], F01 = g_s[B + te], F10 = g_s[2 * B + te], F11 = g_s[3 * B + te];
            const double sd = g_s[4 * B + te];
            if (kChecked) {
                const int4 r0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
                SEM_DCHECK(r0.x == m0.x && r0.y == m0.y && r0.z == m0.z && r0.w == m0.w, "stage meta is this chunk's");
                for (int e = t; e < NP * ne; e += C) {
                    const int li = li_s[(e / ne) * B + e % ne];
                    SEM_DCHECK(li < nint || (li >= ni_al && li < ni_al + nsh), "local index in range (poisoned?)");
                }
            }
            // (1) lagged V update on this thread's rows: V^n = V^{n-1} + h F^T (D w)
            if (kLag && act) {
                const double *w_s = reinterpret_cast<const double *>(st + lay.w);
                double gr[R], gs[R];
#pragma unroll
                for (int r = 0; r < R; r++) gr[r] = gs[r] = 0.0;
                const double *tDr = tab + rb * R * kNPp, *tDs = tDr + NP * kNPp;
#pragma unroll
                for (int q = 0; q < NP; q += 2) {  // q pairs: one 16-byte broadcast read per table row
                    const double w0 = w_s[li_s[q * B + te]];
                    const double w1 = q + 1 < NP ? w_s[li_s[(q + 1) * B + te]] : 0.0;
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        if (rb * R + r < NP) {
                            const double2 dr = *reinterpret_cast<const double2 *>(tDr + r * kNPp + q);
                            const double2 ds = *reinterpret_cast<const double2 *>(tDs + r * kNPp + q);
                            gr[r] = fma(dr.x, w0, gr[r]);
                            gs[r] = fma(ds.x, w0, gs[r]);
                            if (q + 1 < NP) {
                                gr[r] = fma(dr.y, w1, gr[r]);
                                gs[r] = fma(ds.y, w1, gs[r]);
                            }
                        }
                    }
                }
                const double hF00 = a.h * F00, hF01 = a.h * F01, hF10 = a.h * F10, hF11 = a.h * F11;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const int p = rb * R + r;
                    if (p < NP) {
                        v[r] = fma(hF00, gr[r], fma(hF10, gs[r], v[r]));
                        v[R + r] = fma(hF01, gr[r], fma(hF11, gs[r], v[R + r]));
                        vg[p * B] = v[r];
                        vg[(NP + p) * B] = v[R + r];
                    }
                }
            }
            if (kStep) {
                // (2a) Algorithm 2's aux on this thread's rows q: (ar, as)_q = -sd w_q F V_q
                if (act) {
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        const int q = rb * R + r;
                        if (q < NP) {
                            const double sw = -sd * h_wK[q];
                            xs[(2 * q) * B + te] = sw * fma(F00, v[r], F01 * v[R + r]);
                            xs[(2 * q + 1) * B + te] = sw * fma(F10, v[r], F11 * v[R + r]);
                        }
                    }
                }
                consumer_sync<C>();
                // (2b) r_p = sum_q Dr[q][p] ar_q + Ds[q][p] as_q; (3) y_p = (K^e u)_p, this thread's rows
                double rr[R], yy[R];
                const uint16_t *lpo = reinterpret_cast<const uint16_t *>(st + lay.lpos);
                const double *u_s = reinterpret_cast<const double *>(st + lay.u);
                if (act) {
#pragma unroll
                    for (int r = 0; r < R; r++) rr[r] = 0.0;
#pragma unroll
                    for (int q = 0; q < NP; q++) {
                        const double ar = xs[(2 * q) * B + te], as = xs[(2 * q + 1) * B + te];
                        const double *dq = tab + q * kNPp + rb * R;  // Dr[q][p], Ds[q][p]: row q, columns p
#pragma unroll
                        for (int r = 0; r < R; r++)
                            if (rb * R + r < NP) rr[r] = fma(dq[r], ar, fma(dq[NP * kNPp + r], as, rr[r]));
                    }
                    const double grr = sd * fma(F00, F00, F01 * F01);
                    const double gss = sd * fma(F10, F10, F11 * F11);
                    const double grs = sd * fma(F00, F10, F01 * F11);
                    double arr[R], ass[R], ars[R];
#pragma unroll
                    for (int r = 0; r < R; r++) arr[r] = ass[r] = ars[r] = 0.0;
                    const double *tS = tab + 2 * NP * kNPp + rb * R * kNPp;
#pragma unroll
                    for (int q = 0; q < NP; q += 2) {
                        const double u0 = u_s[li_s[q * B + te]];
                        const double u1 = q + 1 < NP ? u_s[li_s[(q + 1) * B + te]] : 0.0;
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            if (rb * R + r < NP) {
                                const double2 srr = *reinterpret_cast<const double2 *>(tS + r * kNPp + q);
                                const double2 sss = *reinterpret_cast<const double2 *>(tS + NP * kNPp + r * kNPp + q);
                                const double2 srs = *reinterpret_cast<const double2 *>(tS + 2 * NP * kNPp + r * kNPp + q);
                                arr[r] = fma(srr.x, u0, arr[r]);
                                ass[r] = fma(sss.x, u0, ass[r]);
                                ars[r] = fma(srs.x, u0, ars[r]);
                                if (q + 1 < NP) {
                                    arr[r] = fma(srr.y, u1, arr[r]);
                                    ass[r] = fma(sss.y, u1, ass[r]);
                                    ars[r] = fma(srs.y, u1, ars[r]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < R; r++) yy[r] = fma(grr, arr[r], fma(gss, ass[r], grs * ars[r]));
                }
                consumer_sync<C>();  // every aux read before the entries overwrite it
                if (act) {
#pragma unroll
                    for (int r = 0; r < R; r++) {
                        const int p = rb * R + r;
                        if (p < NP) ebuf[lpo[p * B + te]] = make_double2(rr[r], yy[r]);
                    }
                }
                consumer_sync<C>();
                mbar_wait(wfull, k & 1);
                // (4) node-centric reduction in fixed (JDS diagonal) order + fused Heun update
                const uint16_t *jd = reinterpret_cast<const uint16_t *>(st + lay.jds);
                const int32_t *shs = reinterpret_cast<const int32_t *>(st + lay.shs);
                const int nwork = nint + nsh;
                for (int wk = t; wk < nwork; wk += C) {
                    const int i = wk < nint ? wk : ni_al + (wk - nint);  // skips the alignment hole
                    const double2 ab = ch.max_count <= 32
                                     ? (i < nint ? jds_sum2<32>(ebuf, jd, m1.x, i) : jds_sum2<32>(ebuf, jd + kJdsW, m1.w, i - ni_al))
                                     : (i < nint ? jds_sum2(ebuf, jd, m1.x, i) : jds_sum2(ebuf, jd + kJdsW, m1.w, i - ni_al));
                    if (i < nint) {
                        const int64_t id = i0 + i;
                        const bool src = id == a.src;
                        heun_update(u_s[i], m_s[i], ab.x, ab.y, src ? f_n : 0.0, src ? f_n1 : 0.0, a.h, a.W[id],
                                    a.U[id]);
                    } else {
                        reinterpret_cast<double2 *>(a.slot)[shs[i - ni_al]] = ab;
                    }
                }
            }
            consumer_sync<C>();
            if (kChecked) {
                unsigned char *stw = sm + s * lay.size;
                double *uw = reinterpret_cast<double *>(stw + lay.u);
                double *ww = reinterpret_cast<double *>(stw + lay.w);
                uint16_t *lw = reinterpret_cast<uint16_t *>(stw + lay.lidx);
                for (int i = t; i < ni_al + nsh; i += C) { uw[i] = poison_f64(); ww[i] = poison_f64(); }
                for (int i = t; i < (kStep ? 2 : 1) * NP * B; i += C) lw[i] = 0xFFFF;
                if (kStep) for (int i = t; i < ni_al; i += C) m_s[i] = poison_f64();
                consumer_sync<C>();
            }
            if (t == 0) {
                mbar_arrive(&empty[s]);
                if (kStep) mbar_arrive(wempty);
            }
        }
        return;
    }

    if constexpr (G == 1) {
    // ===== consumer warps =====
    // the source terms f^n, f^{n+1} of this step, once per thread (cold exp() code out of the loops)
    const double f_n = src_term(a, a.src, a.n), f_n1 = src_term(a, a.src, a.n + 1);
    // each element's own interior nodes (one entry each, last in the interior segment:
    // chunk builders) are finalised by the element's thread; the node phase skips them
    // (P3; at P5 this measured 4 % slower at the 168-register cap, as in K7)
    constexpr int kNI = NP < 21 ? lattice_n_interior(NP) : 0;
    int k = 0;
    for (int64_t pos = blockIdx.x; pos < nch; pos += gridDim.x, k++) {
        const int64_t c = list ? list[pos] : pos;
        const int s = k % kStagesH;
        // this element's V (layout [chunk][2 NP][B]): issued before the stage wait
        double *vg = a.V + (c * 2 * NP) * B + t;
        double v[2 * NP];
#pragma unroll
        for (int j = 0; j < 2 * NP; j++) v[j] = vg[j * B];
        mbar_wait(&full[s], (k / kStagesH) & 1);
        mbar_wait(&gath[s], (k / kStagesH) & 1);
        const unsigned char *st = sm + s * lay.size;
        const int4 m0 = reinterpret_cast<const int4 *>(st + lay.meta)[0];
        const int4 m1 = reinterpret_cast<const int4 *>(st + lay.meta)[1];
        const int i0 = m0.x, nint = m0.y, nsh = m0.w, ne = m1.y, ni_al = m1.z;
        const uint16_t *li_s = reinterpret_cast<const uint16_t *>(st + lay.lidx);
        const double *g_s = reinterpret_cast<const double *>(st + lay.g);
        const double F00 = g_s[t], F01 = g_s[B + t], F10 = g_s[2 * B + t], F11 = g_s[3 * B + t];
        const double sd = g_s[4 * B + t];
        if (kChecked) {  // the stage holds this chunk (a stale or foreign stage fails here)
            const int4 r0 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c];
            const int4 r1 = reinterpret_cast<const int4 *>(ch.cmeta)[2 * c + 1];
            SEM_DCHECK(r0.x == m0.x && r0.y == m0.y && r0.z == m0.z && r0.w == m0.w && r1.x == m1.x &&
                           r1.y == m1.y && r1.z == m1.z && r1.w == m1.w,
                       "stage meta is this chunk's");
            for (int e = t; e < NP * ne; e += B) {
                const int li = li_s[(e / ne) * B + e % ne];
                SEM_DCHECK(li < nint || (li >= ni_al && li < ni_al + nsh), "local index in range (poisoned?)");
            }
        }

        // (1) lagged V update: V^n = V^{n-1} + h Vdot(W^{n-1})  (Algorithm 1, E = 0)
        if (kLag && t < ne) {
            const double *w_s = reinterpret_cast<const double *>(st + lay.w);
            double w[NP];
#pragma unroll
            for (int p = 0; p < NP; p++) w[p] = w_s[li_s[p * B + t]];
            const double hF00 = a.h * F00, hF01 = a.h * F01, hF10 = a.h * F10, hF11 = a.h * F11;
#pragma unroll
            for (int p = 0; p < NP; p++) {
                double gr = 0.0, gs = 0.0;
#pragma unroll
                for (int q = 0; q < NP; q++) {
                    gr = fma(h_Dr[p * NP + q], w[q], gr);
                    gs = fma(h_Ds[p * NP + q], w[q], gs);
                }
                v[p] = fma(hF00, gr, fma(hF10, gs, v[p]));
                v[NP + p] = fma(hF01, gr, fma(hF11, gs, v[NP + p]));
            }
#pragma unroll
            for (int j = 0; j < 2 * NP; j++) vg[j * B] = v[j];
        }

        if (kStep) {
            const uint16_t *lpo = reinterpret_cast<const uint16_t *>(st + lay.lpos);
            const uint16_t *jd = reinterpret_cast<const uint16_t *>(st + lay.jds);
            double rin[NP], yin[NP];  // element-interior rows (registers only at those p)
            const int32_t *shs = reinterpret_cast<const int32_t *>(st + lay.shs);
            const double *u_s = reinterpret_cast<const double *>(st + lay.u);
            if (t < ne) {
                // (2) r = Algorithm 2 element term of V: with aux = detJ w_q V_q (B = -I),
                //     r_p = sum_q Dr[q][p] ar_q + Ds[q][p] as_q,  (ar, as)_q = -J^-1 aux_q
                //     (F = c^2 J^-1, sd = detJ / c^2, so detJ J^-1 = sd F)
                double ar[NP], as[NP];
#pragma unroll
                for (int q = 0; q < NP; q++) {
                    const double sw = -sd * h_wK[q];
                    ar[q] = sw * fma(F00, v[q], F01 * v[NP + q]);
                    as[q] = sw * fma(F10, v[q], F11 * v[NP + q]);
                }
                // (r, k) pairs: at P5 r goes to shared memory now (registers), else it
                // stays in registers and the pair is stored with one 16-byte store
                constexpr bool kSplit = NP > 10;
                double *eb = reinterpret_cast<double *>(ebuf);
                double r[NP];  // at P5 only the element-interior rows stay in registers
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    double acc = 0.0;
#pragma unroll
                    for (int q = 0; q < NP; q++) acc = fma(h_Dr[q * NP + p], ar[q], fma(h_Ds[q * NP + p], as[q], acc));
                    if (kSplit && !(kNI > 0 && lattice_interior(NP, p))) eb[2 * lpo[p * B + t]] = acc;
                    else r[p] = acc;
                }
                // (3) y = K^e u, K^e = Grr Srr + Gss Sss + Grs Srs, G = sd F F^T
                //     (= c^2 detJ J^-1 J^-T, reading R5)
                const double grr = sd * fma(F00, F00, F01 * F01);
                const double gss = sd * fma(F10, F10, F11 * F11);
                const double grs = sd * fma(F00, F10, F01 * F11);
                double u[NP], y[NP];
#pragma unroll
                for (int p = 0; p < NP; p++) { u[p] = u_s[li_s[p * B + t]]; y[p] = 0.0; }
#pragma unroll
                for (int p = 0; p < NP; p++) {
#pragma unroll
                    for (int q = p; q < NP; q++) {
                        const double kk = fma(grr, h_Srr[p * NP + q], fma(gss, h_Sss[p * NP + q], grs * h_Srs[p * NP + q]));
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
                    if (kNI > 0 && lattice_interior(NP, p)) {
                        rin[p] = r[p];
                        yin[p] = y[p];
                    } else if (kSplit) {
                        eb[2 * lpo[p * B + t] + 1] = y[p];
                    } else {
                        ebuf[lpo[p * B + t]] = make_double2(r[p], y[p]);
                    }
                }
            }
            consumer_sync<B>();
            mbar_wait(wfull, k & 1);
            if (kNI > 0 && t < ne) {
#pragma unroll
                for (int p = 0; p < NP; p++) {
                    if (!lattice_interior(NP, p)) continue;
                    const int li = li_s[p * B + t];
                    const int64_t id = i0 + li;
                    const bool src = id == a.src;
                    heun_update(u_s[li], m_s[li], rin[p], yin[p], src ? f_n : 0.0, src ? f_n1 : 0.0, a.h, a.W[id],
                                a.U[id]);
                }
            }
            // (4) node-centric reduction in fixed (JDS diagonal) order + fused Heun update
            const int nint_np = nint - ne * kNI;  // interior nodes left to the node phase
            const int nwork = nint_np + nsh;
            for (int w = t; w < nwork; w += B) {
                const int i = w < nint_np ? w : ni_al + (w - nint_np);  // skips the element-interior nodes and the hole
                const double2 ab = ch.max_count <= 32
                                     ? (i < nint ? jds_sum2<32>(ebuf, jd, m1.x, i) : jds_sum2<32>(ebuf, jd + kJdsW, m1.w, i - ni_al))
                                     : (i < nint ? jds_sum2(ebuf, jd, m1.x, i) : jds_sum2(ebuf, jd + kJdsW, m1.w, i - ni_al));
                if (i < nint) {
                    const int64_t id = i0 + i;
                    const bool src = id == a.src;
                    heun_update(u_s[i], m_s[i], ab.x, ab.y, src ? f_n : 0.0, src ? f_n1 : 0.0, a.h, a.W[id], a.U[id]);
                } else {
                    reinterpret_cast<double2 *>(a.slot)[shs[i - ni_al]] = ab;
                }
            }
        }
        consumer_sync<B>();
        if (kChecked) {  // poison everything handed back: only a refill may be read after this
            unsigned char *stw = sm + s * lay.size;
            double *uw = reinterpret_cast<double *>(stw + lay.u);
            double *ww = reinterpret_cast<double *>(stw + lay.w);
            double *gw = reinterpret_cast<double *>(stw + lay.g);
            uint16_t *lw = reinterpret_cast<uint16_t *>(stw + lay.lidx);
            for (int i = t; i < ni_al + nsh; i += B) { uw[i] = poison_f64(); ww[i] = poison_f64(); }
            for (int i = t; i < 5 * B; i += B) gw[i] = poison_f64();
            for (int i = t; i < (kStep ? 2 : 1) * NP * B; i += B) lw[i] = 0xFFFF;
            if (kStep) {
                for (int i = t; i < m1.w; i += B) ebuf[i] = make_double2(poison_f64(), poison_f64());
                for (int i = t; i < ni_al; i += B) m_s[i] = poison_f64();
            }
            consumer_sync<B>();
            if (t == 0) chaos_delay(0x20000u * blockIdx.x + k);
        }
        if (t == 0) {
            mbar_arrive(&empty[s]);
            if (kStep) mbar_arrive(wempty);
        }
    }
    }
}

// ---- KH8: shared-node fix-up ------------------------------------------------------
__global__ void k_heun_fix(const DevChunks ch, const HeunParams a) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ch.N_sh - ch.N_if) return;
    const int j0 = ch.sh_pstart[s], j1 = ch.sh_pstart[s + 1];
    const int64_t id = ch.N_int + s;
    const double u0 = a.U[id], hm = a.hM[id];
    const double2 *sl = reinterpret_cast<const double2 *>(a.slot);
    double2 part[4];
#pragma unroll
    for (int d = 0; d < 4; d++) part[d] = (j0 + d < j1) ? sl[j0 + d] : make_double2(0.0, 0.0);
    double2 ab = part[0];
#pragma unroll
    for (int d = 1; d < 4; d++) { ab.x += part[d].x; ab.y += part[d].y; }
    for (int j = j0 + 4; j < j1; j++) { ab.x += sl[j].x; ab.y += sl[j].y; }
    const double yn = src_term(a, id, a.n), yn1 = src_term(a, id, a.n + 1);
    heun_update(u0, hm, ab.x, ab.y, yn, yn1, a.h, a.W[id], a.U[id]);
}

// Per element (new order, padded): F = c^2 J^-1 (F[jh][j] = c^2 (J^-1)_{jh j}),
// sd = detJ / c^2, and detJ for the mass.  J columns are v1 - v0, v2 - v0.
__global__ void k_geometry_heun(const double *__restrict__ vxy, const int32_t *__restrict__ tri,
                                const int32_t *__restrict__ perm, const double *__restrict__ c_in, int64_t E,
                                int64_t Epad, double *F00, double *F01, double *F10, double *F11, double *sd,
                                double *__restrict__ detJ, int32_t *bad) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= Epad) return;
    if (k >= E) { F00[k] = F01[k] = F10[k] = F11[k] = sd[k] = detJ[k] = 0.0; return; }
    const int64_t e = perm[k];
    const int32_t v0 = tri[3 * e], v1 = tri[3 * e + 1], v2 = tri[3 * e + 2];
    const double j00 = vxy[2 * v1] - vxy[2 * v0], j01 = vxy[2 * v2] - vxy[2 * v0];
    const double j10 = vxy[2 * v1 + 1] - vxy[2 * v0 + 1], j11 = vxy[2 * v2 + 1] - vxy[2 * v0 + 1];
    const double det = j00 * j11 - j01 * j10;
    const double c = c_in[e], c2 = c * c;
    if (!(det > 0.0)) atomicMin(bad, (int32_t)e);
    // J^-1 = [[j11, -j01], [-j10, j00]] / det, indexed [jh][j]
    F00[k] = c2 * (j11 / det);
    F01[k] = c2 * (-j01 / det);
    F10[k] = c2 * (-j10 / det);
    F11[k] = c2 * (j00 / det);
    sd[k] = det / c2;
    detJ[k] = det;
}

// V in the chunk layout [chunk][2 NP][B] (component j = k NP + p) <-> host layout
// [E][NP][2] in INPUT element order (perm: new -> input).
__global__ void k_v_out(const double *__restrict__ V, const int32_t *__restrict__ perm, int64_t E, int NP, int B,
                        double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= E * NP * 2) return;
    const int64_t e = i / (2 * NP);
    const int j = (int)(i % (2 * NP));  // host order: p * 2 + comp
    const int p = j >> 1, comp = j & 1;
    const int64_t c = e / B, t = e % B;
    out[((int64_t)perm[e] * NP + p) * 2 + comp] = V[(c * 2 * NP + comp * NP + p) * B + t];
}

__global__ void k_v_in(const double *__restrict__ in, const int32_t *__restrict__ perm, int64_t E, int NP, int B,
                       double *__restrict__ V) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= E * NP * 2) return;
    const int64_t e = i / (2 * NP);
    const int j = (int)(i % (2 * NP));
    const int p = j >> 1, comp = j & 1;
    const int64_t c = e / B, t = e % B;
    V[(c * 2 * NP + comp * NP + p) * B + t] = in ? in[((int64_t)perm[e] * NP + p) * 2 + comp] : 0.0;
}

template <typename K>
cudaError_t set_smem_h(K kernel, size_t bytes) {
    return raise_max_smem((const void *)kernel, bytes);
}

int heun_group(int np, int B);
size_t heun_smem_bytes(int np, int B, int L, int W, int Lp, int Ls, int mode, bool tc) {
    const HeunLayout lay(np, B, L, Lp, Ls);
    const bool step = mode <= 1;
    const int g = heun_group(np, B);
    const int kp = (np + 3) / 4 * 4, ks = (kp % 16 == 4 || kp % 16 == 12) ? kp : kp + 4;
    const size_t tabs = tc && heun_tc(np, g) ? 7 * (size_t)((np + 7) / 8 * 8) * ks * 8
                        : g > 1        ? 5 * (size_t)np * (np + (np & 1)) * 8
                                       : 0;
    return (size_t)kStagesH * lay.size + (step ? (size_t)np * B * 16 + (size_t)W * 8 : 0) + (4 * kStagesH + 2) * 8 +
           tabs;
}

using HFn = void (*)(const DevChunks, const HeunParams, int, int, int, int, const int32_t *, int64_t);
template <int NP, int B, int G = 1, bool TC = true>
HFn heun_fn_b(int mode) {
    return mode == 0 ? k_heun<NP, B, 0, G, TC> : mode == 1 ? k_heun<NP, B, 1, G, TC> : k_heun<NP, B, 2, G, TC>;
}
template <int NP, int B, int G>
HFn heun_fn_tc(int mode, bool tc) {
    return tc ? heun_fn_b<NP, B, G, true>(mode) : heun_fn_b<NP, B, G, false>(mode);
}
// consumer threads per element of the Heun kernel: P7 4 (chunks of 64), P5 SEM_HEUN_G5 (default 4:
// B1 1.044 -> 0.779 ms per step against 1 thread per element; 2: 0.803)
int heun_group(int np) {
    static int g5 = -1;
    if (g5 < 0) { const char *e = getenv("SEM_HEUN_G5"); g5 = e ? atoi(e) : 4; if (g5 != 1 && g5 != 2 && g5 != 4) g5 = 4; }
    return np == 36 ? 4 : np == 21 ? g5 : 1;
}
int heun_group(int np, int B) {
    return np == 21 && B < 128 ? 4 : heun_group(np);
}
// tc: the tensor-core element products (only where heun_tc holds); heun_use_tc falls back to the
// DFMA wide path when the tensor-core tables do not fit beside the stages (meshes with large chunks
// of local nodes, e.g. the shuffled order at P7)
HFn heun_fn(int np, int B, int mode, bool tc) {
    if (np == 36) return B == 32 ? heun_fn_tc<36, 32, 4>(mode, tc) : heun_fn_tc<36, 64, 4>(mode, tc);  // P7
    if (np == 21) {                                      // P5 (the paper's Benchmark 1 order)
        const int g = heun_group(21);
        if (B == 64) return heun_fn_tc<21, 64, 4>(mode, tc);
        if (B == 32) return heun_fn_tc<21, 32, 4>(mode, tc);
        return g == 4 ? heun_fn_tc<21, 128, 4>(mode, tc) : g == 2 ? heun_fn_b<21, 128, 2>(mode) : heun_fn_b<21, 128>(mode);
    }
    if (np == 6) return B == 128 ? heun_fn_b<6, 128>(mode) : heun_fn_b<6, 256>(mode);
    return B == 128 ? heun_fn_b<10, 128>(mode) : heun_fn_b<10, 256>(mode);
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

}  // namespace

bool heun_supported(int np, int B) {
    return ((np == 6 || np == 10) && (B == 128 || B == 256)) || (np == 21 && (B == 32 || B == 64 || B == 128)) ||
           (np == 36 && (B == 32 || B == 64));
}

cudaError_t upload_heun_tables(const RefTables &T, cudaStream_t s) {
    cudaError_t e;
    const int n = T.Np;  // packed [p * n + q]; pageable copies are staged before returning
    std::vector<double> pk[5];
    const double(*src[5])[kMaxNp] = {T.Dr, T.Ds, T.Srr, T.Sss, T.Srs};
    for (int k = 0; k < 5; k++) {
        pk[k].resize(n * n);
        for (int p = 0; p < n; p++)
            for (int q = 0; q < n; q++) pk[k][p * n + q] = src[k][p][q];
    }
    if ((e = cudaMemcpyToSymbolAsync(h_Dr, pk[0].data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(h_Ds, pk[1].data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(h_Srr, pk[2].data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(h_Sss, pk[3].data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(h_Srs, pk[4].data(), sizeof(double) * n * n, 0, cudaMemcpyHostToDevice, s))) return e;
    return cudaMemcpyToSymbolAsync(h_wK, T.wK, sizeof(T.wK), 0, cudaMemcpyHostToDevice, s);
}

cudaError_t launch_geometry_heun(const double *vxy, const int32_t *tri_or, const int32_t *perm, const double *c_in,
                                 int64_t E, int64_t Epad, double *const geo[5], double *detJ, int32_t *bad,
                                 cudaStream_t s) {
    k_geometry_heun<<<nblk(Epad), 256, 0, s>>>(vxy, tri_or, perm, c_in, E, Epad, geo[0], geo[1], geo[2], geo[3],
                                               geo[4], detJ, bad);
    return cudaGetLastError();
}

bool heun_use_tc(const DevChunks &ch, int mode) {
    if (!heun_tc(ch.Np, heun_group(ch.Np, ch.B))) return false;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return heun_smem_bytes(ch.Np, ch.B, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, mode, true) <= (size_t)optin;
}

int heun_grid(const DevChunks &ch, int mode) {
    const bool tc = heun_use_tc(ch, mode);
    const size_t smem = heun_smem_bytes(ch.Np, ch.B, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, mode, tc);
    const HFn fn = heun_fn(ch.Np, ch.B, mode, tc);
    set_smem_h(fn, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, ch.B * heun_group(ch.Np, ch.B) + 32, smem);
    if (occ < 1) occ = 1;
    int64_t g = (int64_t)occ * current_sm_count();
    if (persistent_grid_cap() > 0 && g > persistent_grid_cap()) g = persistent_grid_cap();
    if (g > ch.nchunks) g = ch.nchunks;
    return (int)g;
}

cudaError_t launch_heun(const DevChunks &ch, const HeunParams &p, int mode, cudaStream_t s, const int32_t *list,
                        int64_t nlist) {
    const int64_t n = list ? nlist : ch.nchunks;
    if (n == 0) return cudaSuccess;
    const bool tc = heun_use_tc(ch, mode);
    const size_t smem = heun_smem_bytes(ch.Np, ch.B, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, mode, tc);
    const HFn fn = heun_fn(ch.Np, ch.B, mode, tc);
    cudaError_t e = set_smem_h(fn, smem);
    if (e != cudaSuccess) return e;
    int grid = heun_grid(ch, mode);
    if (grid > n) grid = (int)n;
    fn<<<grid, ch.B * heun_group(ch.Np, ch.B) + 32, smem, s>>>(ch, p, ch.max_local, ch.max_win, 2 * kJdsW, ch.max_nsh, list,
                                                         nlist);
    return cudaGetLastError();
}

// ---- multi-GPU interface (SURVEY §8e with the Heun payload: (R(V), K U) pairs) ----
__global__ void k_if_partial2(const DevChunks ch, const double2 *__restrict__ slot, double2 *__restrict__ xbuf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ch.N_if) return;
    const int64_t s = ch.N_sh - ch.N_if + i;
    double2 y = make_double2(0.0, 0.0);
    for (int j = ch.sh_pstart[s]; j < ch.sh_pstart[s + 1]; j++) { y.x += slot[j].x; y.y += slot[j].y; }
    xbuf[i] = y;
}

__global__ void k_pack2(const double2 *__restrict__ xbuf, const int32_t *__restrict__ send_if, int64_t n,
                        double2 *__restrict__ sendbuf) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) sendbuf[k] = xbuf[send_if[k]];
}

// all ranks' (R(V), K U) of interface node i in ascending rank order, then the
// Heun update of U and W (identical bits on every rank holding the node)
__global__ void k_heun_if(const DevChunks ch, const HeunParams a, const double2 *__restrict__ xbuf,
                          const int32_t *__restrict__ sum_start, const int32_t *__restrict__ sum_src) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ch.N_if) return;
    double2 ab = make_double2(0.0, 0.0);
    for (int j = sum_start[i]; j < sum_start[i + 1]; j++) { ab.x += xbuf[sum_src[j]].x; ab.y += xbuf[sum_src[j]].y; }
    const int64_t id = ch.N_int + ch.N_sh - ch.N_if + i;
    const double u0 = a.U[id], hm = a.hM[id];
    const double yn = src_term(a, id, a.n), yn1 = src_term(a, id, a.n + 1);
    heun_update(u0, hm, ab.x, ab.y, yn, yn1, a.h, a.W[id], a.U[id]);
}

cudaError_t launch_heun_if_partial(const DevChunks &ch, const double *slot, double *xbuf, const int32_t *send_if,
                                   int64_t n_send, double *sendbuf, cudaStream_t s) {
    if (ch.N_if == 0) return cudaSuccess;
    k_if_partial2<<<nblk(ch.N_if), 256, 0, s>>>(ch, reinterpret_cast<const double2 *>(slot),
                                                reinterpret_cast<double2 *>(xbuf));
    if (n_send > 0)
        k_pack2<<<nblk(n_send), 256, 0, s>>>(reinterpret_cast<const double2 *>(xbuf), send_if, n_send,
                                             reinterpret_cast<double2 *>(sendbuf));
    return cudaGetLastError();
}

cudaError_t launch_heun_if(const DevChunks &ch, const HeunParams &p, const double *xbuf, const int32_t *sum_start,
                           const int32_t *sum_src, cudaStream_t s) {
    if (ch.N_if == 0) return cudaSuccess;
    k_heun_if<<<nblk(ch.N_if), 256, 0, s>>>(ch, p, reinterpret_cast<const double2 *>(xbuf), sum_start, sum_src);
    return cudaGetLastError();
}

cudaError_t launch_heun_fix(const DevChunks &ch, const HeunParams &p, cudaStream_t s) {
    if (ch.N_sh - ch.N_if == 0) return cudaSuccess;
    // threads per KH8 block: 128 (C4 Heun step 1.0048 -> 1.0030 ms against 256); SEM_KH8_THREADS overrides
    static const int bt = [] {
        const char *v = getenv("SEM_KH8_THREADS");
        const int b = v ? atoi(v) : 128;
        return (b == 64 || b == 128 || b == 256 || b == 512) ? b : 128;
    }();
    const int64_t n = ch.N_sh - ch.N_if;
    k_heun_fix<<<(unsigned)((n + bt - 1) / bt), bt, 0, s>>>(ch, p);
    return cudaGetLastError();
}

cudaError_t launch_v_out(const double *V, const int32_t *perm, int64_t E, int np, int B, double *out, cudaStream_t s) {
    if (E == 0) return cudaSuccess;
    k_v_out<<<nblk(E * np * 2), 256, 0, s>>>(V, perm, E, np, B, out);
    return cudaGetLastError();
}

cudaError_t launch_v_in(const double *in, const int32_t *perm, int64_t E, int np, int B, double *V, cudaStream_t s) {
    if (E == 0) return cudaSuccess;
    k_v_in<<<nblk(E * np * 2), 256, 0, s>>>(in, perm, E, np, B, V);
    return cudaGetLastError();
}

}  // namespace sem
