// step.cu -- sm_100a kernels of the leapfrog step (product path).
//
//  K6  launch_geometry   G_e = c_e^2 detJ J^-1 J^-T (3 fp64), detJ
//      assemble_mass     M-bar_nu = sum detJ w^M_q, dt^2 / M-bar
//  K7  launch_k7         per chunk (one CTA): gather U^n into shared memory,
//                        y_e = K^e u_e, colour-ordered shared-memory scatter,
//                        fused leapfrog update of the chunk's interior nodes,
//                        partial sums for shared nodes                   (Alg. 1+2+3)
//  K8  launch_k8         shared nodes: add the per-chunk partials in chunk
//                        order, then the same fused update
//
// Element stiffness (readings R2, R5): K^e = Grr*Srr + Gss*Sss + Grs*Srs, with
// S_ab = D_a^T W D_b (+ transpose for rs) from the reference tables.  It is
// the composition of Algorithm 1's gradient and Algorithm
// 2's weighted divergence with F = c^2 I, B = -I, and the
// FK/BK precalculation pushed one step further
// into the reference matrices, as PAPER.md:1568 suggests.
#include <cuda_runtime.h>

#include "kernels.h"

namespace sem {

namespace {

constexpr int kThreads = 256;

__constant__ double c_Srr[kMaxNp][kMaxNp];
__constant__ double c_Sss[kMaxNp][kMaxNp];
__constant__ double c_Srs[kMaxNp][kMaxNp];
__constant__ double c_wM[kMaxNp];

inline unsigned blocks_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    return (unsigned)b;
}

__device__ __forceinline__ double ricker_dev(double t, double f0, double t0) {
    const double tau = t - t0;
    double a = 3.14159265358979323846 * f0 * tau;
    a = a * a;
    return (1.0 - 2.0 * a) * exp(-a);
}

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

// ---- lumped mass with the chunk machinery ------------------------------------
template <int NP>
__global__ void __launch_bounds__(kThreads) k_mass_chunk(const DevChunks ch, const double *__restrict__ detJ,
                                                         double dt2, double *__restrict__ partial,
                                                         double *__restrict__ dt2M) {
    extern __shared__ double smem[];
    const int c = blockIdx.x, t = threadIdx.x, B = ch.B;
    const int i0 = ch.int_start[c], nint = ch.int_start[c + 1] - i0;
    const int s0 = ch.shl_start[c], nsh = ch.shl_start[c + 1] - s0;
    double *y_s = smem;
    for (int i = t; i < nint + nsh; i += B) y_s[i] = 0.0;
    const int64_t e = (int64_t)c * B + t;
    uint16_t li[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) li[p] = ch.lidx[(int64_t)c * NP * B + p * B + t];
    const int col = ch.color[e];
    const double dj = detJ[e];
    __syncthreads();
    const int ncol = ch.ncolors[c];
    for (int k = 0; k < ncol; k++) {
        if (col == k) {
#pragma unroll
            for (int p = 0; p < NP; p++) y_s[li[p]] += 1.0 * dj * c_wM[p];
        }
        __syncthreads();
    }
    for (int i = t; i < nint; i += B) dt2M[i0 + i] = dt2 / y_s[i];
    for (int k = t; k < nsh; k += B) partial[ch.shl_slot[s0 + k]] = y_s[nint + k];
}

__global__ void k_mass_fix(const DevChunks ch, const double *__restrict__ partial, double dt2,
                           double *__restrict__ dt2M) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ch.N_sh) return;
    double m = 0.0;
    for (int j = ch.sh_pstart[s]; j < ch.sh_pstart[s + 1]; j++) m += partial[j];
    dt2M[ch.N_int + s] = dt2 / m;
}

// ---- K7: stiffness apply + fused leapfrog for one chunk ----------------------
template <int NP>
__global__ void __launch_bounds__(kThreads) k7_step(const DevChunks ch, const StepParams a) {
    extern __shared__ double smem[];
    const int c = blockIdx.x, t = threadIdx.x, B = ch.B;
    const int i0 = ch.int_start[c], nint = ch.int_start[c + 1] - i0;
    const int s0 = ch.shl_start[c], nsh = ch.shl_start[c + 1] - s0;
    double *u_s = smem;
    double *y_s = smem + ch.max_local;

    // element data of this thread (coalesced: [chunk][p][t] and SoA G)
    const int64_t e = (int64_t)c * B + t;
    uint16_t li[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) li[p] = ch.lidx[(int64_t)c * NP * B + p * B + t];
    const double grr = a.Grr[e], gss = a.Gss[e], grs = a.Grs[e];
    const int col = ch.color[e];

    // gather U^n: the chunk's interior window is contiguous, shared nodes listed
    for (int i = t; i < nint; i += B) { u_s[i] = a.U[i0 + i]; y_s[i] = 0.0; }
    for (int k = t; k < nsh; k += B) {
        u_s[nint + k] = a.U[ch.N_int + ch.shl_node[s0 + k]];
        y_s[nint + k] = 0.0;
    }
    __syncthreads();

    double u[NP], y[NP];
#pragma unroll
    for (int p = 0; p < NP; p++) { u[p] = u_s[li[p]]; y[p] = 0.0; }
    // y = K^e u with K^e symmetric: build each K_pq once (p <= q)
#pragma unroll
    for (int p = 0; p < NP; p++) {
#pragma unroll
        for (int q = p; q < NP; q++) {
            const double k = fma(grr, c_Srr[p][q], fma(gss, c_Sss[p][q], grs * c_Srs[p][q]));
            if (q == p) {
                y[p] = fma(k, u[p], y[p]);
            } else {
                y[p] = fma(k, u[q], y[p]);
                y[q] = fma(k, u[p], y[q]);
            }
        }
    }
    // conflict-free, deterministic scatter: one colour at a time
    const int ncol = ch.ncolors[c];
    for (int k = 0; k < ncol; k++) {
        if (col == k) {
#pragma unroll
            for (int p = 0; p < NP; p++) y_s[li[p]] += y[p];
        }
        __syncthreads();
    }
    // fused update of interior nodes: U^{n+1} = 2U^n - U^{n-1} + dt^2/M (f - K U^n)
    for (int i = t; i < nint; i += B) {
        const int id = i0 + i;
        const double f = (id == a.src) ? a.amp * ricker_dev((double)a.n * a.dt, a.f0, a.t0) : 0.0;
        a.Uprev[id] = 2.0 * u_s[i] - a.Uprev[id] + a.dt2M[id] * (f - y_s[i]);
    }
    for (int k = t; k < nsh; k += B) a.partial[ch.shl_slot[s0 + k]] = y_s[nint + k];
}

// ---- K8: shared-node fix-up --------------------------------------------------
__global__ void k8_fix(const DevChunks ch, const StepParams a) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= ch.N_sh) return;
    double y = 0.0;
    for (int j = ch.sh_pstart[s]; j < ch.sh_pstart[s + 1]; j++) y += a.partial[j];
    const int64_t id = ch.N_int + s;
    const double f = (id == a.src) ? a.amp * ricker_dev((double)a.n * a.dt, a.f0, a.t0) : 0.0;
    a.Uprev[id] = 2.0 * a.U[id] - a.Uprev[id] + a.dt2M[id] * (f - y);
}

__global__ void k_scatter_f64(const double *__restrict__ in, const int32_t *__restrict__ map,
                              int64_t n, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[map[i]] = in[i];
}

__global__ void k_gather_f64(const double *__restrict__ in, const int32_t *__restrict__ map,
                             int64_t n, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[map[i]];
}

__global__ void k_nonfinite(const double *__restrict__ a, int64_t n, int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !isfinite(a[i])) atomicMin(flag, (int32_t)i);
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

cudaError_t upload_ref_tables(const RefTables &T, cudaStream_t s) {
    cudaError_t e;
    if ((e = cudaMemcpyToSymbolAsync(c_Srr, T.Srr, sizeof(T.Srr), 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Sss, T.Sss, sizeof(T.Sss), 0, cudaMemcpyHostToDevice, s))) return e;
    if ((e = cudaMemcpyToSymbolAsync(c_Srs, T.Srs, sizeof(T.Srs), 0, cudaMemcpyHostToDevice, s))) return e;
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

cudaError_t assemble_mass(const DevChunks &ch, const double *detJ, double dt, double *partial,
                          double *dt2M, cudaStream_t s) {
    const size_t smem = sizeof(double) * ch.max_local;
    const double dt2 = dt * dt;
    cudaError_t e;
    if (ch.Np == 6) {
        if ((e = set_smem(k_mass_chunk<6>, smem))) return e;
        k_mass_chunk<6><<<(unsigned)ch.nchunks, ch.B, smem, s>>>(ch, detJ, dt2, partial, dt2M);
    } else {
        if ((e = set_smem(k_mass_chunk<10>, smem))) return e;
        k_mass_chunk<10><<<(unsigned)ch.nchunks, ch.B, smem, s>>>(ch, detJ, dt2, partial, dt2M);
    }
    if (ch.N_sh > 0) k_mass_fix<<<blocks_for(ch.N_sh), kThreads, 0, s>>>(ch, partial, dt2, dt2M);
    return cudaGetLastError();
}

cudaError_t launch_k7(const DevChunks &ch, const StepParams &p, cudaStream_t s) {
    const size_t smem = 2 * sizeof(double) * ch.max_local;
    cudaError_t e;
    if (ch.Np == 6) {
        if ((e = set_smem(k7_step<6>, smem))) return e;
        k7_step<6><<<(unsigned)ch.nchunks, ch.B, smem, s>>>(ch, p);
    } else {
        if ((e = set_smem(k7_step<10>, smem))) return e;
        k7_step<10><<<(unsigned)ch.nchunks, ch.B, smem, s>>>(ch, p);
    }
    return cudaGetLastError();
}

cudaError_t launch_k8(const DevChunks &ch, const StepParams &p, cudaStream_t s) {
    if (ch.N_sh == 0) return cudaSuccess;
    k8_fix<<<blocks_for(ch.N_sh), kThreads, 0, s>>>(ch, p);
    return cudaGetLastError();
}

cudaError_t launch_scatter_f64(const double *in, const int32_t *map, int64_t n, double *out,
                               cudaStream_t s) {
    k_scatter_f64<<<blocks_for(n), kThreads, 0, s>>>(in, map, n, out);
    return cudaGetLastError();
}

cudaError_t launch_gather_f64(const double *in, const int32_t *map, int64_t n, double *out,
                              cudaStream_t s) {
    k_gather_f64<<<blocks_for(n), kThreads, 0, s>>>(in, map, n, out);
    return cudaGetLastError();
}

cudaError_t launch_nonfinite(const double *a, int64_t n, int32_t *flag, cudaStream_t s) {
    k_nonfinite<<<blocks_for(n), kThreads, 0, s>>>(a, n, flag);
    return cudaGetLastError();
}

}  // namespace sem
