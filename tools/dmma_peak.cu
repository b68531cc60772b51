// dmma_peak.cu -- FP64 tensor-core (DMMA) throughput microbenchmark beside the DFMA one
// (tools/dfma_peak.cu): the roof of the tensor-core element products (K7 at P6/P7, Heun at P5/P7).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_peak tools/dmma_peak.cu
//   ./dmma_peak > profiles/dmma_peak.json
// Legs: mma.sync m8n8k4 f64 (8 independent accumulator tiles per warp), m16n8k16 f64 (4 tiles),
// and m8n8k4 with DFMA chains interleaved in the same warps (do the two share the FP64 pipe?).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5, %6, %7, %8, %9, %10, %11}, "
        "{%12, %13, %14, %15}, {%0, %1, %2, %3};\n"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// MODE 0: m8n8k4 only; 1: m16n8k16 only; 2: m8n8k4 + 8 DFMA chains per mma; 3: DFMA chains only
template <int MODE>
__global__ void k_peak(double *out, int iters) {
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double acc[8][2], x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { acc[i][0] = acc[i][1] = i; x[i] = i * 0.5; }
    double d4[4][4], a8[8], b4[4];
#pragma unroll
    for (int i = 0; i < 4; i++) { d4[i][0] = d4[i][1] = d4[i][2] = d4[i][3] = i; b4[i] = b + i * 1e-9; }
#pragma unroll
    for (int i = 0; i < 8; i++) a8[i] = a + i * 1e-9;
    for (int it = 0; it < iters; it++) {
        if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 4; i++) mma16816(d4[i], a8, b4);
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (MODE != 3) mma884(acc[i][0], acc[i][1], a, b);
                if (MODE >= 2) {
#pragma unroll
                    for (int j = 0; j < 8; j++) x[j] = fma(x[j], a, b);
                }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1] + x[i];
#pragma unroll
    for (int i = 0; i < 4; i++) s += d4[i][0] + d4[i][1] + d4[i][2] + d4[i][3];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
float time_leg(double *out, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_peak<MODE><<<blocks, threads>>>(out, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        k_peak<MODE><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = nsm * 4, iters = 2048;
    const double warps = (double)blocks * threads / 32;
    const float t0 = time_leg<0>(out, blocks, threads, iters);
    const float t1 = time_leg<1>(out, blocks, threads, iters);
    const float t2 = time_leg<2>(out, blocks, threads, iters);
    const float t3 = time_leg<3>(out, blocks, threads, iters);
    const double f884 = 2.0 * 256 * 8 * iters * warps, f16816 = 2.0 * 2048 * 4 * iters * warps;
    const double fdfma = 2.0 * 64 * iters * warps * 32;  // 8 x 8 chains per iteration per thread
    printf("{\"dmma_m8n8k4_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, "
           "\"mixed_ms\": %.4f, \"dmma_alone_ms\": %.4f, \"dfma_alone_ms\": %.4f, \"dfma_alone_tflops\": %.3f, "
           "\"mixed_vs_sum\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, \"how\": \"mma.sync f64, %d x %d threads, "
           "%d iterations, independent accumulators, best of 10, CUDA events; mixed = the same m8n8k4 work with "
           "64 DFMA per thread per iteration interleaved (mixed_vs_sum = mixed / (dmma alone + dfma alone): "
           "1 = one shared pipe, max/sum = separate pipes)\"}\n",
           f884 / (t0 * 1e-3) / 1e12, f16816 / (t1 * 1e-3) / 1e12, t2, t0, t3, fdfma / (t3 * 1e-3) / 1e12,
           t2 / (t0 + t3), nsm, clk / 1e3, blocks, threads, iters);
    return cudaGetLastError() != cudaSuccess;
}
