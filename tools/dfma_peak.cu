// dfma_peak.cu -- FP64 FMA throughput microbenchmark ("measure a DFMA
// microbenchmark and report it"; the FP64 roof of the P5/P7 kernels).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dfma_peak tools/dfma_peak.cu
//   ./dfma_peak > profiles/dfma_peak.json
// Each thread runs 16 independent FMA chains; best of 10 timed launches.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = nsm * 8, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flop = 2.0 * 16 * (double)iters * threads * blocks;
    const double tf = flop / (best * 1e-3) / 1e12;
    printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
           "\"per_sm_per_clk_fma_at_max_clock\": %.2f, \"how\": \"16 independent DFMA chains per thread, "
           "%d x %d threads, %d iterations, best of 10, CUDA events\"}\n",
           tf, best, nsm, clk / 1e3, tf * 1e12 / 2 / nsm / (clk * 1e3), blocks, threads, iters);
    return cudaGetLastError() != cudaSuccess;
}
