// dev_common.cuh -- device helpers shared by the step kernels (step.cu, heun.cu):
// the Ricker wavelet (Algorithm 3 source, reading R7), mbarrier / TMA bulk-copy
// / cp.async PTX wrappers and the consumer-warp named barrier.  Product path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace sem {
namespace {

__device__ __forceinline__ double ricker_dev(double t, double f0, double t0) {
    const double tau = t - t0;
    double a = 3.14159265358979323846 * f0 * tau;
    a = a * a;
    return (1.0 - 2.0 * a) * exp(-a);
}

// ---- checked builds (-DSEM_CHECKED; tools/checked_build.sh) --------------------
// compute-sanitizer is closed on this GPU pool, so the asynchronous pipelines are checked by
// a build of their own: device-side bounds and consistency asserts (SEM_DCHECK: printf + trap,
// which surfaces as SEM_E_CUDA), poisoning of every shared-memory buffer before it is handed
// back to its producer (a read of a stage, window or entry buffer that the barriers did not
// order after its refill sees NaN or an out-of-range index instead of stale data), and
// pseudo-random delays (chaos_delay) that perturb the producer / consumer timing.
#ifdef SEM_CHECKED
#define SEM_DCHECK(cond, what)                                                                           \
    do {                                                                                                 \
        if (!(cond)) {                                                                                   \
            printf("SEM_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,        \
                   (int)blockIdx.x, (int)threadIdx.x);                                                   \
            __trap();                                                                                    \
        }                                                                                                \
    } while (0)
constexpr bool kChecked = true;
__device__ __forceinline__ void chaos_delay(unsigned key) {
    unsigned h = key * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    if ((h & 3) == 0) __nanosleep(100 + (h >> 16) % 4000);
}
#else
#define SEM_DCHECK(cond, what) \
    do {                       \
    } while (0)
constexpr bool kChecked = false;
__device__ __forceinline__ void chaos_delay(unsigned) {}
#endif
__device__ __forceinline__ double poison_f64() { return __longlong_as_double(0x7FF8DEADDEADDEADll); }

// ---- PTX helpers: mbarrier + TMA bulk copy -----------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The same wait written out at the call site (distinct source lines for ncu's
// per-line stall attribution: which barrier the consumers wait on).
#define MBAR_WAIT_INLINE(bar, parity)                                              \
    asm volatile(                                                                  \
        "{\n"                                                                      \
        ".reg .pred p;\n"                                                          \
        "WAIT_%=:\n"                                                               \
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"                  \
        "@!p bra WAIT_%=;\n"                                                       \
        "}\n" ::"r"(smem_u32(bar)),                                                \
        "r"(parity)                                                                \
        : "memory")

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void tma_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 8-byte asynchronous global -> shared copy (LDGSTS) and the per-thread
// mbarrier arrive that fires when all of this thread's cp.async have landed.
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int B>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(B) : "memory");
}

// ---- host helpers of the persistent launches -----------------------------------
// cudaFuncSetAttribute applies per device context: the raised max-dynamic-smem value
// is cached per (device, kernel), only ever raised, under a lock.
inline cudaError_t raise_max_smem(const void *kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> cur;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t &c = cur[{dev, kernel}];
    if (bytes <= c) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c = bytes;
    return e;
}
// SM count of the current device
inline int current_sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
}
// SEM_K7_GRID=n caps the persistent step kernels' grids (K7, KH7) at n CTAs, so tests can
// force many chunks per CTA (stage reuse, window hand-off) on small meshes; 0/unset = none.
// Read at every launch configuration (host side, outside any captured graph's replays).
inline int64_t persistent_grid_cap() {
    const char *e = getenv("SEM_K7_GRID");
    const long long n = e ? atoll(e) : 0;
    return (int64_t)(n > 0 ? n : 0);
}

}  // namespace
// Programmatic dependent launch (sm_90+): let the next kernel in the stream start its
// prologue now / wait until the preceding kernel has completed and its writes are visible.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace sem
