// common.cuh — device helpers shared by the query-path kernels.
#pragma once

#include <cstdint>

#include "pqtg_internal.h"

namespace pqtg {
namespace dev {

constexpr int kThreads = 256;
constexpr uint64_t kSentinel = ~0ull;

// Per-query stage clock (pqtg_workspace_query_times): thread 0 of a query's CTA stores its start
// complemented (so one atomicMax from a zeroed record keeps the earliest start) and every warp's
// lane 0 its end (the latest end wins); p.qtime is [query][3 stages][start, end] in
// globaltimer nanoseconds, or null when the workspace does not collect them.
// Programmatic dependent launch (PDL): a dependent kernel waits for its predecessor's results
// (and their memory flush) with griddep_wait(); a kernel lets its dependents launch early with
// griddep_launch(). Both are no-ops when the launch has no programmatic dependency.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <class PR>
__device__ __forceinline__ void qt_begin(const PR& p, uint64_t q, int stage) {
    if (p.qtime && threadIdx.x == 0) atomicMax(p.qtime + (q * 3 + stage) * 2, ~gtimer_ns());
}
template <class PR>
__device__ __forceinline__ void qt_end(const PR& p, uint64_t q, int stage) {
    if (p.qtime && (threadIdx.x & 31) == 0) atomicMax(p.qtime + (q * 3 + stage) * 2 + 1, gtimer_ns());
}

__device__ __forceinline__ float sq_step(float acc, float a, float b) {
    const float d = __fsub_rn(a, b);
    return __fadd_rn(acc, __fmul_rn(d, d));
}

// fp32 -> u32 preserving order (with -0.0 folded onto +0.0 so it ties like operator<).
// one 256-bit read-only global load (sm_100: LDG.E.ENL2.256), p 32-byte aligned
__device__ __forceinline__ void ldg256(const void* p, uint4& a, uint4& b) {
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
}

__device__ __forceinline__ uint32_t orderable(float x) {
    uint32_t u = __float_as_uint(x);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float unorderable(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
    return __uint_as_float(u);
}

// pick_slope_table (binorder.cpp:52-65): fp64 gaps, nearest slope 1.08^k in log space,
// k = clamp(lround(log(gb / ga) / log(1.08)), -5, 4). The fp64 log is a long dependent
// sequence on one thread, so a fp32 estimate decides whenever it is provably on the same side
// of every rounding boundary: its error (fp32 logf <= 2 ulp plus the ratio's rounding) is
// below 2e-4 for |log ratio| <= 64, and the estimate must be >= 1e-3 from a half-integer or
// beyond the clamp; otherwise the reference's fp64 formula runs.
__device__ inline uint32_t pick_slope(const float* a, const float* b, uint32_t len, double log108) {
    if (len < 2) return kSlopeOne;
    const double ga = (double)a[1] - (double)a[0];
    const double gb = (double)b[1] - (double)b[0];
    if (!(ga > 0.0) || !(gb > 0.0)) return kSlopeOne;
    const double ratio = gb / ga;
    const float rf = (float)ratio;
    const float lf = logf(rf);
    long long k;
    if (rf > 0.0f && rf < 3.0e38f && fabsf(lf) <= 64.0f) {
        const float kf = lf * (float)(1.0 / log108);
        const float frac = fabsf(kf - truncf(kf));  // distance pattern to the .5 boundary
        if (kf <= -6.0f || kf >= 5.0f) return kf < 0.0f ? 0u : 9u;  // clamped either way
        if (fabsf(frac - 0.5f) >= 1e-3f) {
            k = (long long)roundf(kf);  // round half away from zero, as lround
            k = k < -5 ? -5 : (k > 4 ? 4 : k);
            return (uint32_t)(k + 5);
        }
    }
    k = llround(log(ratio) / log108);
    k = k < -5 ? -5 : (k > 4 ? 4 : k);
    return (uint32_t)(k + 5);
}

// pick_slope_table for one of a query's pair streams from its sorted level-2 lists l2d[P][W]
// in global memory: pair 0 = lists (0,1), pair 1 = lists (2,3) when P = 4 (binorder.cpp:52-65,
// :237); kSlopeOne for the streams a query does not have.
__device__ inline uint32_t query_slope(const DevParams& p, const float* l2d, uint32_t pair) {
    const uint32_t W = p.W;
    if (p.P < 2 || W < 2 || (pair == 1 && p.P != 4)) return kSlopeOne;
    const float* la = l2d + (size_t)(2 * pair) * W;
    const float* lb = la + W;
    const float a[2] = {la[0], la[1]}, b[2] = {lb[0], lb[1]};
    return pick_slope(a, b, W, p.log108);
}

// ------------------------------------------------------------------ bulk async copies
__device__ __forceinline__ uint32_t smem_addr(const void* ptr) {
    return (uint32_t)__cvta_generic_to_shared(ptr);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// TMA 1-D bulk copy global -> shared (SASS UBLKCP); completes `bytes` on the mbarrier.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase), "r"(0x989680u)  // suspend hint: sleep until the phase flips, not spin
        : "memory");
}

// ------------------------------------------------------------------ block scan helpers
__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive block scan of one u64 per thread; returns the exclusive prefix, *total = sum.
__device__ inline uint64_t block_excl_scan(uint64_t v, uint64_t* warp_sums, uint64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    uint64_t incl = warp_incl_scan(v);
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t s = lane < nwarps ? warp_sums[lane] : 0;
        s = warp_incl_scan(s);
        if (lane < nwarps) warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t before = warp == 0 ? 0 : warp_sums[warp - 1];
    *total = warp_sums[nwarps - 1];
    __syncthreads();
    return before + incl - v;
}


}  // namespace dev
}  // namespace pqtg
