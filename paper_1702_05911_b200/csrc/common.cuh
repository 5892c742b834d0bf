// common.cuh — device helpers shared by the query-path kernels.
#pragma once

#include <cstdint>

#include "pqtg_internal.h"

namespace pqtg {
namespace dev {

constexpr int kThreads = 256;
constexpr uint64_t kSentinel = ~0ull;

__device__ __forceinline__ float sq_step(float acc, float a, float b) {
    const float d = __fsub_rn(a, b);
    return __fadd_rn(acc, __fmul_rn(d, d));
}

// fp32 -> u32 preserving order (with -0.0 folded onto +0.0 so it ties like operator<).
__device__ __forceinline__ uint32_t orderable(float x) {
    uint32_t u = __float_as_uint(x);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float unorderable(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
    return __uint_as_float(u);
}

// pick_slope_table (binorder.cpp:52-65): fp64 gaps, nearest slope 1.08^k in log space.
__device__ inline uint32_t pick_slope(const float* a, const float* b, uint32_t len, double log108) {
    if (len < 2) return kSlopeOne;
    const double ga = (double)a[1] - (double)a[0];
    const double gb = (double)b[1] - (double)b[0];
    if (!(ga > 0.0) || !(gb > 0.0)) return kSlopeOne;
    const double ratio = gb / ga;
    long long k = llround(log(ratio) / log108);
    k = k < -5 ? -5 : (k > 4 ? 4 : k);
    return (uint32_t)(k + 5);
}

// pick_slope_table for a query's pair streams from its sorted level-2 lists l2d[P][W] in
// global memory: (lists 0,1) and, for P = 4, (lists 2,3) (binorder.cpp:52-65, :237).
__device__ inline void query_slopes(const DevParams& p, const float* l2d, uint32_t& ta, uint32_t& tb) {
    ta = kSlopeOne;
    tb = kSlopeOne;
    const uint32_t W = p.W;
    if (p.P < 2 || W < 2) return;
    float a[2], b[2];
    a[0] = l2d[0];
    a[1] = l2d[1];
    b[0] = l2d[W];
    b[1] = l2d[W + 1];
    ta = pick_slope(a, b, W, p.log108);
    if (p.P == 4) {
        a[0] = l2d[2 * W];
        a[1] = l2d[2 * W + 1];
        b[0] = l2d[3 * W];
        b[1] = l2d[3 * W + 1];
        tb = pick_slope(a, b, W, p.log108);
    }
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
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
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
