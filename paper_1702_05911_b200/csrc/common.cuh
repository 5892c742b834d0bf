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
