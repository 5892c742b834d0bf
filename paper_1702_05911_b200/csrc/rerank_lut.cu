// rerank_lut.cu — K5 variant: thread-per-candidate line-quantized re-rank with a per-query
// (b2, E, c2) table (linequant.cpp:169-182, search.cpp:221-257), for 1-byte pair ids and a
// compile-time p_line.
//
// Each thread owns one candidate at a time: its code row (L × (λ, pair) bytes, slot order) is
// loaded into registers with 16-byte loads, then the fine parts are summed in the reference's
// order with one 16-byte shared-memory lookup per part into
//     lut[f][pid] = (b2, E = (a2 - b2) - c2, c2, 0),   b2 = fine[f][i], a2 = fine[f][j],
// i.e. the exact fp32 intermediates of line_part_distance, so part = (b2 + (λ·λ)·c2) + λ·E
// rounds identically. Parts are compile-time, so a part costs ~12 instructions; lookups of
// 32 random pairs share banks (the price of this variant; rerank_fast.cu avoids it).
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kLutThreads = 256;
constexpr uint32_t kLutPairs = 128;  // LUT row stride in pairs (npairs <= 128, i.e. k1 <= 16)

struct LutLayout {
    size_t lut, keys, sel, fine, pairs, coff, total;
};

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline LutLayout lut_layout(uint32_t L, uint32_t k1, uint32_t npairs, uint32_t budget,
                                                uint32_t sel_cap) {
    LutLayout l{};
    size_t o = 0;
    l.lut = o;  // offset 0: part offsets are compile-time immediates
    o += (size_t)L * kLutPairs * 16;
    l.keys = o;
    o += a16((size_t)budget * 8);
    l.sel = o;
    o += a16((size_t)sel_cap * 8);
    l.fine = o;
    o += a16((size_t)L * k1 * 4);
    l.pairs = o;
    o += a16((size_t)npairs * 4);
    l.coff = o;
    o += a16((size_t)budget * 4);
    l.total = o;
    return l;
}

}  // namespace

template <int LT>
__global__ void __launch_bounds__(kLutThreads)
    rerank_lut_kernel(DevParams p, uint32_t k, uint32_t sel_cap, const float* __restrict__ fine_in,
                      const uint2* __restrict__ ranges, const uint32_t* __restrict__ nranges,
                      const uint32_t* __restrict__ ncand, uint32_t* __restrict__ out_ids,
                      float* __restrict__ out_dists, uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k1 = p.k1, npairs = p.npairs, budget = p.budget;
    const LutLayout lay = lut_layout(LT, k1, npairs, budget, sel_cap);
    unsigned char* lut = smem;
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + lay.keys);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + lay.sel);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    uint32_t* spairs = reinterpret_cast<uint32_t*>(smem + lay.pairs);
    uint32_t* coff = reinterpret_cast<uint32_t*>(smem + lay.coff);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    const int tid = threadIdx.x;
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2* qr = ranges + q * (uint64_t)budget;

    for (uint32_t i = tid; i < LT * k1; i += blockDim.x) fine[i] = fine_in[q * LT * k1 + i];
    for (uint32_t i = tid; i < npairs; i += blockDim.x) spairs[i] = __ldg(p.pairs + i);
    for (uint32_t r = tid; r < R; r += blockDim.x) coff[r] = qr[r].y;
    if (tid == 0) s_count = 0;
    __syncthreads();
    for (uint32_t idx = tid; idx < LT * npairs; idx += blockDim.x) {
        const uint32_t f = idx / npairs, pid = idx - f * npairs;
        const uint32_t pr = spairs[pid];
        const float b2 = fine[f * k1 + (pr & 0xFFFFu)];
        const float a2 = fine[f * k1 + (pr >> 16)];
        const float c2 = __ldg(p.c2 + idx);  // c2 is [f][pid]: idx == f * npairs + pid
        reinterpret_cast<float4*>(lut)[f * kLutPairs + pid] =
            make_float4(b2, __fsub_rn(__fsub_rn(a2, b2), c2), c2, 0.0f);
    }
    __syncthreads();

    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    const bool sharded = p.shard_hi > p.shard_lo;
    constexpr int kVec = (2 * LT + 15) / 16;
    uint32_t mine = 0;
    for (uint32_t j = tid; j < C; j += blockDim.x) {
        uint32_t lo = 0, hi = R - 1;  // range holding candidate j
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (coff[mid] <= j) lo = mid; else hi = mid - 1;
        }
        const uint64_t pos = (uint64_t)__ldg(&qr[lo].x) + (j - coff[lo]);
        uint64_t key = kSentinel;
        if (!sharded || (pos >= p.shard_lo && pos < p.shard_hi)) {
            const uint64_t lp = pos - p.shard_lo;
            const uint32_t id = __ldg(p.ids + lp);
            uint4 v[kVec];
            const uint4* r4 = reinterpret_cast<const uint4*>(p.codes + lp * p.row_bytes);
#pragma unroll
            for (int i = 0; i < kVec; ++i) v[i] = __ldg(r4 + i);
            const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
            float total = 0.0f;
#pragma unroll
            for (int f = 0; f < LT; ++f) {
                const uint32_t half = (w[f >> 1] >> ((f & 1) * 16)) & 0xFFFFu;  // (λ | pid << 8)
                const float4 e = *reinterpret_cast<const float4*>(lut + ((size_t)f * kLutPairs * 16) +
                                                                  ((half >> 4) & 0xFF0u));
                const float lam = __fmul_rn(__uint2float_rn(half & 0xFFu), inv255);
                const float part = __fadd_rn(__fadd_rn(e.x, __fmul_rn(__fmul_rn(lam, lam), e.z)), __fmul_rn(lam, e.y));
                total = __fadd_rn(total, part);
            }
            key = ((uint64_t)orderable(total) << 32) | id;
            ++mine;
        }
        keys[j] = key;
    }
    if (mine) atomicAdd(&s_count, mine);
    __syncthreads();
    const uint32_t nvalid = s_count;
    const uint32_t kk = nvalid < k ? nvalid : k;
    block_topk(keys, C, kk, sel, sel_cap, hist, s_sel);
    write_topk(sel, kk, k, q, out_ids, out_dists, out_counts);
}

namespace {
uint32_t np2(uint32_t x) {
    uint32_t r = 1;
    while (r < x) r <<= 1;
    return r;
}
}  // namespace

size_t rerank_lut_smem(const DevParams& p, uint32_t k) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    return lut_layout(p.L, p.k1, p.npairs, p.budget, np2(kk > 0 ? kk : 1)).total;
}

bool rerank_lut_ok(const DevParams& p, uint32_t k) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return p.pw == 1 && p.npairs <= kLutPairs && (p.L == 32 || p.L == 16) &&
           rerank_lut_smem(p, k) + 4096 <= (size_t)optin;
}

void configure_rerank_lut() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, rerank_lut_kernel<32>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(rerank_lut_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, rerank_lut_kernel<16>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(rerank_lut_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

void launch_rerank_lut(const DevParams& p, uint64_t nq, uint32_t k, Workspace& ws, uint32_t* ids, float* dists,
                       uint32_t* counts, cudaStream_t s) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    const uint32_t cap = np2(kk > 0 ? kk : 1);
    const size_t sm = rerank_lut_smem(p, k);
    if (p.L == 32)
        rerank_lut_kernel<32><<<(unsigned)nq, kLutThreads, sm, s>>>(p, k, cap, ws.fine, ws.ranges, ws.nranges,
                                                                   ws.ncand, ids, dists, counts);
    else
        rerank_lut_kernel<16><<<(unsigned)nq, kLutThreads, sm, s>>>(p, k, cap, ws.fine, ws.ranges, ws.nranges,
                                                                   ws.ncand, ids, dists, counts);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
