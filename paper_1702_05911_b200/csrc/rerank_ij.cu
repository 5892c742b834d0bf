// rerank_ij.cu — K5 fast path: line-quantized re-rank (linequant.cpp:169-182) + top-k
// (search.cpp:221-257) for indexes with k1 <= 16 and 1-byte pairs, whose device codes store
// each part's centroid pair as (i << 4 | j) instead of the pair id (index_prep.cpp).
//
// One thread per candidate; the code row (L × (λ, ij) bytes, slot order) is read with 16-byte
// loads into registers and its parts are summed in the reference's order. Per part:
//     b2 = fine[f][i]                   a 16-float row per part: the 32 lanes of a warp touch
//                                       at most 16 addresses, all in distinct banks
//                                       (duplicates broadcast) — conflict-free;
//     (E, c2) = T[f][i << 4 | j]        per-query table, E = (a2 − b2) − c2 with a2 = fine[f][j]
//                                       and c2 = d2[f][i][j]: the reference's own intermediate
//                                       (linequant.hpp:85), built once per query;
//     part = (b2 + (λ·λ)·c2) + λ·E      exactly linequant.hpp:83-85's rounding.
// Shared memory: T (L × 2 KB), fine (L × 64 B), candidate keys, range offsets (cached up to
// kRangeCache, else read from global memory); 512 threads per CTA, two CTAs per SM.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kIjThreads = 512;
constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // no id: the candidate belongs to another shard
constexpr uint32_t kRangeCache = 1024;

struct IjLayout {
    size_t t, fine, keys, sel, coff, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline IjLayout ij_layout(uint32_t L, uint32_t budget, uint32_t sel_cap) {
    IjLayout l{};
    size_t o = 0;
    l.t = o;  // offset 0: compile-time part offsets become load immediates
    o += (size_t)L * 256 * 8;
    l.fine = o;
    o += (size_t)L * 16 * 4;
    l.keys = o;
    o += al16((size_t)budget * 8);
    l.sel = o;
    o += al16((size_t)sel_cap * 8);
    l.coff = o;
    o += al16((size_t)(budget < kRangeCache ? budget : kRangeCache) * 4);
    l.total = o;
    return l;
}

}  // namespace

template <int LT>
__global__ void __launch_bounds__(kIjThreads, 2)
    rerank_ij_kernel(DevParams p, uint32_t k, uint32_t sel_cap, const float* __restrict__ fine_in,
                     const uint2* __restrict__ ranges, const uint32_t* __restrict__ nranges,
                     const uint32_t* __restrict__ ncand, uint32_t* __restrict__ out_ids,
                     float* __restrict__ out_dists, uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k1 = p.k1, budget = p.budget;
    const IjLayout lay = ij_layout(LT, budget, sel_cap);
    float2* T = reinterpret_cast<float2*>(smem);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + lay.keys);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + lay.sel);
    uint32_t* coff = reinterpret_cast<uint32_t*>(smem + lay.coff);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    const int tid = threadIdx.x;
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2* qr = ranges + q * (uint64_t)budget;

    for (uint32_t i = tid; i < LT * 16; i += blockDim.x) {
        const uint32_t f = i >> 4, c = i & 15;
        fine[i] = c < k1 ? fine_in[q * LT * k1 + f * k1 + c] : 0.0f;
    }
    const bool cached = R <= kRangeCache;
    if (cached)
        for (uint32_t r = tid; r < R; r += blockDim.x) coff[r] = qr[r].y;
    if (tid == 0) s_count = 0;
    __syncthreads();
    // T[f][i << 4 | j] = (E, c2) for every pair; entries with i >= j are never referenced
    for (uint32_t idx = tid; idx < LT * 256; idx += blockDim.x) {
        const uint32_t f = idx >> 8, i = (idx >> 4) & 15u, j = idx & 15u;
        if (i < k1 && j < k1) {
            const float c2 = __ldg(p.c2ij + idx);
            const float b2 = fine[f * 16 + i], a2 = fine[f * 16 + j];
            T[idx] = make_float2(__fsub_rn(__fsub_rn(a2, b2), c2), c2);
        }
    }
    __syncthreads();

    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    const bool sharded = p.shard_hi > p.shard_lo;
    constexpr int kVec = (2 * LT + 15) / 16;
    uint32_t mine = 0;
    // candidate j's code row and id, fetched one iteration ahead (software pipelining)
    auto fetch = [&](uint32_t j, uint4* v, uint32_t& id) {
        uint32_t lo = 0, hi = R - 1;  // range holding candidate j
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            const uint32_t cm = cached ? coff[mid] : __ldg(&qr[mid].y);
            if (cm <= j) lo = mid; else hi = mid - 1;
        }
        const uint2 rl = __ldg(qr + lo);
        const uint64_t pos = (uint64_t)rl.x + (j - rl.y);
        id = kInvalid;
        if (!sharded || (pos >= p.shard_lo && pos < p.shard_hi)) {
            const uint64_t lp = pos - p.shard_lo;
            id = __ldg(p.ids + lp);
            const uint4* r4 = reinterpret_cast<const uint4*>(p.codes + lp * p.row_bytes);
#pragma unroll
            for (int i = 0; i < kVec; ++i) v[i] = __ldg(r4 + i);
        }
    };
    uint4 vn[kVec];
    uint32_t idn = kInvalid;
    if (tid < C) fetch(tid, vn, idn);
    for (uint32_t j = tid; j < C; j += blockDim.x) {
        uint4 v[kVec];
#pragma unroll
        for (int i = 0; i < kVec; ++i) v[i] = vn[i];
        const uint32_t id = idn;
        if (j + blockDim.x < C) fetch(j + blockDim.x, vn, idn);
        uint64_t key = kSentinel;
        if (id != kInvalid) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
            float total = 0.0f;
#pragma unroll
            for (int f = 0; f < LT; ++f) {
                const uint32_t half = w[f >> 1] >> ((f & 1) * 16);  // λ | (i << 4 | j) << 8
                const uint32_t ij = (half >> 8) & 0xFFu;
                const float b2 = fine[f * 16 + (ij >> 4)];
                const float2 ec = T[f * 256 + ij];
                const float lam = __fmul_rn(__uint2float_rn(half & 0xFFu), inv255);
                const float part = __fadd_rn(__fadd_rn(b2, __fmul_rn(__fmul_rn(lam, lam), ec.y)), __fmul_rn(lam, ec.x));
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

template <int LT>
void allow(int optin) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, rerank_ij_kernel<LT>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(rerank_ij_kernel<LT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

size_t ij_smem(const DevParams& p, uint32_t k) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    return ij_layout(p.L, p.budget, np2(kk > 0 ? kk : 1)).total;
}

}  // namespace

bool rerank_ij_ok(const DevParams& p, uint32_t k) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return p.code_ij && (p.L == 16 || p.L == 32 || p.L == 64) && ij_smem(p, k) + 4096 <= (size_t)optin;
}

void configure_rerank_ij() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    allow<16>(optin);
    allow<32>(optin);
    allow<64>(optin);
}

void launch_rerank_ij(const DevParams& p, uint64_t nq, uint32_t k, const WsSlice& ws, uint32_t* ids, float* dists,
                      uint32_t* counts, cudaStream_t s) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    const uint32_t cap = np2(kk > 0 ? kk : 1);
    const size_t sm = ij_smem(p, k);
#define PQTG_IJ(LT)                                                                                         \
    rerank_ij_kernel<LT><<<(unsigned)nq, kIjThreads, sm, s>>>(p, k, cap, ws.fine, ws.ranges, ws.nranges, \
                                                             ws.ncand, ids, dists, counts)
    switch (p.L) {
    case 16: PQTG_IJ(16); break;
    case 32: PQTG_IJ(32); break;
    default: PQTG_IJ(64); break;
    }
#undef PQTG_IJ
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
