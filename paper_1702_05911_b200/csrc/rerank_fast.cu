// rerank_fast.cu — K5 fast path: line-quantized re-rank (linequant.cpp:169-182) + top-k
// (search.cpp:221-257) for p_line == 32 and 1-byte pair ids.
//
// Layout of the work: a CTA owns one query; its candidates are split into 8 contiguous
// warp slices; lane l of a warp re-ranks candidates aw + 32r + l (round r). Each lane sums
// its candidate's 32 fine parts in the reference's order, but lane l runs ONE PART BEHIND
// lane l-1 (a skewed pipeline): at every step the 32 lanes touch 32 different fine parts,
// so lookups into the per-query tables, laid out [pair][part], hit 32 different banks.
//
//   per-query tables   lut[pid][f] = (b2, (a2 - b2) - c2)   and   lc2[pid][f] = c2
//                      (b2 = fine[f][i], a2 = fine[f][j], (i, j) = pairs[pid]); every value is
//                      exactly the fp32 intermediate the reference computes, so
//                      part = (b2 + (λ·λ)·c2) + λ·E  rounds identically.
//   code staging       each lane prefetches its next rows with cp.async (16 B) into a private
//                      4-round ring in shared memory, 2 rounds ahead of use.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kFastWarps = 8;
constexpr int kFastThreads = kFastWarps * 32;
constexpr int kSlotBytes = 64;                      // one row: 32 × (λ, pair) bytes
constexpr int kLaneBytes = 4 * kSlotBytes + 16;     // 4-round ring + pad
constexpr uint32_t kInvalidId = 0xFFFFFFFFu;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct FastLayout {
    size_t ring, ids, lut, lc2, fine, pairs, ranges, keys, sel, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline FastLayout fast_layout(uint32_t npairs, uint32_t k1, uint32_t budget, uint32_t sel_cap) {
    FastLayout l{};
    size_t o = 0;
    l.ring = o;
    o += (size_t)kFastThreads * kLaneBytes;
    l.ids = o;
    o += (size_t)kFastThreads * 4 * 4;
    l.lut = o;
    o += align16((size_t)npairs * 32 * 8);
    l.lc2 = o;
    o += align16((size_t)npairs * 32 * 4);
    l.fine = o;
    o += align16((size_t)32 * k1 * 4);
    l.pairs = o;
    o += align16((size_t)npairs * 4);
    l.ranges = o;
    o += align16((size_t)budget * 8);
    l.keys = o;
    o += align16((size_t)budget * 8);
    l.sel = o;
    o += align16((size_t)sel_cap * 8);
    l.total = o;
    return l;
}

}  // namespace

__global__ void __launch_bounds__(kFastThreads, 1)
    rerank_skew_kernel(DevParams p, uint32_t k, uint32_t sel_cap, const float* __restrict__ fine_in,
                       const uint2* __restrict__ ranges, const uint32_t* __restrict__ nranges,
                       const uint32_t* __restrict__ ncand, uint32_t* __restrict__ out_ids,
                       float* __restrict__ out_dists, uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t budget = p.budget, npairs = p.npairs, k1 = p.k1;
    const FastLayout lay = fast_layout(npairs, k1, budget, sel_cap);
    uint8_t* ring = smem + lay.ring;
    uint32_t* ring_ids = reinterpret_cast<uint32_t*>(smem + lay.ids);
    float2* lut = reinterpret_cast<float2*>(smem + lay.lut);
    float* lc2 = reinterpret_cast<float*>(smem + lay.lc2);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    uint2* rg = reinterpret_cast<uint2*>(smem + lay.ranges);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + lay.keys);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + lay.sel);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2* qr = ranges + q * (uint64_t)budget;

    for (uint32_t i = tid; i < 32 * k1; i += blockDim.x) fine[i] = fine_in[q * 32 * k1 + i];
    for (uint32_t r = tid; r < R; r += blockDim.x) rg[r] = qr[r];
    uint32_t* spairs = reinterpret_cast<uint32_t*>(smem + lay.pairs);
    for (uint32_t i = tid; i < npairs; i += blockDim.x) spairs[i] = __ldg(p.pairs + i);
    {
        uint4* z = reinterpret_cast<uint4*>(ring + (size_t)tid * kLaneBytes);
        for (int i = 0; i < kLaneBytes / 16; ++i) z[i] = make_uint4(0, 0, 0, 0);  // pid 0 in unused slots
    }
    if (tid == 0) s_count = 0;
    __syncthreads();
    // per-query tables, [pid][f] so that lanes at distinct parts hit distinct banks
#pragma unroll 4
    for (uint32_t idx = tid; idx < npairs * 32; idx += blockDim.x) {
        const uint32_t pid = idx >> 5, f = idx & 31;
        const uint32_t pr = spairs[pid];
        const float b2 = fine[f * k1 + (pr & 0xFFFFu)];
        const float a2 = fine[f * k1 + (pr >> 16)];
        const float c2 = __ldg(p.c2 + (size_t)f * npairs + pid);
        lut[idx] = make_float2(b2, __fsub_rn(__fsub_rn(a2, b2), c2));
        lc2[idx] = c2;
    }
    __syncthreads();

    // ---- skewed per-warp pipeline
    const uint32_t aw = (uint32_t)((uint64_t)C * warp / kFastWarps);
    const uint32_t bw = (uint32_t)((uint64_t)C * (warp + 1) / kFastWarps);
    const uint32_t nround = (bw - aw + 31) >> 5;
    uint8_t* my = ring + (size_t)tid * kLaneBytes;
    uint32_t* myid = ring_ids + tid * 4;
    const bool sharded = p.shard_hi > p.shard_lo;
    uint32_t cursor = 0;
    bool first = true;

    auto stage = [&](uint32_t r) {
        const uint32_t c = aw + 32 * r + lane;
        const uint32_t slot = r & 3;
        bool issued = false;
        if (r < nround && c < bw) {
            // range holding candidate c: last rr with rg[rr].y <= c (candidate offsets ascend)
            uint32_t lo = first ? 0 : cursor;
            uint32_t hi = first ? R - 1 : min(R - 1, cursor + 32);
            first = false;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (rg[mid].y <= c) lo = mid; else hi = mid - 1;
            }
            cursor = lo;
            const uint64_t pos = (uint64_t)rg[lo].x + (c - rg[lo].y);
            if (!sharded || (pos >= p.shard_lo && pos < p.shard_hi)) {
                const uint64_t lp = pos - p.shard_lo;
                const uint8_t* src = p.codes + lp * kSlotBytes;
                uint8_t* dst = my + slot * kSlotBytes;
#pragma unroll
                for (int i = 0; i < kSlotBytes / 16; ++i) cp_async16(dst + 16 * i, src + 16 * i);
                cp_async4(myid + slot, p.ids + lp);
                issued = true;
            }
        }
        if (!issued) myid[slot] = kInvalidId;
        cp_async_commit();
    };

    stage(0);
    stage(1);
    stage(2);
    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    const int32_t nparts = (int32_t)nround * 32;
    uint32_t mine = 0;
    float acc = 0.0f, done = 0.0f;
    // One fine part of lane l's current candidate; g = lane's running part counter.
    // Branch-free: the finished sum of a candidate (f == 31) is parked in `done` and the
    // accumulator restarts, so the unrolled steps carry no control flow.
    auto step = [&](int32_t g) {
        const uint32_t f = (uint32_t)g & 31u;
        const uint32_t code = *reinterpret_cast<const uint16_t*>(my + (((uint32_t)g & 127u) << 1));
        const uint32_t li = ((code >> 8) << 5) | f;
        const float2 be = lut[li];
        const float c2 = lc2[li];
        const float lam = __fmul_rn(__uint2float_rn(code & 0xFFu), inv255);
        const float part = __fadd_rn(__fadd_rn(be.x, __fmul_rn(__fmul_rn(lam, lam), c2)), __fmul_rn(lam, be.y));
        acc = __fadd_rn(acc, part);
        const bool fin = f == 31u;
        done = fin ? acc : done;
        acc = fin ? 0.0f : acc;
    };
    for (uint32_t m = 0; nround > 0 && m <= nround; ++m) {
        if (m > 0) stage(m + 2);
        cp_async_wait<2>();  // rounds <= m have landed (each lane reads only its own ring)
        const int32_t pb = (int32_t)(m * 32) - lane;
        if (m >= 1 && m < nround) {  // every lane busy for all 32 steps
#pragma unroll
            for (int t = 0; t < 32; ++t) step(pb + t);
        } else {                     // pipeline fill / drain
#pragma unroll 4
            for (int t = 0; t < 32; ++t) {
                const int32_t g = pb + t;
                if (g >= 0 && g < nparts) step(g);
            }
        }
        // each lane finished exactly one candidate in this phase: lane 0 its round m,
        // lanes l > 0 their round m - 1 (at t = l - 1)
        const int32_t r = lane == 0 ? (int32_t)m : (int32_t)m - 1;
        if (r >= 0 && r < (int32_t)nround) {
            const uint32_t c = aw + 32 * (uint32_t)r + lane;
            if (c < bw) {
                const uint32_t id = myid[r & 3];
                uint64_t key = kSentinel;
                if (id != kInvalidId) {
                    key = ((uint64_t)orderable(done) << 32) | id;
                    ++mine;
                }
                keys[c] = key;
            }
        }
    }
    cp_async_wait<0>();
    if (mine) atomicAdd(&s_count, mine);
    __syncthreads();
    const uint32_t nvalid = s_count;
    const uint32_t kk = nvalid < k ? nvalid : k;
    block_topk(keys, C, kk, sel, sel_cap, hist, s_sel);
    write_topk(sel, kk, k, q, out_ids, out_dists, out_counts);
}

namespace {
uint32_t next_pow2_u32(uint32_t x) {
    uint32_t r = 1;
    while (r < x) r <<= 1;
    return r;
}
}  // namespace

size_t rerank_fast_smem(const DevParams& p, uint32_t k) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    return fast_layout(p.npairs, p.k1, p.budget, next_pow2_u32(kk > 0 ? kk : 1)).total;
}

bool rerank_fast_ok(const DevParams& p, uint32_t k) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return p.L == 32 && p.pw == 1 && p.row_bytes == (uint32_t)kSlotBytes &&
           rerank_fast_smem(p, k) + 4096 <= (size_t)optin;
}

void configure_rerank_fast() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, rerank_skew_kernel));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(rerank_skew_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

void launch_rerank_fast(const DevParams& p, uint64_t nq, uint32_t k, Workspace& ws, uint32_t* ids, float* dists,
                        uint32_t* counts, cudaStream_t s) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    const uint32_t cap = next_pow2_u32(kk > 0 ? kk : 1);
    rerank_skew_kernel<<<(unsigned)nq, kFastThreads, rerank_fast_smem(p, k), s>>>(
        p, k, cap, ws.fine, ws.ranges, ws.nranges, ws.ncand, ids, dists, counts);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
