// rerank_fast.cu — K5 fast path: line-quantized re-rank (linequant.cpp:169-182) + top-k
// (search.cpp:221-257) for p_line == 32 and 1-byte pair ids.
//
// Work layout: one CTA (16 warps) per query; the query's candidates are cut into 16
// contiguous warp slices; lane l re-ranks candidates aw + 32r + l (round r). Each lane sums
// its candidate's 32 fine parts in the reference's order, but lane l runs ONE PART BEHIND
// lane l-1 (a skewed pipeline): at every step the 32 lanes touch 32 different fine parts,
// so lookups into the per-query table, laid out [pair][part], hit 32 different banks.
//
//   per-query table   row pid = 32 × float4 (b2, E, c2, 0), E = (a2 - b2) - c2,
//                     b2 = fine[f][i], a2 = fine[f][j], (i, j) = pairs[pid]: exactly the fp32
//                     intermediates of the reference, so part = (b2 + (λ·λ)·c2) + λ·E rounds
//                     identically. One 16-byte load per part.
//   code staging      each lane prefetches its next row (64 B) with cp.async into a private
//                     3-round ring in shared memory, one phase (32 steps) ahead of use.
//   top-k             (dist, id) keys of all candidates in shared memory, block radix select.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kFastWarps = 16;
constexpr int kFastThreads = kFastWarps * 32;
constexpr int kSlotBytes = 64;                   // one row: 32 × (λ, pair) bytes
constexpr int kLaneBytes = 3 * kSlotBytes + 16;  // 3-round ring + pad
constexpr uint32_t kRangeCache = 1024;           // ranges cached in shared memory
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
    size_t lut, ring, ids, fine, pairs, ranges, keys, sel, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline FastLayout fast_layout(uint32_t npairs, uint32_t k1, uint32_t budget, uint32_t sel_cap) {
    FastLayout l{};
    size_t o = 0;
    l.lut = o;  // offset 0: lookups use immediate offsets
    o += (size_t)npairs * 512;
    l.ring = o;
    o += (size_t)kFastThreads * kLaneBytes;
    l.ids = o;
    o += align16((size_t)kFastThreads * 3 * 4);
    l.fine = o;
    o += align16((size_t)32 * k1 * 4);
    l.pairs = o;
    o += align16((size_t)npairs * 4);
    l.ranges = o;
    o += align16((size_t)(budget < kRangeCache ? budget : kRangeCache) * 8);
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
    unsigned char* lut = smem;  // [pid][32] float4
    uint8_t* ring = smem + lay.ring;
    uint32_t* ring_ids = reinterpret_cast<uint32_t*>(smem + lay.ids);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    uint32_t* spairs = reinterpret_cast<uint32_t*>(smem + lay.pairs);
    uint2* rg_s = reinterpret_cast<uint2*>(smem + lay.ranges);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + lay.keys);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + lay.sel);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2* qr = ranges + q * (uint64_t)budget;
    const bool cached = R <= kRangeCache;
    const uint2* rg = cached ? rg_s : qr;

    for (uint32_t i = tid; i < 32 * k1; i += blockDim.x) fine[i] = fine_in[q * 32 * k1 + i];
    if (cached)
        for (uint32_t r = tid; r < R; r += blockDim.x) rg_s[r] = qr[r];
    for (uint32_t i = tid; i < npairs; i += blockDim.x) spairs[i] = __ldg(p.pairs + i);
    {
        uint4* z = reinterpret_cast<uint4*>(ring + (size_t)tid * kLaneBytes);
        for (int i = 0; i < kLaneBytes / 16; ++i) z[i] = make_uint4(0, 0, 0, 0);  // pid 0 in unused slots
    }
    if (tid == 0) s_count = 0;
    __syncthreads();
#pragma unroll 4
    for (uint32_t idx = tid; idx < npairs * 32; idx += blockDim.x) {
        const uint32_t pid = idx >> 5, f = idx & 31;
        const uint32_t pr = spairs[pid];
        const float b2 = fine[f * k1 + (pr & 0xFFFFu)];
        const float a2 = fine[f * k1 + (pr >> 16)];
        const float c2 = __ldg(p.c2 + (size_t)f * npairs + pid);
        reinterpret_cast<float4*>(lut + (size_t)pid * 512)[f] =
            make_float4(b2, __fsub_rn(__fsub_rn(a2, b2), c2), c2, 0.0f);
    }
    __syncthreads();

    // ---- skewed per-warp pipeline
    const uint32_t aw = (uint32_t)((uint64_t)C * warp / kFastWarps);
    const uint32_t bw = (uint32_t)((uint64_t)C * (warp + 1) / kFastWarps);
    const uint32_t nround = (bw - aw + 31) >> 5;
    uint8_t* my = ring + (size_t)tid * kLaneBytes;
    uint32_t* myid = ring_ids + tid * 3;
    const bool sharded = p.shard_hi > p.shard_lo;
    uint32_t cursor = 0;
    bool first = true;

    auto stage = [&](uint32_t r) {
        const uint32_t c = aw + 32 * r + lane;
        const uint32_t slot = r % 3;
        bool issued = false;
        if (r < nround && c < bw) {
            // range holding candidate c: last rr with rg[rr].y <= c (candidate offsets ascend);
            // successive rounds move c by 32, so at most 32 ranges past the cursor
            uint32_t lo = first ? 0 : cursor;
            uint32_t hi = first ? R - 1 : min(R - 1, cursor + 32);
            first = false;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (rg[mid].y <= c) lo = mid; else hi = mid - 1;
            }
            cursor = lo;
            const uint2 e = rg[lo];
            const uint64_t pos = (uint64_t)e.x + (c - e.y);
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

    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    uint32_t mine = 0;
    float acc = 0.0f, done = 0.0f;
    stage(0);
    stage(1);
    for (uint32_t m = 0; nround > 0 && m <= nround; ++m) {
        if (m > 0) stage(m + 1);
        cp_async_wait<1>();  // round m has landed (each lane reads only its own ring)
        // byte offsets of lane l's current (round m) and previous (round m-1) rows, minus 2t
        const int32_t off_cur = (int32_t)((m % 3) * kSlotBytes) - 2 * lane;
        const int32_t off_prev = (int32_t)(((m + 2) % 3) * kSlotBytes + kSlotBytes) - 2 * lane;
        const int32_t nl16 = -16 * lane;
        // One fine part per lane per step, branch-free: the finished sum of a candidate
        // (part 31, reached by lane (t + 1) & 31 at step t) is parked in `done`. Fill and
        // drain phases run the same code: before its first and after its last candidate a
        // lane accumulates stale ring rows into "rounds" -1 / nround, whose keys are never
        // written, and the part-31 reset clears acc before every real candidate.
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int32_t off = (t >= lane ? off_cur : off_prev) + 2 * t;
            const uint32_t code = *reinterpret_cast<const uint16_t*>(my + off);
            const uint32_t f16 = (uint32_t)(nl16 + 16 * t) & 496u;
            const uint32_t li = ((code << 1) & 0x1FE00u) | f16;  // pid * 512 + f * 16
            const float4 e = *reinterpret_cast<const float4*>(lut + li);
            const float lam = __fmul_rn(__uint2float_rn(code & 0xFFu), inv255);
            const float part = __fadd_rn(__fadd_rn(e.x, __fmul_rn(__fmul_rn(lam, lam), e.z)), __fmul_rn(lam, e.y));
            acc = __fadd_rn(acc, part);
            const bool fin = lane == ((t + 1) & 31);
            done = fin ? acc : done;
            acc = fin ? 0.0f : acc;
        }
        // each lane finished one candidate this phase: lane 0 its round m, lanes l > 0 their
        // round m - 1 (at step l - 1)
        const int32_t r = lane == 0 ? (int32_t)m : (int32_t)m - 1;
        if (r >= 0 && r < (int32_t)nround) {
            const uint32_t c = aw + 32 * (uint32_t)r + lane;
            if (c < bw) {
                const uint32_t id = myid[r % 3];
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
