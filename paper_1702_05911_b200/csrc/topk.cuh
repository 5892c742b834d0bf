// topk.cuh — block-wide exact top-k over distinct u64 (orderable dist << 32 | id) keys in
// shared memory: an MSB-first 8-bit radix select finds the kk-th smallest key, the kk keys
// at or below it are collected, then a bitonic sort orders them. Keys equal to kSentinel
// (candidates another shard owns) are ignored. Reproduces partial_sort by candidate_less
// (search.cpp:39-41, :239-240) because (dist, id) keys are distinct.
#pragma once

#include "common.cuh"

namespace pqtg {
namespace dev {

struct TopkShared {
    uint32_t nsel, digit, before, bucket;
    unsigned long long kand, kor;
};

// All threads of the block call this; keys[0..C) in smem; result: sel[0..kk) ascending.
__device__ inline void block_topk(const uint64_t* keys, uint32_t C, uint32_t kk, uint64_t* sel,
                                  uint32_t sel_cap, uint32_t* hist, TopkShared& sh) {
    const int tid = threadIdx.x;
    if (kk == 0) return;
    if (tid == 0) {
        sh.nsel = 0;
        sh.kand = ~0ull;
        sh.kor = 0ull;
    }
    __syncthreads();
    // bits shared by every key need no radix pass: start below the highest differing bit
    {
        uint64_t a = ~0ull, o = 0ull;
        for (uint32_t j = tid; j < C; j += blockDim.x) {
            const uint64_t key = keys[j];
            if (key != kSentinel) {
                a &= key;
                o |= key;
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a &= __shfl_xor_sync(0xffffffffu, a, d);
            o |= __shfl_xor_sync(0xffffffffu, o, d);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAnd(&sh.kand, (unsigned long long)a);
            atomicOr(&sh.kor, (unsigned long long)o);
        }
    }
    __syncthreads();
    const uint64_t diff = sh.kand ^ sh.kor;
    const int hb = diff ? 63 - __clzll((long long)diff) : 0;  // highest differing bit
    uint64_t mask = hb >= 63 ? 0ull : (~0ull << (hb + 1));
    uint64_t prefix = sh.kand & mask;
    uint32_t need = kk;
    int shift = hb >= 7 ? hb - 7 : 0;
    for (;;) {
        for (uint32_t i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (uint32_t j = tid; j < C; j += blockDim.x) {
            const uint64_t key = keys[j];
            if (key != kSentinel && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t sum = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) sum += hist[tid * 8 + b];
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += t;
            }
            const uint32_t excl = incl - sum;
            if (excl < need && need <= incl) {
                uint32_t acc = excl;
                for (int b = 0; b < 8; ++b) {
                    const uint32_t h = hist[tid * 8 + b];
                    if (acc + h >= need) {
                        sh.digit = tid * 8 + b;
                        sh.before = acc;
                        sh.bucket = h;
                        break;
                    }
                    acc += h;
                }
            }
        }
        __syncthreads();
        prefix |= (uint64_t)sh.digit << shift;
        mask |= 0xFFull << shift;
        need -= sh.before;
        const bool done = sh.bucket == need || shift == 0;
        __syncthreads();
        if (done) break;
        // next 8-bit window; the last one may overlap bits already fixed in the prefix,
        // which only narrows its histogram
        shift = shift >= 8 ? shift - 8 : 0;
    }
    const uint64_t top = prefix >> shift;
    for (uint32_t j = tid; j < C; j += blockDim.x) {
        const uint64_t key = keys[j];
        if (key != kSentinel && (key >> shift) <= top) {
            const uint32_t at = atomicAdd(&sh.nsel, 1u);
            if (at < sel_cap) sel[at] = key;
        }
    }
    __syncthreads();
    uint32_t n2 = 1;
    while (n2 < kk) n2 <<= 1;
    for (uint32_t i = kk + tid; i < n2; i += blockDim.x) sel[i] = kSentinel;
    __syncthreads();
    for (uint32_t size = 2; size <= n2; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < n2 / 2; i += blockDim.x) {
                const uint32_t a = 2 * i - (i & (stride - 1));
                const uint32_t b = a + stride;
                const bool up = (a & size) == 0;
                const uint64_t x = sel[a], y = sel[b];
                if ((x > y) == up) {
                    sel[a] = y;
                    sel[b] = x;
                }
            }
            __syncthreads();
        }
    }
}

// Write the sorted top-kk (padded to k with (UINT32_MAX, +inf)) and the count.
__device__ inline void write_topk(const uint64_t* sel, uint32_t kk, uint32_t k, uint64_t q,
                                  uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        uint32_t id = 0xFFFFFFFFu;
        float d = __uint_as_float(0x7F800000u);
        if (i < kk) {
            id = (uint32_t)(sel[i] & 0xFFFFFFFFu);
            d = unorderable((uint32_t)(sel[i] >> 32));
        }
        out_ids[q * k + i] = id;
        out_dists[q * k + i] = d;
    }
    if (threadIdx.x == 0) out_counts[q] = kk;
}

}  // namespace dev
}  // namespace pqtg
