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
    uint32_t grouped, shift;  // block_select_wide<GROUP>: sel is grouped by digit, hist[b] = end of digit b
};

// Radix select over keys[0..C) given the AND / OR of its valid keys (bits shared by every
// key need no pass): the kk smallest keys land in sel[0..kk), unordered. All threads call it.
__device__ inline void block_select(const uint64_t* keys, uint32_t C, uint32_t kk, uint64_t kand, uint64_t kor,
                                    uint64_t* sel, uint32_t sel_cap, uint32_t* hist, TopkShared& sh) {
    const int tid = threadIdx.x;
    if (tid == 0) sh.nsel = 0;
    const uint64_t diff = kand ^ kor;
    const int hb = diff ? 63 - __clzll((long long)diff) : 0;  // highest differing bit
    uint64_t mask = hb >= 63 ? 0ull : (~0ull << (hb + 1));
    uint64_t prefix = kand & mask;
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
}

// One wide radix pass instead of several 8-bit ones: a (1 << BITS)-bin histogram of the
// BITS bits below the valid keys' common prefix (hist must be zeroed by the caller) finds the
// bin holding the kk-th smallest key; every key in that bin or below — m >= kk keys, usually
// only a few more than kk — is collected into sel[0..m). When m would exceed sel_cap, it falls
// back to the exact 8-bit select (m = kk). Returns m; all threads call it.
template <int BITS, int THREADS, bool GROUP = false>
__device__ inline uint32_t block_select_wide(const uint64_t* keys, uint32_t C, uint32_t kk, uint64_t kand,
                                             uint64_t kor, uint32_t* hist, uint64_t* sel, uint32_t sel_cap,
                                             uint32_t* wsum, TopkShared& sh) {
    constexpr uint32_t NB = 1u << BITS;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t diff = kand ^ kor;
    const int hb = diff ? 63 - __clzll((long long)diff) : 0;
    const int shift = hb >= BITS - 1 ? hb - (BITS - 1) : 0;
    // four keys' loads in flight per thread before their histogram updates
    for (uint32_t j0 = tid; j0 < C; j0 += 4 * blockDim.x) {
        uint64_t kv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t j = j0 + u * blockDim.x;
            kv[u] = j < C ? keys[j] : kSentinel;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (kv[u] != kSentinel) atomicAdd(&hist[(kv[u] >> shift) & (NB - 1)], 1u);
    }
    if (tid == 0) sh.nsel = 0;
    __syncthreads();
    // block scan of the bins, NB / blockDim consecutive bins per thread
    constexpr uint32_t per = NB / THREADS;  // blockDim.x == THREADS divides NB
    static_assert(per >= 1 && per * THREADS == NB, "THREADS must divide the bin count");
    uint32_t h[per], sum = 0;
#pragma unroll
    for (uint32_t b = 0; b < per; ++b) {
        h[b] = hist[tid * per + b];
        sum += h[b];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t i = 0; i < warp; ++i) before += wsum[i];
    incl += before;
    const uint32_t excl = incl - sum;
    if (excl < kk && kk <= incl) {
        uint32_t acc = excl;
        bool found = false;
#pragma unroll
        for (uint32_t b = 0; b < per; ++b) {
            if (!found && acc + h[b] >= kk) {
                sh.digit = tid * per + b;
                sh.before = acc;
                sh.bucket = h[b];
                found = true;
            }
            acc += h[b];
        }
    }
    __syncthreads();
    const uint32_t m = sh.before + sh.bucket;
    if (m > sel_cap) {  // a crowded bin: exact select instead
        const uint32_t kk2 = kk;
        if (GROUP && tid == 0) sh.grouped = 0;
        __syncthreads();
        block_select(keys, C, kk2, kand, kor, sel, sel_cap, hist, sh);
        return kk2;
    }
    if constexpr (GROUP) {
        // the kept keys are placed grouped by digit: each bin's counter becomes its start (the
        // exclusive scan), and a key's slot is its bin's counter, post-incremented
        uint32_t acc = excl;
#pragma unroll
        for (uint32_t b = 0; b < per; ++b) {
            hist[tid * per + b] = acc;
            acc += h[b];
        }
        if (tid == 0) {
            sh.grouped = 1;
            sh.shift = (uint32_t)shift;
        }
        __syncthreads();
    }
    const uint64_t top = ((kand & (hb >= 63 ? 0ull : (~0ull << (hb + 1)))) >> shift) | sh.digit;
    for (uint32_t j0 = tid; j0 < C; j0 += 4 * blockDim.x) {
        uint64_t kv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t j = j0 + u * blockDim.x;
            kv[u] = j < C ? keys[j] : kSentinel;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (kv[u] != kSentinel && (kv[u] >> shift) <= top) {
                if constexpr (GROUP) sel[atomicAdd(&hist[(kv[u] >> shift) & (NB - 1)], 1u)] = kv[u];
                else sel[atomicAdd(&sh.nsel, 1u)] = kv[u];
            }
    }
    __syncthreads();
    return m;
}

// block_sort_write for a selection grouped by digit (block_select_wide<GROUP>, sh.grouped): after
// the placement hist[b] is the end of bin b's keys in sel and hist[b - 1] its start, and every key
// of a lower bin is smaller, so a key's rank is its bin's start plus the count of smaller keys in
// its own bin -- a few compares instead of a count over all m keys.
// block_rank_keys for a selection grouped by digit: the kk smallest keys to out[0..kk) in order
template <int BITS>
__device__ inline void block_rank_keys_grouped(const uint64_t* sel, uint32_t m, uint32_t kk, const uint32_t* hist,
                                               uint32_t shift, uint64_t* out) {
    constexpr uint32_t NB = 1u << BITS;
    for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
        const uint64_t me = sel[p];
        const uint32_t b = (uint32_t)(me >> shift) & (NB - 1);
        const uint32_t s = b ? hist[b - 1] : 0u, e = hist[b];
        uint32_t rank = s;
        for (uint32_t j = s; j < e; ++j) rank += sel[j] < me;
        if (rank < kk) out[rank] = me;
    }
}

template <int BITS>
__device__ inline void block_sort_write_grouped(const uint64_t* sel, uint32_t m, uint32_t kk, uint32_t k, uint64_t q,
                                                const uint32_t* hist, uint32_t shift, uint32_t* out_ids,
                                                float* out_dists, uint32_t* out_counts) {
    constexpr uint32_t NB = 1u << BITS;
    for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
        const uint64_t me = sel[p];
        const uint32_t b = (uint32_t)(me >> shift) & (NB - 1);
        const uint32_t s = b ? hist[b - 1] : 0u, e = hist[b];
        uint32_t rank = s;
        for (uint32_t j = s; j < e; ++j) rank += sel[j] < me;
        if (rank < kk) {
            out_ids[q * k + rank] = (uint32_t)(me & 0xFFFFFFFFu);
            out_dists[q * k + rank] = unorderable((uint32_t)(me >> 32));
        }
    }
    for (uint32_t i = kk + threadIdx.x; i < k; i += blockDim.x) {
        out_ids[q * k + i] = 0xFFFFFFFFu;
        out_dists[q * k + i] = __uint_as_float(0x7F800000u);
    }
    if (threadIdx.x == 0) out_counts[q] = kk;
}

// Bitonic sort of sel[0..kk) (padded with kSentinel to a power of two <= sel_cap).
__device__ inline void block_bitonic(uint64_t* sel, uint32_t kk) {
    const int tid = threadIdx.x;
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

// All threads of the block call this; keys[0..C) in smem; result: sel[0..kk) ascending.
__device__ inline void block_topk(const uint64_t* keys, uint32_t C, uint32_t kk, uint64_t* sel,
                                  uint32_t sel_cap, uint32_t* hist, TopkShared& sh) {
    const int tid = threadIdx.x;
    if (kk == 0) return;
    if (tid == 0) {
        sh.kand = ~0ull;
        sh.kor = 0ull;
    }
    __syncthreads();
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
    block_select(keys, C, kk, sh.kand, sh.kor, sel, sel_cap, hist, sh);
    block_bitonic(sel, kk);
}

// Order the m >= kk distinct keys sel[0..m), write the kk smallest (padded to k with
// (UINT32_MAX, +inf)) and the count. Up to blockDim.x keys: every key's rank is counted
// directly — g threads per key, each over a strided share of the others, summed with
// shuffles — and a key of rank < kk is stored at its rank (one barrier-free pass instead of
// a bitonic network); more keys fall back to the bitonic sort.
__device__ inline void block_sort_write(uint64_t* sel, uint32_t m, uint32_t kk, uint32_t k, uint64_t q,
                                        uint32_t* out_ids, float* out_dists, uint32_t* out_counts) {
    const uint32_t tid = threadIdx.x;
    uint32_t n2 = 1;
    while (n2 < m) n2 <<= 1;
    if (n2 <= blockDim.x) {
        uint32_t g = blockDim.x / n2;
        g = g > 32 ? 32 : g;
        const uint32_t e = tid / g, sub = tid - e * g;
        const bool own = e < m;
        const uint64_t me = own ? sel[e] : 0ull;
        uint32_t rank = 0;
        if (own) {
            uint32_t j = sub;
            for (; j + 3 * g < m; j += 4 * g) {  // four loads in flight
                const uint64_t a = sel[j], b = sel[j + g], c = sel[j + 2 * g], d = sel[j + 3 * g];
                rank += (uint32_t)(a < me) + (uint32_t)(b < me) + (uint32_t)(c < me) + (uint32_t)(d < me);
            }
            for (; j < m; j += g) rank += sel[j] < me;
        }
        for (uint32_t o = 1; o < g; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (own && sub == 0 && rank < kk) {
            out_ids[q * k + rank] = (uint32_t)(me & 0xFFFFFFFFu);
            out_dists[q * k + rank] = unorderable((uint32_t)(me >> 32));
        }
    } else {
        block_bitonic(sel, m);
        for (uint32_t i = tid; i < kk; i += blockDim.x) {
            out_ids[q * k + i] = (uint32_t)(sel[i] & 0xFFFFFFFFu);
            out_dists[q * k + i] = unorderable((uint32_t)(sel[i] >> 32));
        }
    }
    for (uint32_t i = kk + tid; i < k; i += blockDim.x) {
        out_ids[q * k + i] = 0xFFFFFFFFu;
        out_dists[q * k + i] = __uint_as_float(0x7F800000u);
    }
    if (tid == 0) out_counts[q] = kk;
}

// The kk smallest of the m >= kk distinct keys sel[0..m) to out[0..kk) in ascending order (the
// rank count of block_sort_write, storing keys).
__device__ inline void block_rank_keys(uint64_t* sel, uint32_t m, uint32_t kk, uint64_t* out) {
    const uint32_t tid = threadIdx.x;
    uint32_t n2 = 1;
    while (n2 < m) n2 <<= 1;
    if (n2 <= blockDim.x) {
        uint32_t g = blockDim.x / n2;
        g = g > 32 ? 32 : g;
        const uint32_t e = tid / g, sub = tid - e * g;
        const bool own = e < m;
        const uint64_t me = own ? sel[e] : 0ull;
        uint32_t rank = 0;
        if (own) {
            uint32_t j = sub;
            for (; j + 3 * g < m; j += 4 * g) {  // four loads in flight
                const uint64_t a = sel[j], b = sel[j + g], c = sel[j + 2 * g], d = sel[j + 3 * g];
                rank += (uint32_t)(a < me) + (uint32_t)(b < me) + (uint32_t)(c < me) + (uint32_t)(d < me);
            }
            for (; j < m; j += g) rank += sel[j] < me;
        }
        for (uint32_t o = 1; o < g; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (own && sub == 0 && rank < kk) out[rank] = me;
    } else {
        block_bitonic(sel, m);
        for (uint32_t i = tid; i < kk; i += blockDim.x) out[i] = sel[i];
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
