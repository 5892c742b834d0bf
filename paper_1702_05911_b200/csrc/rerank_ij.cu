// rerank_ij.cu — K5 fast path: line-quantized re-rank (linequant.cpp:169-182) + top-k
// (search.cpp:221-257) for indexes with k1 <= 16 and 1-byte pairs, whose device codes store
// each part's centroid pair as t = i << 4 | ((i + j) & 15) instead of the pair id (index_prep.cpp).
//
// One thread per candidate; the code row (L × (λ, ij) bytes, slot order) is read with 16-byte
// loads into registers and its parts are summed in the reference's order. Per part:
//     b2 = fine[f][i]                   a 16-float row per part: the 32 lanes of a warp touch
//                                       at most 16 addresses, all in distinct banks
//                                       (duplicates broadcast) — conflict-free;
//     (E, c2) = T[f][t]                 per-query table, E = (a2 − b2) − c2 with a2 = fine[f][j]
//                                       and c2 = d2[f][i][j]: the reference's own intermediate
//                                       (linequant.hpp:85), built once per query;
//     part = (b2 + (λ·λ)·c2) + λ·E      exactly linequant.hpp:83-85's rounding.
// Shared memory: T (L × 2 KB), fine (L × 64 B), candidate keys, range offsets (cached up to
// kRangeCache, else read from global memory); ij_threads(L) threads per CTA.
//
// DIRECT (k1 <= 32 two-byte codes only): no T. Building T costs L × 496 entries per query, as
// much as scoring ~500 candidates — the share of a 4096-candidate budget that one of eight
// position shards re-ranks. DIRECT computes E per part from fine[f][i], fine[f][j] (j from a
// per-pair table) and c2 = d2[f][pair] (read through L1), the same three roundings, and leaves
// the shared memory small enough for two CTAs per SM.
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;
namespace cg = cooperative_groups;

// phase clocks of CTA (0, 0) of the last re-rank launch (PQTG_PHASES=1: tools/phase_probe.py);
// null otherwise. [0] start, [1] prologue done, [2] range map done, [3] candidates scored,
// [4] selected, [5] written (split: the slice's list), [6] merged and [7] arrived (split's last slice)
__device__ unsigned long long* g_phase = nullptr;
#define PQTG_PHASE(i)                                                                                  \
    do {                                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0 && (blockIdx.y == 0 || (i) >= 6) && g_phase) g_phase[i] = gtimer_ns(); \
    } while (0)

#define PQTG_PHASE_VAL(i, v)                                                                           \
    do {                                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0 && g_phase) g_phase[i] = (v);                          \
    } while (0)

namespace {

// threads per CTA: 512, two CTAs (queries) per SM. (1024-thread CTAs, one query per SM, cut the
// last wave's idle time but measured 20% slower on B200: MIO-queue stalls.)
// DIRECT (a shard's ~1 candidate per thread): 256-thread CTAs, four per SM, so an SM overlaps four
// queries' serial prologue / selection chains instead of two
__host__ __device__ constexpr int ij_threads(int L, bool direct = false) { return direct ? 256 : (L >= 64 ? 512 : 512); }
constexpr int kScanItems = 8;  // rid entries per thread per scan tile
constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // no id: the candidate belongs to another shard
constexpr uint32_t kRangeCache = 512;       // ranges whose (start − offset) is kept in smem

struct IjLayout {
    size_t t, fine, keys, sel, rid, delta, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// a 4-byte shared-memory load at a 32-bit shared-window address (the PK loop builds addresses
// with LOP3 from an aligned base; ptxas folds the constant part into the LDS immediate)
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

constexpr int kSelBits = 10;                 // wide radix-select digit (block_select_wide)
constexpr uint32_t kSelMin = 512;           // sel capacity for the wide select's bin

// sel capacity: a power of two >= max(kk, kSelMin)
__host__ __device__ inline uint32_t ij_sel_cap(uint32_t kk) {
    uint32_t c = kSelMin;
    while (c < kk) c <<= 1;
    return c;
}

// K1M = 16: 1-byte codes t = i << 4 | ((i + j) & 15), T[f] has 256 entries, fine rows 16 floats.
// K1M = 32: 2-byte codes v = pid | i << 9 (k1 <= 32, 496 pairs), T[f] has 512 entries by pair id,
// fine rows 32 floats.
__host__ __device__ constexpr uint32_t t_entries(int K1M) { return K1M == 16 ? 256u : 512u; }

__host__ __device__ inline IjLayout ij_layout(uint32_t L, uint32_t budget, uint32_t sel_cap, int K1M = 16,
                                              bool direct = false, bool gkeys = false, bool pk = false) {
    IjLayout l{};
    size_t o = 0;
    l.t = o;  // T (DIRECT: the pairs' j, u16; PK: c2 by code), fine, delta and rid sit at compile-time offsets
    // PK: a 1 KB-aligned (at run time) c2 table L × 1 KB followed by the fine rows
    o += direct ? (size_t)0
                : (pk ? (size_t)L * 1024 + (size_t)L * K1M * 4 + 1024 : (size_t)L * t_entries(K1M) * 8);
    l.fine = o;
    o += (size_t)L * K1M * 4;
    l.delta = o;
    o += (size_t)kRangeCache * 4;
    // rid: u16 range index per candidate, padded to whole 4096-candidate scan tiles; after
    // the candidate loop the same bytes hold the select histogram and sel
    l.rid = o;
    const size_t tile = (size_t)kScanItems * ij_threads((int)L, direct);
    const size_t rid_bytes = al16((budget + tile - 1) / tile * tile * 2);
    const size_t sel_bytes = ((size_t)4 << kSelBits) + (size_t)sel_cap * 8;
    l.sel = o + ((size_t)4 << kSelBits);
    o += rid_bytes > sel_bytes ? rid_bytes : sel_bytes;
    l.keys = o;
    if (!gkeys) o += al16((size_t)budget * 8);  // gkeys: the candidate keys live in the workspace (HBM/L2)
    l.total = o;
    return l;
}

// rid[j] = index of the range holding candidate j, for j < C: rid is zero except
// rid[offset of range r] = r, so an inclusive max-scan gives it (range offsets increase
// with r). TH threads × 8 consecutive u16 per scan tile.
template <int TH>
__device__ inline void range_index_scan(uint16_t* rid, uint32_t C, uint32_t* wmax) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < C; base += kScanItems * TH) {
        uint4* v4 = reinterpret_cast<uint4*>(rid + base) + tid;
        uint4 v = *v4;
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t run = 0, e[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            run = max(run, w[i] & 0xFFFFu);
            e[2 * i] = run;
            run = max(run, w[i] >> 16);
            e[2 * i + 1] = run;
        }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl = max(incl, t);
        }
        if (lane == 31) wmax[warp] = incl;
        __syncthreads();
        uint32_t before = carry;
        for (uint32_t i = 0; i < warp; ++i) before = max(before, wmax[i]);
        const uint32_t up = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane > 0) before = max(before, up);
        uint32_t r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = max(before, e[i]);
        *v4 = make_uint4(r[0] | (r[1] << 16), r[2] | (r[3] << 16), r[4] | (r[5] << 16), r[6] | (r[7] << 16));
        for (uint32_t i = 0; i < TH / 32; ++i) carry = max(carry, wmax[i]);
        __syncthreads();
    }
}

}  // namespace

// MODE (K1M = 16): 0 = per-query table T[f][t] = (E, c2) (default); 1 = packed two-candidate loop
// (PK); 2 = the scalar loop reading c2 by code and a2 = fine[f][j], E formed per candidate (C3);
// 3 = E[f][t] and c2[f][t] as two 4-byte tables in T's bytes (S2: a 4-byte gather spreads a warp's
// distinct pairs over 32 banks instead of the 16 bank pairs of an 8-byte one). Modes 1 and 2 use
// the c2-table layout (CT).
template <int LT, int K1M, bool DIRECT, int MODE = 0>
__global__ void __launch_bounds__(ij_threads(LT, DIRECT), DIRECT ? 4 : ((LT >= 64 || K1M == 32 || MODE == 7) ? 1 : 2))
    rerank_ij_kernel(DevParams p, uint32_t k, uint32_t sel_cap, const float* __restrict__ fine_in,
                     const uint2* __restrict__ ranges, const uint32_t* __restrict__ nranges,
                     const uint32_t* __restrict__ ncand, uint32_t* __restrict__ out_ids,
                     float* __restrict__ out_dists, uint32_t* __restrict__ out_counts, uint64_t* __restrict__ gkeys,
                     uint64_t* __restrict__ split_keys,
                     uint32_t* __restrict__ split_ctr) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool PK = MODE == 1, C3 = MODE == 2, CT = MODE == 1 || MODE == 2, S2 = MODE == 3, COOP = MODE == 4,
                   HALF = MODE == 8 && K1M == 16 && LT == 32 && !DIRECT;
    // GRP (the default): the final top-k ranks each kept key within its radix bin only -- the kept
    // keys are placed grouped by bin, and every key of a lower bin is smaller (DEEP100M re-rank
    // 1227 -> 1183 us against ranking each key over all kept keys, which PQTG_RERANK=ungrouped keeps)
    constexpr bool GRP = MODE != 10;
    const uint32_t k1 = p.k1, budget = p.budget;
    constexpr uint32_t TE = t_entries(K1M);
    const IjLayout lay = ij_layout(LT, budget, sel_cap, K1M, DIRECT, gkeys != nullptr, CT);
    const IjLayout fix = ij_layout(LT, 0, 0, K1M, DIRECT, false, CT);
    float2* T = reinterpret_cast<float2*>(smem);
    // PK (packed, K1M = 16): c2 by device code, Ct[f][t] = d2[f][i][j], at a 1 KB-aligned shared
    // address, then the fine rows: the scoring loop forms each lookup's address with one LOP3
    // (offset | aligned base) instead of an add
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t c2s = (s_base + 1023u) & ~1023u, fs = c2s + LT * 1024u;
    float* Ct = reinterpret_cast<float*>(smem + (c2s - s_base));
    float* fine = CT ? reinterpret_cast<float*>(smem + (fs - s_base)) : reinterpret_cast<float*>(smem + fix.fine);
    // candidate keys: shared memory, or this query's row of the workspace's key buffer when the
    // budget is too large for shared memory (budget > ~8k)
    uint64_t* keys = gkeys ? gkeys + blockIdx.x * (uint64_t)budget : reinterpret_cast<uint64_t*>(smem + lay.keys);
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem + lay.sel);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + fix.rid);  // aliases rid
    uint16_t* rid = reinterpret_cast<uint16_t*>(smem + fix.rid);
    uint32_t* delta = reinterpret_cast<uint32_t*>(smem + fix.delta);
    constexpr int kIjThreads = ij_threads(LT, DIRECT);
    __shared__ uint32_t wmax[kIjThreads / 32];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    PQTG_PHASE(0);
    const uint2* qr = ranges + q * (uint64_t)budget;

    // every global load of the prologue is issued before the first barrier: the query's fine
    // LUT, the first kIjThreads ranges and this thread's column of d2 (T build below)
    constexpr uint32_t kPairLanes = K1M == 16 ? 128 : 512;  // >= the pair count
    constexpr uint32_t kFLanes = kIjThreads >= (int)kPairLanes ? kIjThreads / kPairLanes : 1;
    constexpr uint32_t kFPer = (LT + kFLanes - 1) / kFLanes;
    const uint32_t pi = tid & (kPairLanes - 1), f0 = tid / kPairLanes;
    const bool pair_lane = pi < p.npairs;
    uint32_t pi_i = 0, pi_j = 0;
    float c2v[kFPer];
    uint32_t slot[kFPer];  // K1M = 16: the pair's T slot per part (the per-part bank map, or fixed)
    if (pair_lane) {
        const uint32_t pr = __ldg(p.pairs + pi);
        pi_i = pr & 0xFFFFu;
        pi_j = pr >> 16;
        if constexpr (DIRECT) {
            // (the codes carry j: nothing to stage)
        } else
#pragma unroll
        for (uint32_t u = 0; u < kFPer; ++u) {
            const uint32_t f = f0 + u * kFLanes;
            if constexpr (K1M == 16) {
                if (!CT && p.c2slot) {
                    const uint2 cs = f < LT ? __ldg(p.c2slot + f * p.npairs + pi) : make_uint2(0, 0);
                    c2v[u] = __uint_as_float(cs.x);
                    slot[u] = cs.y;
                } else {
                    slot[u] = pi_i << 4 | ((pi_i + pi_j) & 15u);
                    c2v[u] = f < LT ? __ldg(p.c2ij + f * 256 + slot[u]) : 0.0f;
                }
            } else
                c2v[u] = f < LT ? __ldg(p.c2 + f * p.npairs + pi) : 0.0f;
        }
    }
    // the query's fine LUT (the traversal's) into shared memory, and T[f][t(i, j)] = (E, c2) for
    // every pair i < j (linequant.cpp:76-82; other entries are never referenced; thread: one pair,
    // every (blockDim / 128)-th part)
    auto copy_fine = [&](bool l2_only) {
        for (uint32_t i = tid; i < LT * K1M; i += blockDim.x) {
            const uint32_t f = i / K1M, c = i % K1M;
            const float* src = fine_in + q * LT * k1 + f * k1 + c;
            fine[i] = c < k1 ? (l2_only ? __ldcg(src) : *src) : 0.0f;
        }
    };
    auto build_T = [&] {
        if (!DIRECT && pair_lane) {
#pragma unroll
            for (uint32_t u = 0; u < kFPer; ++u) {
                const uint32_t f = f0 + u * kFLanes;
                // the pair's T slot: its device code in part f (K1M = 16) or its pair id (K1M = 32)
                const uint32_t ij = K1M == 16 ? slot[u] : pi;
                if (f < LT) {
                    const float b2 = fine[f * K1M + pi_i], a2 = fine[f * K1M + pi_j];
                    if constexpr (CT) {
                        Ct[f * TE + ij] = c2v[u];
                    } else if constexpr (S2) {
                        float* Et = reinterpret_cast<float*>(smem);
                        Et[f * TE + ij] = __fsub_rn(__fsub_rn(a2, b2), c2v[u]);
                        Et[LT * TE + f * TE + ij] = c2v[u];
                    } else {
                        T[f * TE + ij] = make_float2(__fsub_rn(__fsub_rn(a2, b2), c2v[u]), c2v[u]);
                    }
                }
            }
        }
    };
    // Everything above reads the index only; the bin selection's ranges are read below, after the
    // wait of a PDL dependent (a chained chunk). The traversal's fine LUT is complete already: the
    // bin selection's CTAs passed their own wait on it before this grid could launch, so a chained
    // re-rank stages the LUT and builds T while the bin selection still runs (from L2: no L1 line
    // of an earlier search's LUT).
    if (p.chain) {
        copy_fine(true);
        __syncthreads();
        build_T();
        griddep_wait();
        griddep_launch();
    }
    qt_begin(p, q, 2);
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2 rg0 = tid < R ? (p.chain ? __ldcg(qr + tid) : __ldg(qr + tid)) : make_uint2(0, 0);
    // every index is a position range [shard_lo, shard_hi): [0, n) unsharded, possibly empty
    // on a shard (then every candidate is skipped and the query returns count 0)
    constexpr bool sharded = true;
    const bool cached = R <= (kRangeCache < (uint32_t)kIjThreads ? kRangeCache : (uint32_t)kIjThreads);
    // a position shard with cached ranges re-ranks only its own candidates: the ranges are
    // clipped to [shard_lo, shard_hi) and renumbered densely (thread r = range r), so the loop,
    // the scan and the select run over this shard's candidates only
    const bool clip = sharded && cached;
    const uint32_t y1 = clip && tid < R ? (tid + 1 < R ? __ldg(&qr[tid + 1].y) : C) : 0u;
    if (!p.chain) copy_fine(false);
    const uint32_t Cpad = (C + kScanItems * kIjThreads - 1) / (kScanItems * kIjThreads) * (kScanItems * kIjThreads);
    for (uint32_t i = tid; i < Cpad / 2; i += blockDim.x) reinterpret_cast<uint32_t*>(rid)[i] = 0;
    if (tid == 0) {
        s_count = 0;
        s_sel.kand = ~0ull;
        s_sel.kor = 0ull;
    }
    __syncthreads();
    uint32_t Cn = C;  // candidates scored by this CTA
    if (clip) {
        __shared__ uint32_t wsum[kIjThreads / 32];
        uint64_t a = 0;
        uint32_t len = 0;
        if (tid < R) {
            const uint64_t x = rg0.x, e = x + (y1 - rg0.y);
            a = x > p.shard_lo ? x : p.shard_lo;
            const uint64_t b = e < p.shard_hi ? e : p.shard_hi;
            len = b > a ? (uint32_t)(b - a) : 0u;
        }
        const uint32_t lane = tid & 31, warp = tid >> 5;
        uint32_t incl = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= (uint32_t)d) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t off = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kIjThreads / 32; ++w) {
            const uint32_t v = wsum[w];
            off += (uint32_t)w < warp ? v : 0u;
            tot += v;
        }
        if (len) {
            const uint32_t y = off + incl - len;
            rid[y] = (uint16_t)tid;
            delta[tid] = (uint32_t)a - y;
        }
        Cn = tot;
    } else {
        for (uint32_t r = tid; r < R; r += blockDim.x) {
            const uint2 rg = r == tid ? rg0 : __ldg(qr + r);
            rid[rg.y] = (uint16_t)r;
            if (cached) delta[r] = rg.x - rg.y;
        }
    }
    if (!p.chain) build_T();
    __syncthreads();
    PQTG_PHASE(1);
    range_index_scan<kIjThreads>(rid, Cn, wmax);
    PQTG_PHASE(2);

    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    constexpr int kVec = ((K1M == 16 ? 2 : 3) * LT + 15) / 16;
    // 256-bit row loads (MODE 5, PQTG_RERANK=narrow, keeps the 16-byte loads and the I2F of
    // round 2's measurements for comparison)
    constexpr bool kWide = MODE != 5;
    // λq by I2F; MODE 6 (PQTG_RERANK=prmt) builds 2^23 + q with a byte permute and removes 2^23
    // with an FADD instead (measured slower: DEEP100M 1223 -> 1231 us, SIFT1M 1074 -> 1105 us)
    constexpr bool I2F = MODE != 6;
    uint32_t mine = 0;
    uint32_t kand = ~0u, kor = 0u;  // AND / OR of this thread's orderable distances
    // candidate j's code row and id, fetched one iteration ahead (software pipelining)
    auto fetch = [&](uint32_t j, uint4* v, uint32_t& id) {
        const uint32_t r = rid[j];
        uint64_t pos;
        if (cached) {
            pos = (uint32_t)(delta[r] + j);
        } else {
            const uint2 rl = __ldg(qr + r);
            pos = (uint64_t)rl.x + (j - rl.y);
        }
        id = kInvalid;
        if (!sharded || clip || (pos >= p.shard_lo && pos < p.shard_hi)) {
            const uint64_t lp = pos - p.shard_lo;
            id = __ldg(p.ids + lp);
            const uint4* r4 = reinterpret_cast<const uint4*>(p.codes + lp * p.row_bytes);
            if constexpr (kVec % 2 == 0 && kWide) {
                // rows of a multiple of 32 bytes: 32-byte loads, half the load instructions (and
                // L1 wavefronts) of 16-byte ones
#pragma unroll
                for (int i = 0; i < kVec; i += 2) ldg256(r4 + i, v[i], v[i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < kVec; ++i) v[i] = __ldg(r4 + i);
            }
        }
    };
    // COOP: a warp's 32 code rows are read kVec lanes per row (each row's kVec 16-byte pieces in
    // one load instruction, 32 / kVec rows per instruction: 32 / kVec lines per load instead of
    // 32), then transposed by shuffles so every lane holds its own candidate's row. Lane
    // l = kVec·g + u loads, in round r, piece (u − r) mod kVec of the warp's candidate
    // (32 / kVec)·r + g; in shuffle round s every lane m receives piece s of its candidate from
    // lane kVec·(m mod 32/kVec) + (s + m / (32/kVec)) mod kVec, which sends its round (u − s) mod
    // kVec value (the sources of one shuffle round are distinct). issue() starts the loads,
    // finish() runs the shuffles one candidate later, so the loads stay in flight over a score.
    constexpr uint32_t kRowsPer = 32 / kVec;  // rows per load round
    auto issue = [&](uint32_t j, uint32_t jlim, uint4* x, uint32_t& id) {
        uint32_t lp = kInvalid;
        id = kInvalid;
        if (j < jlim) {
            const uint32_t r = rid[j];
            uint64_t pos;
            if (cached) {
                pos = (uint32_t)(delta[r] + j);
            } else {
                const uint2 rl = __ldg(qr + r);
                pos = (uint64_t)rl.x + (j - rl.y);
            }
            if (clip || (pos >= p.shard_lo && pos < p.shard_hi)) {
                lp = (uint32_t)(pos - p.shard_lo);
                id = __ldg(p.ids + lp);
            }
        }
        const uint32_t lane = tid & 31, g = lane / kVec, u = lane % kVec;
#pragma unroll
        for (uint32_t r = 0; r < kVec; ++r) {
            const uint32_t slp = __shfl_sync(0xffffffffu, lp, kRowsPer * r + g);
            x[r] = slp != kInvalid ? __ldg(reinterpret_cast<const uint4*>(p.codes + (uint64_t)slp * p.row_bytes) +
                                           ((u + kVec - r) % kVec))
                                   : make_uint4(0, 0, 0, 0);
        }
    };
    auto finish = [&](const uint4* x, uint4* v) {
        const uint32_t lane = tid & 31, u = lane % kVec;
        const uint32_t src0 = kVec * (lane % kRowsPer), rr = lane / kRowsPer;
#pragma unroll
        for (uint32_t s = 0; s < kVec; ++s) {
            const uint32_t want = (u + kVec - s) % kVec;
            uint4 snd = x[0];
#pragma unroll
            for (uint32_t r = 1; r < kVec; ++r)
                if (want == r) snd = x[r];
            const uint32_t src = src0 + (s + rr) % kVec;
            v[s].x = __shfl_sync(0xffffffffu, snd.x, src);
            v[s].y = __shfl_sync(0xffffffffu, snd.y, src);
            v[s].z = __shfl_sync(0xffffffffu, snd.z, src);
            v[s].w = __shfl_sync(0xffffffffu, snd.w, src);
        }
    };
    // one candidate's line distance -> its (dist, id) key
    auto score = [&](uint32_t j, const uint4* v, uint32_t id) {
        uint64_t key = kSentinel;
        if (id != kInvalid) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(v);
            float total = 0.0f;
#pragma unroll
            for (int f = 0; f < LT; ++f) {
                uint32_t lq, ti, fi;  // λq, T slot, fine index
                if constexpr (K1M == 16) {
                    const uint32_t half = w[f >> 1] >> ((f & 1) * 16);  // λ | t << 8, t = i << 4 | ((i + j) & 15)
                    ti = (half >> 8) & 0xFFu;
                    fi = ti >> 4;
                    lq = half & 0xFFu;
                } else if constexpr (DIRECT) {
                    lq = (w[f >> 2] >> ((f & 3) * 8)) & 0xFFu;                 // λ block
                    ti = (w[LT / 4 + (f >> 1)] >> ((f & 1) * 16)) & 0x3FFu;   // i | j << 5
                    fi = ti & 31u;
                } else {
                    lq = (w[f >> 2] >> ((f & 3) * 8)) & 0xFFu;                 // λ block
                    const uint32_t v2 = (w[LT / 4 + (f >> 1)] >> ((f & 1) * 16)) & 0xFFFFu;  // pid | i << 9
                    ti = v2 & 0x1FFu;
                    fi = v2 >> 9;
                }
                const float b2 = fine[f * K1M + fi];
                float2 ec;
                if constexpr (DIRECT) {  // E and c2 of this part, in T's roundings
                    const float a2 = fine[f * K1M + (ti >> 5)];
                    ec.y = __ldg(p.c2v + f * 1024 + ti);
                    ec.x = __fsub_rn(__fsub_rn(a2, b2), ec.y);
                } else if constexpr (C3) {  // c2 by code, a2 = fine[f][j] with j = (t − i) & 15
                    const float a2 = fine[f * K1M + ((ti - fi) & 15u)];
                    ec.y = Ct[f * TE + ti];
                    ec.x = __fsub_rn(__fsub_rn(a2, b2), ec.y);
                } else if constexpr (S2) {  // E and c2 from two 4-byte tables (32 banks each)
                    const float* Et = reinterpret_cast<const float*>(smem);
                    ec.x = Et[f * TE + ti];
                    ec.y = Et[LT * TE + f * TE + ti];
                } else {
                    ec = T[f * TE + ti];
                }
                float qf;  // λq as a float: exact either way (q <= 255)
                if constexpr (I2F) {
                    qf = __uint2float_rn(lq);
                } else {
                    // one byte permute builds 2^23 + q (0x4B0000qq) from the code word, one FADD
                    // removes 2^23: no I2F (one more instruction per part than I2F.U8)
                    const uint32_t bsel = K1M == 16 ? (0x7540u | ((f & 1) * 2)) : (0x7540u | (f & 3));
                    const uint32_t src = K1M == 16 ? w[f >> 1] : w[f >> 2];
                    qf = __fsub_rn(__uint_as_float(__byte_perm(src, 0x4B000000u, bsel)), 8388608.0f);
                }
                const float lam = __fmul_rn(qf, inv255);
                const float part = __fadd_rn(__fadd_rn(b2, __fmul_rn(__fmul_rn(lam, lam), ec.y)), __fmul_rn(lam, ec.x));
                total = __fadd_rn(total, part);
            }
            const uint32_t od = orderable(total);
            key = ((uint64_t)od << 32) | id;
            kand &= od;
            kor |= od;
            ++mine;
        }
        keys[j] = key;
    };
    // PK: two candidates per thread scored together in packed fp32 pairs (sm_100 FADD2/FMUL2,
    // __fadd2_rn/__fmul2_rn: each lane rounds like __fadd_rn/__fmul_rn, so linequant.cpp:171-181's
    // order holds for each candidate; no FFMA/FFMA2 may appear in this kernel's SASS). Per part
    // the three table values come from conflict-light lookups: b2 = fine[f][i] and a2 = fine[f][j]
    // (one 16-float row: distinct centroids sit in distinct banks) and c2 = Ct[f][t] (t's low
    // nibble (i + j) & 15 spreads a part's pairs over the banks); E = (a2 - b2) - c2 is formed per
    // candidate in linequant.hpp:85's rounding. This trades T's 8-byte gather (2.3x its ideal
    // wavefronts on DEEP-shaped codes, tools/bank_probe.py) for two conflict-free 4-byte reads.
    // λ = fl(q · fl(1/255)) with q = (2^23 + q) − 2^23 built from the code byte by one byte
    // permute (exact for q <= 255) instead of an I2F.
    // this CTA's slice of the query's candidates: all of them, or, when a small batch spreads each
    // query over S = gridDim.y CTAs, every S-th one from blockIdx.y (interleaved, so every slice
    // samples near and far bins alike and the slices' top-k lists have similar ranges, which keeps
    // the merge's cut tight). Slice candidate u is candidate y + u·S; its key goes to keys[kb + u]
    // (slices own disjoint key ranges, in candidate order).
    const uint32_t S_ = gridDim.y, y_ = blockIdx.y;
    const uint32_t jn = Cn > y_ ? (Cn - y_ + S_ - 1) / S_ : 0u;
    const uint32_t kb = y_ * (Cn / S_) + (y_ < Cn % S_ ? y_ : Cn % S_);
    const uint32_t jhi = kb + jn;
    auto score2 = [&](uint32_t ja, const uint4* va, uint32_t ida, uint32_t jb, const uint4* vb, uint32_t idb) {
        const uint32_t* wa = reinterpret_cast<const uint32_t*>(va);
        const uint32_t* wb = reinterpret_cast<const uint32_t*>(vb);
        float2 tot = make_float2(0.0f, 0.0f);
        const float2 magic = make_float2(-8388608.0f, -8388608.0f);
        const float2 inv2 = make_float2(inv255, inv255);
#pragma unroll
        for (int f = 0; f < LT; ++f) {
            constexpr uint32_t kSel[2] = {0x7540u, 0x7542u};  // byte 0 / 2 -> low byte of 0x4B0000xx
            const int sh = (f & 1) * 16;                      // this part's (λ, t) half of the word
            const uint32_t xa = wa[f >> 1], xb = wb[f >> 1];
            // shared addresses: c2 at c2s | t·4, b2 at fs | i·4, a2 at fs | j·4 with j = (t − i) & 15
            // (c2s is 1 KB-, fs 64 B-aligned and c2s ≡ fs mod 64, so (ca − ba) & 0x3C = (t − i)·4 & 0x3C)
            const uint32_t ca = ((xa >> (sh + 6)) & 0x3FCu) | c2s, cb = ((xb >> (sh + 6)) & 0x3FCu) | c2s;
            const uint32_t ba = ((xa >> (sh + 10)) & 0x3Cu) | fs, bb = ((xb >> (sh + 10)) & 0x3Cu) | fs;
            const uint32_t aa = ((ca - ba) & 0x3Cu) | fs, ab = ((cb - bb) & 0x3Cu) | fs;
            const float2 b2 = make_float2(lds_f32(ba + f * K1M * 4), lds_f32(bb + f * K1M * 4));
            const float2 a2 = make_float2(lds_f32(aa + f * K1M * 4), lds_f32(ab + f * K1M * 4));
            const float2 c2 = make_float2(lds_f32(ca + f * 1024), lds_f32(cb + f * 1024));
            const float2 e = __fadd2_rn(__fadd2_rn(a2, make_float2(-b2.x, -b2.y)), make_float2(-c2.x, -c2.y));
            const float2 q = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(xa, 0x4B000000u, kSel[f & 1])),
                                                    __uint_as_float(__byte_perm(xb, 0x4B000000u, kSel[f & 1]))),
                                        magic);
            const float2 lam = __fmul2_rn(q, inv2);
            const float2 l2c = __fmul2_rn(__fmul2_rn(lam, lam), c2);
            const float2 le = __fmul2_rn(lam, e);
            // the two adds that take a product stay scalar: ptxas (12.9) contracts FMUL2 -> FADD2
            // into FFMA2 even for explicit .rn and -fmad=false, which would change the rounding
            const float2 part = make_float2(__fadd_rn(__fadd_rn(b2.x, l2c.x), le.x),
                                            __fadd_rn(__fadd_rn(b2.y, l2c.y), le.y));
            tot = __fadd2_rn(tot, part);
        }
        uint64_t key = kSentinel;
        if (ida != kInvalid) {
            const uint32_t od = orderable(tot.x);
            key = ((uint64_t)od << 32) | ida;
            kand &= od;
            kor |= od;
            ++mine;
        }
        keys[ja] = key;
        if (jb < jhi) {
            key = kSentinel;
            if (idb != kInvalid) {
                const uint32_t od = orderable(tot.y);
                key = ((uint64_t)od << 32) | idb;
                kand &= od;
                kor |= od;
                ++mine;
            }
            keys[jb] = key;
        }
    };
    // two row buffers in turn: the next candidate's row is in flight while this one is scored,
    // with no register copies between iterations
    const uint32_t step = blockDim.x;
    if constexpr (PK) {
        // candidates j and j + step of this thread together; both rows are loaded before scoring
        uint4 va[kVec], vb[kVec];
        for (uint32_t u = tid; u < jn; u += 2 * step) {
            const uint32_t u2 = u + step;
            uint32_t ida = kInvalid, idb = kInvalid;
            fetch(y_ + u * S_, va, ida);
            if (u2 < jn) fetch(y_ + u2 * S_, vb, idb);
            score2(kb + u, va, ida, kb + u2, vb, idb);
        }
    } else if constexpr (DIRECT) {
        // a shard's share of the candidates is about one per thread: one row buffer (the
        // 64-register budget of two CTAs per SM has no room for a second)
        uint4 va[kVec];
        uint32_t ida = kInvalid;
        for (uint32_t u = tid; u < jn; u += step) {
            fetch(y_ + u * S_, va, ida);
            score(kb + u, va, ida);
        }
    } else if (HALF && S_ == 1) {
        // HALF (MODE 8, K1M = 16, L = 32): each 64-byte row in two 32-byte halves with three
        // half-row buffers in rotation: the next row's first half loads before this row's first
        // 16 parts, its second half (into the buffer just consumed) before the last 16 -- 24
        // registers of row buffers instead of 32, left to the scheduler for shared-memory loads
        auto rowptr = [&](uint32_t j, uint32_t& id) -> const uint4* {
            const uint32_t r = rid[j];
            uint64_t pos;
            if (cached) {
                pos = (uint32_t)(delta[r] + j);
            } else {
                const uint2 rl = __ldg(qr + r);
                pos = (uint64_t)rl.x + (j - rl.y);
            }
            id = kInvalid;
            if (clip || (pos >= p.shard_lo && pos < p.shard_hi)) {
                const uint64_t lp = pos - p.shard_lo;
                id = __ldg(p.ids + lp);
                return reinterpret_cast<const uint4*>(p.codes + lp * p.row_bytes);
            }
            return nullptr;
        };
        auto acc16 = [&](const uint4* h, float total, const int fbase) -> float {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(h);
#pragma unroll
            for (int ff = 0; ff < 16; ++ff) {
                const int f = fbase + ff;
                const uint32_t half = w[ff >> 1] >> ((ff & 1) * 16);
                const uint32_t ti = (half >> 8) & 0xFFu, fi = ti >> 4, lq = half & 0xFFu;
                const float b2 = fine[f * K1M + fi];
                const float2 ec = T[f * TE + ti];
                const float lam = __fmul_rn(__uint2float_rn(lq), inv255);
                total = __fadd_rn(total, __fadd_rn(__fadd_rn(b2, __fmul_rn(__fmul_rn(lam, lam), ec.y)), __fmul_rn(lam, ec.x)));
            }
            return total;
        };
        // one candidate: F / S its row halves, N the next row's first half; the next row's second
        // half goes to F once F is scored. Returns whether there is a next candidate.
        auto iter = [&](uint32_t j, uint4* F, uint4* S, uint4* N, uint32_t id, uint32_t& idn) -> bool {
            const bool more = j + step < jn;
            const uint4* nrow = nullptr;
            idn = kInvalid;
            if (more) {
                nrow = rowptr(j + step, idn);
                if (nrow) ldg256(nrow, N[0], N[1]);
            }
            float total = 0.0f;
            if (id != kInvalid) total = acc16(F, total, 0);
            if (nrow) ldg256(nrow + 2, F[0], F[1]);
            uint64_t key = kSentinel;
            if (id != kInvalid) {
                total = acc16(S, total, 16);
                const uint32_t od = orderable(total);
                key = ((uint64_t)od << 32) | id;
                kand &= od;
                kor |= od;
                ++mine;
            }
            keys[j] = key;
            return more;
        };
        uint4 A[2], B[2], Cb[2];
        uint32_t id = kInvalid, idn = kInvalid;
        if (tid < jn) {
            const uint4* row = rowptr(tid, id);
            if (row) {
                ldg256(row, A[0], A[1]);
                ldg256(row + 2, B[0], B[1]);
            }
            for (uint32_t j = tid;;) {
                if (!iter(j, A, B, Cb, id, idn)) break;
                j += step;
                id = idn;
                if (!iter(j, Cb, A, B, id, idn)) break;
                j += step;
                id = idn;
                if (!iter(j, B, Cb, A, id, idn)) break;
                j += step;
                id = idn;
            }
        }
    } else if (COOP && S_ == 1) {
        // warp-uniform trip count (every lane takes part in the shuffles); a lane past the end
        // scores nothing
        uint4 x[kVec], v[kVec];
        uint32_t idn = kInvalid, id = kInvalid;
        const uint32_t lane = tid & 31;
        if (tid - lane < jn) issue(tid, jn, x, idn);
        for (uint32_t j = tid; j - lane < jn; j += step) {
            finish(x, v);
            id = idn;
            if (j + step - lane < jn) issue(j + step, jn, x, idn);
            if (j < jn) score(j, v, id);
        }
    } else if (S_ == 1) {  // one CTA per query (the throughput path): candidate u is candidate u
        uint4 va[kVec], vb[kVec];
        uint32_t ida = kInvalid, idb = kInvalid;
        if (tid < jn) fetch(tid, va, ida);
        for (uint32_t j = tid; j < jn; j += 2 * step) {
            const uint32_t j2 = j + step;
            if (j2 < jn) fetch(j2, vb, idb);
            score(j, va, ida);
            if (j2 >= jn) break;
            if (j2 + step < jn) fetch(j2 + step, va, ida);
            score(j2, vb, idb);
        }
    } else {
        uint4 va[kVec], vb[kVec];
        uint32_t ida = kInvalid, idb = kInvalid;
        if (tid < jn) fetch(y_ + tid * S_, va, ida);
        for (uint32_t u = tid; u < jn; u += 2 * step) {
            const uint32_t u2 = u + step;
            if (u2 < jn) fetch(y_ + u2 * S_, vb, idb);
            score(kb + u, va, ida);
            if (u2 >= jn) break;
            if (u2 + step < jn) fetch(y_ + (u2 + step) * S_, va, ida);
            score(kb + u2, vb, idb);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, d);
        kor |= __shfl_xor_sync(0xffffffffu, kor, d);
        mine += __shfl_xor_sync(0xffffffffu, mine, d);
    }
    if ((tid & 31) == 0 && mine) {
        atomicAdd(&s_count, mine);
        // ids are taken as all-different: only the distance bits' common prefix is skipped
        atomicAnd(&s_sel.kand, ((unsigned long long)kand << 32));
        atomicOr(&s_sel.kor, ((unsigned long long)kor << 32) | 0xFFFFFFFFull);
    }
    __syncthreads();
    PQTG_PHASE(3);
    const uint32_t nvalid = s_count;
    const uint32_t kk = nvalid < k ? nvalid : k;
    uint32_t m = 0;
    // (ranking a split slice's ~256 keys directly, without the select, measured slower at batch 1:
    // the count is quadratic and the one SM is issue-bound on it -- select 1.3 + rank 1.5 µs
    // against 3.8 µs)
    if (kk) {
        for (uint32_t i = tid; i < (1u << kSelBits); i += blockDim.x) hist[i] = 0;
        __syncthreads();
        if (GRP)
            m = block_select_wide<kSelBits, kIjThreads, true>(keys + kb, jn, kk, s_sel.kand, s_sel.kor, hist, sel,
                                                              sel_cap, wmax, s_sel);
        else
            m = block_select_wide<kSelBits, kIjThreads>(keys + kb, jn, kk, s_sel.kand, s_sel.kor, hist, sel, sel_cap,
                                                        wmax, s_sel);
    }
    PQTG_PHASE(4);
    if (gridDim.y == 1) {
        if (GRP && kk && s_sel.grouped)
            block_sort_write_grouped<kSelBits>(sel, m, kk, k, q, hist, s_sel.shift, out_ids, out_dists, out_counts);
        else
            block_sort_write(sel, m, kk, k, q, out_ids, out_dists, out_counts);
        PQTG_PHASE(5);
        qt_end(p, q, 2);
        return;
    }
    // split: this slice's top-kk keys to its list (sorted, padded to k with kSentinel), then the
    // query's last-arriving slice ranks the union's top k (threadfence-reduction pattern: no
    // second launch)
    const uint32_t S = gridDim.y;
    if (p.split_cluster) {
        // the query's slices are one cluster: slice y ranks its list into keys[y·k ..) of its own
        // shared memory, every slice reads the others' lists through distributed shared memory,
        // and after a second barrier (no slice's memory is read any more) each one cuts the lists
        // the same way and ranks 1/S of the kept keys (below)
        const uint32_t y = blockIdx.y;
        if (GRP && kk && s_sel.grouped) block_rank_keys_grouped<kSelBits>(sel, m, kk, hist, s_sel.shift, keys + y * k);
        else block_rank_keys(sel, m, kk, keys + y * k);
        for (uint32_t i = kk + tid; i < k; i += blockDim.x) keys[y * k + i] = kSentinel;
        PQTG_PHASE(5);
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        PQTG_PHASE(7);
        for (uint32_t i = tid; i < (S - 1) * k; i += blockDim.x) {
            const uint32_t rr = i / k, r = rr + (rr >= y), j = i - rr * k;
            keys[r * k + j] = cl.map_shared_rank(keys, r)[r * k + j];
        }
        cl.sync();
    } else {
        uint64_t* lst = split_keys + ((uint64_t)q * kSplitMax + blockIdx.y) * k;
        if (GRP && kk && s_sel.grouped) block_rank_keys_grouped<kSelBits>(sel, m, kk, hist, s_sel.shift, lst);
        else block_rank_keys(sel, m, kk, lst);
        for (uint32_t i = kk + tid; i < k; i += blockDim.x) lst[i] = kSentinel;
        PQTG_PHASE(5);
        __threadfence();
        __syncthreads();
        __shared__ uint32_t s_last;
        if (tid == 0) s_last = atomicAdd(&split_ctr[q], 1u) == S - 1;
        __syncthreads();
        if (!s_last) return;
        PQTG_PHASE(7);
        __threadfence();
        // the S lists (contiguous, stride k) into keys[0, S·k) in one pass; the kept keys' list
        // map goes behind them (2·S·k keys <= budget, rerank_split)
        const uint64_t* src = split_keys + (uint64_t)q * kSplitMax * k;
        for (uint32_t i = tid; i < S * k; i += blockDim.x) keys[i] = __ldcg(src + i);
        if (tid == 0) split_ctr[q] = 0;  // ready for the next call
        __syncthreads();
    }
    PQTG_PHASE(8);
    // per list (lane g): its length n_g (keys below kSentinel); k2 = min(k, Σ n_g). The first
    // c = ceil(k2 / S) keys of every list are <= M, the largest of their last keys, so when those
    // prefixes hold >= k2 keys the top k2 of the union are all <= M: each list is cut at M, and a
    // kept key's rank among the kept keys is its rank in the union.
    __shared__ uint32_t s_len[kSplitMax], s_off[kSplitMax + 1], s_k2;
    auto lower = [&](const uint64_t* l, uint32_t n, uint64_t x) {  // keys of sorted l[0, n) below x
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (l[mid] < x) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    if (tid < 32) {
        const uint32_t n = tid < S ? lower(keys + tid * k, k, kSentinel) : 0u;
        uint32_t tot = n;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
        const uint32_t k2 = tot < k ? tot : k;
        const uint32_t c = (k2 + S - 1) / S;
        uint32_t have = n < c ? n : c;
        uint64_t mx = have ? keys[tid * k + have - 1] : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, mx, d);
            mx = o > mx ? o : mx;
            have += __shfl_xor_sync(0xffffffffu, have, d);
        }
        const uint64_t thr = have >= k2 ? mx : kSentinel - 1;
        const uint32_t len = tid < S ? lower(keys + tid * k, n, thr + 1) : 0u;  // keys <= thr
        uint32_t incl = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
            if (tid >= (uint32_t)d) incl += v;
        }
        if (tid < S) s_len[tid] = len;
        if (tid <= S) s_off[tid] = incl - len;
        if (tid == 0) {
            s_k2 = k2;
            s_sel.kand = ~0ull;
            s_sel.kor = 0ull;
        }
    }
    __syncthreads();
    PQTG_PHASE(9);
    // the kept keys, compacted behind the lists, ranked by counting and written at their ranks
    const uint32_t k2 = s_k2, E = s_off[S];
    PQTG_PHASE_VAL(12, E);
    uint64_t* kept = keys + (uint64_t)S * k;
    for (uint32_t i = tid; i < S * k; i += blockDim.x) {
        const uint32_t g = i / k, j = i - g * k;
        if (j < s_len[g]) kept[s_off[g] + j] = keys[i];
    }
    __syncthreads();
    PQTG_PHASE(10);
    if (p.split_cluster) {
        // this slice's share of the kept keys, each counted against all of them by g threads
        const uint32_t y = blockIdx.y, lo = E * y / S, nm = E * (y + 1) / S - lo;
        uint32_t n2 = 1;
        while (n2 < nm) n2 <<= 1;
        uint32_t g = blockDim.x / n2;
        g = g > 32 ? 32 : (g ? g : 1);
        for (uint32_t base = 0; base < nm; base += blockDim.x / g) {
            const uint32_t e = base + tid / g, sub = tid % g;
            const bool own = e < nm;
            const uint64_t me = own ? kept[lo + e] : 0ull;
            uint32_t cnt = 0;
            if (own) {
                uint32_t j = sub;
                for (; j + 3 * g < E; j += 4 * g)  // four loads in flight
                    cnt += (uint32_t)(kept[j] < me) + (uint32_t)(kept[j + g] < me) + (uint32_t)(kept[j + 2 * g] < me) +
                           (uint32_t)(kept[j + 3 * g] < me);
                for (; j < E; j += g) cnt += kept[j] < me;
            }
            for (uint32_t o = 1; o < g; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (own && sub == 0 && cnt < k2) {
                out_ids[q * k + cnt] = (uint32_t)(me & 0xFFFFFFFFu);
                out_dists[q * k + cnt] = unorderable((uint32_t)(me >> 32));
            }
        }
        if (y == 0) {
            for (uint32_t i = k2 + tid; i < k; i += blockDim.x) {
                out_ids[q * k + i] = 0xFFFFFFFFu;
                out_dists[q * k + i] = __uint_as_float(0x7F800000u);
            }
            if (tid == 0) out_counts[q] = k2;
        }
    } else if (E <= blockDim.x) {
        block_sort_write(kept, E, k2, k, q, out_ids, out_dists, out_counts);
    } else {  // a loose cut: select the top k2 of the kept keys first
        uint64_t a = ~0ull, o = 0ull;
        for (uint32_t j = tid; j < E; j += blockDim.x) {
            a &= kept[j];
            o |= kept[j];
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a &= __shfl_xor_sync(0xffffffffu, a, d);
            o |= __shfl_xor_sync(0xffffffffu, o, d);
        }
        if ((tid & 31) == 0) {
            atomicAnd(&s_sel.kand, (unsigned long long)a);
            atomicOr(&s_sel.kor, (unsigned long long)o);
        }
        for (uint32_t i = tid; i < (1u << kSelBits); i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint32_t m2 = block_select_wide<kSelBits, kIjThreads>(kept, E, k2, s_sel.kand, s_sel.kor, hist, sel,
                                                                    sel_cap, wmax, s_sel);
        block_sort_write(sel, m2, k2, k, q, out_ids, out_dists, out_counts);
    }
    PQTG_PHASE(6);
    qt_end(p, q, 2);
}

namespace {

template <int LT, int K1M, bool DIRECT = false, int MODE = 0>
void allow(int optin) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, rerank_ij_kernel<LT, K1M, DIRECT, MODE>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(rerank_ij_kernel<LT, K1M, DIRECT, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes));
}

// The packed two-candidate loop (PK) is an opt-in variant (PQTG_RERANK=packed): bit-exact (the
// GPU parity suite passes with it as the default), but slower on B200 -- DEEP100M 1438 vs 1402 us,
// SIFT1M 1388 vs 1133 us, GIST1M 157 vs 130 us per batch (profiles/r02/rerank_packed_ab.md): it
// cuts the L1 data-pipe wavefronts 20% (134 M -> 108 M per 5000 queries) but adds 20% more
// instructions, and the scalar loop was co-limited by both.
int ij_mode() {
    static const int mode = [] {
        const char* e = std::getenv("PQTG_RERANK");
        if (e && std::strcmp(e, "packed") == 0) return 1;
        if (e && std::strcmp(e, "c3") == 0) return 2;
        if (e && std::strcmp(e, "split") == 0) return 3;
        if (e && std::strcmp(e, "coop") == 0) return 4;
        if (e && std::strcmp(e, "narrow") == 0) return 5;
        if (e && std::strcmp(e, "prmt") == 0) return 6;
        if (e && std::strcmp(e, "onecta") == 0) return 7;  // one CTA per SM, up to 128 registers
        if (e && std::strcmp(e, "half") == 0) return 8;    // half-row buffers in rotation
        if (e && std::strcmp(e, "grouped") == 0) return 9;  // = the default (top-k ranked within radix bins)
        if (e && std::strcmp(e, "ungrouped") == 0) return 10;  // top-k ranked over all kept keys
        return 0;
    }();
    return mode;
}

int code_k1m(const DevParams& p) { return p.code_ij ? 16 : (p.code_pi ? 32 : 0); }

// DIRECT when this index re-ranks a small share of each query's candidates: a position shard
// holding at most a quarter of the lists (about budget / 4 candidates per query)
bool ij_direct(const DevParams& p) { return code_k1m(p) == 32 && p.code_j; }  // decided at upload

int optin_smem() {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return optin;
}

int ij_mode();

size_t ij_smem(const DevParams& p, uint32_t k, bool gkeys) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    const bool pk = code_k1m(p) == 16 && (ij_mode() == 1 || ij_mode() == 2);
    return ij_layout(p.L, p.budget, ij_sel_cap(kk), code_k1m(p) ? code_k1m(p) : 16, ij_direct(p), gkeys, pk).total;
}

}  // namespace

bool rerank_needs_fixed_slots() { return ij_mode() == 1 || ij_mode() == 2; }

// keys go to the workspace when the shared-memory layout with them does not fit
bool rerank_ij_gkeys(const DevParams& p, uint32_t k) { return ij_smem(p, k, false) + 4096 > (size_t)optin_smem(); }

namespace {

}  // namespace

bool rerank_ij_ok(const DevParams& p, uint32_t k) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int k1m = code_k1m(p);
    const bool shape = k1m == 16 ? (p.L == 16 || p.L == 32 || p.L == 64) : (k1m == 32 && (p.L == 16 || p.L == 32));
    return shape && p.budget <= 65535 && p.npairs <= (k1m == 16 ? 128u : 512u) &&
           ij_smem(p, k, true) + 4096 <= (size_t)optin;
}

unsigned long long* phase_buffer() {
    static unsigned long long* buf = [] {
        unsigned long long* b = nullptr;
        const char* e = std::getenv("PQTG_PHASES");
        if (e && std::strcmp(e, "1") == 0 && cudaMalloc(&b, 16 * sizeof(unsigned long long)) == cudaSuccess) {
            cudaMemset(b, 0, 16 * sizeof(unsigned long long));  // device memory: no page faults in the clocks
            cudaMemcpyToSymbol(g_phase, &b, sizeof(b));
        }
        return b;
    }();
    return buf;
}

void configure_rerank_ij() {
    phase_buffer();
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    allow<16, 16>(optin);
    allow<32, 16>(optin);
    allow<64, 16>(optin);
    allow<16, 16, false, 1>(optin);
    allow<32, 16, false, 1>(optin);
    allow<64, 16, false, 1>(optin);
    allow<16, 16, false, 2>(optin);
    allow<16, 16, false, 3>(optin);
    allow<32, 16, false, 3>(optin);
    allow<64, 16, false, 3>(optin);
    allow<32, 16, false, 2>(optin);
    allow<16, 16, false, 4>(optin);
    allow<32, 16, false, 4>(optin);
    allow<64, 16, false, 4>(optin);
    allow<16, 16, false, 5>(optin);
    allow<32, 16, false, 5>(optin);
    allow<64, 16, false, 5>(optin);
    allow<16, 16, false, 6>(optin);
    allow<32, 16, false, 6>(optin);
    allow<64, 16, false, 6>(optin);
    allow<32, 16, false, 7>(optin);
    allow<32, 16, false, 8>(optin);
    allow<32, 16, false, 9>(optin);
    allow<32, 16, false, 10>(optin);
    allow<64, 16, false, 2>(optin);
    allow<16, 32>(optin);
    allow<32, 32>(optin);
    allow<16, 32, true>(optin);
    allow<32, 32, true>(optin);
}

// CTAs per query: a batch below one query per SM can spread each query's candidates over up to
// kSplitMax CTAs; each slice ranks its top-k keys into a list and the query's last-arriving
// slice merges the lists (default; PQTG_SPLIT=0 keeps one CTA per query)
uint32_t rerank_split(const DevParams& p, uint64_t nq, uint32_t k) {
    static const bool off = [] {
        const char* e = std::getenv("PQTG_SPLIT");
        return e && std::strcmp(e, "0") == 0;
    }();
    if (off || nq == 0 || nq >= kSplitBelow || p.budget < 1024 || !rerank_ij_ok(p, k)) return 1;
    // the last slice gathers the S lists of k keys into its key array, with room behind: 2·S·k <= budget
    // 8 slices (a portable cluster): batch 1 as fast as 12 or 16 (29.7-30.0 µs), batch 10 faster
    // (31.7 against 33.6 µs with 16: a merge of 8 lists instead of 16); PQTG_SPLIT_MAX (2..16)
    // overrides for experiments
    static const uint64_t smax = [] {
        const char* e = std::getenv("PQTG_SPLIT_MAX");
        const long v = e ? std::strtol(e, nullptr, 10) : 0;
        return v >= 2 && v <= (long)kSplitMax ? (uint64_t)v : (uint64_t)8;
    }();
    const uint64_t s = std::min<uint64_t>(std::min<uint64_t>((2 * kSplitBelow) / nq, p.budget / 256),
                                          std::min<uint64_t>(p.budget / (2ull * k), smax));
    return s >= 2 ? (uint32_t)s : 1u;
}

// Whether S-CTA clusters of this re-rank variant (threads, sm bytes) can be resident
// (cudaOccupancyMaxActiveClusters; clusters above 8 CTAs need the non-portable opt-in), per device;
// PQTG_SPLIT_CLUSTER=0 keeps the global-memory merge
template <class Kernel>
bool split_cluster_ok(Kernel kernel, uint32_t S, int threads, size_t sm) {
    static const bool off = [] {
        const char* e = std::getenv("PQTG_SPLIT_CLUSTER");
        return e && std::strcmp(e, "0") == 0;
    }();
    if (off || S < 2 || S > kSplitMax) return false;
    int dev = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<std::tuple<const void*, uint32_t, int, size_t, int>, bool> known;
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), S, threads, sm, dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto it = known.find(key);
    if (it != known.end()) return it->second;
    bool ok = S <= 8 || cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    if (ok) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(1, S, 1);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 1;
        at.val.clusterDim.y = S;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        int n = 0;
        ok = cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) == cudaSuccess && n > 0;
    }
    cudaGetLastError();
    known[key] = ok;
    return ok;
}

void launch_rerank_ij(const DevParams& p, uint64_t nq, uint32_t k, const WsSlice& ws, uint32_t* ids, float* dists,
                      uint32_t* counts, cudaStream_t s) {
    const uint32_t S = rerank_split(p, nq, k);
    if (S > 1 && (!ws.split_keys || ws.split_k < k || ws.split_q < nq)) throw Error{PQTG_ERR_ARG, "workspace has no split lists"};
    const uint32_t kk = k < p.budget ? k : p.budget;
    const uint32_t cap = ij_sel_cap(kk);
    const bool gk = rerank_ij_gkeys(p, k);
    if (gk && !ws.keys) throw Error{PQTG_ERR_ARG, "workspace has no candidate-key buffer for this budget"};
    const size_t sm = ij_smem(p, k, gk);
    uint64_t* gkeys = gk ? ws.keys : nullptr;
    // a split query's S slices as one cluster (lists through DSMEM) when its shape can be resident
    auto launch_ij = [&](auto kernel, int threads) {
        DevParams pl = p;
        pl.split_cluster = (S > 1 && !gk && split_cluster_ok(kernel, S, threads, sm)) ? 1u : 0u;
        launch_kernel_cluster(p.chain, dim3(1, pl.split_cluster ? S : 1, 1), kernel, dim3((unsigned)nq, S),
                              dim3(threads), sm, s, pl, k, cap, ws.fine, ws.ranges, ws.nranges, ws.ncand, ids, dists,
                              counts, gkeys, ws.split_keys, ws.split_ctr);
    };
#define PQTG_IJ(LT, K, D, ...) launch_ij(rerank_ij_kernel<LT, K, D, ##__VA_ARGS__>, ij_threads(LT, D))
    if (code_k1m(p) == 32) {
        const bool direct = ij_direct(p);
        if (p.L == 16) {
            if (direct) PQTG_IJ(16, 32, true); else PQTG_IJ(16, 32, false);
        } else {
            if (direct) PQTG_IJ(32, 32, true); else PQTG_IJ(32, 32, false);
        }
    } else if (ij_mode() == 1) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 1); break;
        case 32: PQTG_IJ(32, 16, false, 1); break;
        default: PQTG_IJ(64, 16, false, 1); break;
        }
    } else if (ij_mode() == 2) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 2); break;
        case 32: PQTG_IJ(32, 16, false, 2); break;
        default: PQTG_IJ(64, 16, false, 2); break;
        }
    } else if (ij_mode() == 9 && p.L == 32) {
        PQTG_IJ(32, 16, false, 9);
    } else if (ij_mode() == 10 && p.L == 32) {
        PQTG_IJ(32, 16, false, 10);
    } else if (ij_mode() == 8 && p.L == 32) {
        PQTG_IJ(32, 16, false, 8);
    } else if (ij_mode() == 7 && p.L == 32) {
        PQTG_IJ(32, 16, false, 7);
    } else if (ij_mode() == 6) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 6); break;
        case 32: PQTG_IJ(32, 16, false, 6); break;
        default: PQTG_IJ(64, 16, false, 6); break;
        }
    } else if (ij_mode() == 5) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 5); break;
        case 32: PQTG_IJ(32, 16, false, 5); break;
        default: PQTG_IJ(64, 16, false, 5); break;
        }
    } else if (ij_mode() == 4) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 4); break;
        case 32: PQTG_IJ(32, 16, false, 4); break;
        default: PQTG_IJ(64, 16, false, 4); break;
        }
    } else if (ij_mode() == 3) {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false, 3); break;
        case 32: PQTG_IJ(32, 16, false, 3); break;
        default: PQTG_IJ(64, 16, false, 3); break;
        }
    } else {
        switch (p.L) {
        case 16: PQTG_IJ(16, 16, false); break;
        case 32: PQTG_IJ(32, 16, false); break;
        default: PQTG_IJ(64, 16, false); break;
        }
    }
#undef PQTG_IJ
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
