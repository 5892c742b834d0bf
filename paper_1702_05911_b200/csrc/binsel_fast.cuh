// binsel_fast.cuh — K3 fast path body (bin selection + gather) as a device function over a
// group of kBsThreads threads with a caller-chosen barrier, so it can run inside other kernels
// (a fused bin-selection + re-rank kernel measured slower: DESIGN.md §5). The stand-alone kernel
// is binsel_fast.cu; references: binorder.cpp:178-283, search.cpp:139-217.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using namespace dev;

namespace bsf {

constexpr int kBsThreads = 256;
constexpr int kFilterWarps = kBsThreads / 32 - 1;  // warp 0 walks the queue
constexpr int kFilterThreads = kFilterWarps * 32;
constexpr int kMaxItems = 8;
constexpr uint32_t kQueueCap = kFilterThreads * kMaxItems;
constexpr int kWalkAhead = 4;  // walker batches whose bin extents are in flight
// the walker's visited set: a shared open-addressing table of slot + 1 (0 = free); past half
// full it moves to the query's global table, which is sized for the whole budget
constexpr uint32_t kVisLog2 = 10;
constexpr uint32_t kVis = 1u << kVisLog2;

__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t H) {
    const uint64_t x = (uint64_t)a + b;
    return (uint32_t)(x >= H ? x - H : x);
}

struct BsLayout {
    size_t terms, ta, tb, queue, hash, svis, total;
};

__host__ __device__ inline BsLayout bs_layout(uint32_t PW, uint32_t W2ab, uint32_t ts) {
    BsLayout l{};
    size_t o = 0;
    l.terms = o;
    o += ((size_t)PW * 4 + 15) & ~size_t(15);
    l.ta = o;
    o += (size_t)W2ab * 4;
    l.tb = o;
    o += (size_t)W2ab * 4;
    l.queue = o;
    o += (size_t)2 * kQueueCap * 8;  // double-buffered
    l.hash = o;
    o += (size_t)ts * 4;
    l.svis = o;  // the walker's shared visited set
    o += (size_t)kVis * 4;
    l.total = o;
    return l;
}

// One filter pass for one thread: NIT stream positions base + it·NT + ft (NT filter threads). Slot = the sum of
// pre-reduced per-part terms mod H (pqtree.cpp:12-25); non-empty = the slot's bitmap bit.
// Loads of all items are issued before any is consumed; positions are 32-bit.
__device__ __forceinline__ uint32_t add_mod_fast(uint32_t a, uint32_t b, uint32_t H) {
    const uint32_t x = a + b;  // a, b < H < 2^31
    return min(x, x - H);      // x - H wraps above x when x < H
}

// The non-empty bits of NIT slots: the fine bitmap word of each, looked up only when the coarse
// bitmap (1 bit per 2^coarse_shift slots, L1-resident, built for sparse indexes) has the group.
template <int NIT>
__device__ __forceinline__ void probe_bitmap(const DevParams& p, const uint32_t* slot, uint32_t* word) {
    if (p.bitmap_coarse) {
        uint32_t cw[NIT];
#pragma unroll
        for (int it = 0; it < NIT; ++it) cw[it] = __ldg(p.bitmap_coarse + ((slot[it] >> p.coarse_shift) >> 5));
#pragma unroll
        for (int it = 0; it < NIT; ++it)
            word[it] = ((cw[it] >> ((slot[it] >> p.coarse_shift) & 31u)) & 1u) ? __ldg(p.bitmap + (slot[it] >> 5)) : 0u;
    } else {
#pragma unroll
        for (int it = 0; it < NIT; ++it) word[it] = __ldg(p.bitmap + (slot[it] >> 5));
    }
}

template <int P, int NIT, int NT = kFilterThreads>
__device__ __forceinline__ void filter(const DevParams& p, uint32_t base, uint32_t total, int ft, int lane, int fw,
                                       uint32_t ta, uint32_t tb, uint32_t W, uint32_t H, const uint32_t* terms,
                                       const uint32_t* tA, const uint32_t* tB, uint32_t W2ab, uint32_t* slot,
                                       uint32_t* ball, uint32_t* wcnt) {
    const uint32_t W2 = (uint32_t)p.W2;
    const uint32_t mcount = (uint32_t)p.merge_count;
    const uint32_t end = base + NIT * NT;  // positions of this pass: [base, end)
    // uniform fast path: the whole pass lies inside the stream and (P = 4) inside the
    // materialized merge prefix, so no item needs a bounds or closed-form check
    const bool fast = end <= total &&
                      (P != 4 || (end <= mcount && p.merge16 && (W2ab == W2 || end <= p.merge_fold_end) &&
                                  H < 0x80000000u)) &&
                      (P != 2 || H < 0x80000000u);
    uint32_t word[NIT];
    if (fast) {
        if constexpr (P == 4) {
            const uint32_t* mp = p.merge16 + base + ft;  // fast path: every (u, v) of the pass is folded
            uint32_t e[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) e[it] = __ldg(mp + it * NT);
#pragma unroll
            for (int it = 0; it < NIT; ++it) slot[it] = add_mod_fast(tA[e[it] & 0xFFFFu], tB[e[it] >> 16], H);
        } else if constexpr (P == 2) {
            const uint32_t* sp = p.pair_streams + (size_t)ta * W2 + base + ft;
            uint32_t e[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) e[it] = __ldg(sp + it * NT);
#pragma unroll
            for (int it = 0; it < NIT; ++it) slot[it] = add_mod_fast(terms[e[it] & 0xFFFFu], terms[W + (e[it] >> 16)], H);
        } else {
#pragma unroll
            for (int it = 0; it < NIT; ++it) slot[it] = terms[base + it * NT + ft];
        }
        probe_bitmap<NIT>(p, slot, word);
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            ball[it] = __ballot_sync(0xffffffffu, (word[it] >> (slot[it] & 31)) & 1u);
            if (lane == 0) wcnt[it * (NT / 32) + fw] = __popc(ball[it]);
        }
    } else {
        uint2 ent[NIT];
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const uint32_t s = base + it * NT + ft;
            ent[it] = make_uint2(0, 0);
            if (s < total) {
                if constexpr (P == 2) {
                    ent[it].x = __ldg(p.pair_streams + (size_t)ta * W2 + s);
                } else if constexpr (P == 4) {
                    if (s < mcount) {
                        ent[it] = __ldg(p.merge + s);
                    } else {  // closed-form sweep rows past the slope-1 table (binorder.cpp:96-108)
                        const uint32_t j = s - mcount;
                        const uint32_t u = j / W2;
                        ent[it] = make_uint2((uint32_t)p.merge_row0 + u, j - u * W2);
                    }
                }
            }
        }
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const uint32_t s = base + it * NT + ft;
            uint32_t sl = 0;
            if constexpr (P == 1) {
                sl = terms[s < total ? s : 0];
            } else if constexpr (P == 2) {
                const uint32_t e = ent[it].x;
                sl = add_mod(terms[e & 0xFFFFu], terms[W + (e >> 16)], H);
            } else {
                if (ent[it].x < W2ab && ent[it].y < W2ab) {  // both pair ranks inside the folded prefix
                    sl = add_mod(tA[ent[it].x], tB[ent[it].y], H);
                } else {
                    const uint32_t ea = __ldg(p.pair_streams + (size_t)ta * W2 + ent[it].x);
                    const uint32_t eb = __ldg(p.pair_streams + (size_t)tb * W2 + ent[it].y);
                    sl = add_mod(add_mod(terms[ea & 0xFFFFu], terms[W + (ea >> 16)], H),
                                 add_mod(terms[2 * W + (eb & 0xFFFFu)], terms[3 * W + (eb >> 16)], H), H);
                }
            }
            slot[it] = sl;
        }
        probe_bitmap<NIT>(p, slot, word);
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const uint32_t s = base + it * NT + ft;
            ball[it] = __ballot_sync(0xffffffffu, s < total && ((word[it] >> (slot[it] & 31)) & 1u));
            if (lane == 0) wcnt[it * (NT / 32) + fw] = __popc(ball[it]);
        }
    }
#pragma unroll
    for (int it = NIT; it < kMaxItems; ++it) ball[it] = 0;
}

// The walker (one warp): the next n queued non-empty tuples (stream position, slot) in stream
// order, 32 at a time — first occurrences by __match_any_sync within the batch plus the visited
// set across batches (HASH), the bins' extents, a warp prefix sum of their sizes and the budget
// cut (search.cpp:194-214). Emits (start position, candidate offset) ranges; c / r / maxord
// (candidates, ranges, last stream position used) carry across calls.
struct WalkState {
    uint32_t c, r, maxord, nvis;
    bool spilled;
};

template <bool HASH>
__device__ __forceinline__ void walk_queue(const DevParams& p, const uint2* qp, uint32_t n, WalkState& st,
                                           uint32_t budget, uint2* qranges, uint32_t* svis, uint32_t* hkeys,
                                           uint32_t ts_log2, int lane) {
    const uint32_t TS = 1u << ts_log2;
    uint32_t c = st.c, r = st.r, maxord = st.maxord, nvis = st.nvis;
    bool spilled = st.spilled;
    const uint32_t lt = (1u << lane) - 1u;
    // the bins' extents are loaded kWalkAhead batches ahead: with offsets larger than L2
    // (H = 2^26) each batch's extents are a DRAM round trip, the walker's critical path
    uint32_t pf_lo[kWalkAhead], pf_hi[kWalkAhead];
    auto prefetch = [&](uint32_t b0, int k) {
        const uint32_t idx = b0 + lane;
        if (idx < n) {
            const uint32_t sl = qp[idx].y;
            pf_lo[k] = __ldg(p.offsets + sl);
            pf_hi[k] = __ldg(p.offsets + sl + 1);
        }
    };
#pragma unroll
    for (int k = 0; k < kWalkAhead; ++k) prefetch(k * 32u, k);
    for (uint32_t g0 = 0; g0 < n && c < budget; g0 += 32u * kWalkAhead) {
#pragma unroll
        for (int k = 0; k < kWalkAhead; ++k) {
            const uint32_t b0 = g0 + 32u * k;
            if (b0 >= n || c >= budget) break;
            const uint32_t idx = b0 + lane;
            const bool has = idx < n;
            const uint2 e = has ? qp[idx] : make_uint2(0, kEmptyKey);
            uint32_t start = 0, cnt = 0;
            if (has) {
                start = pf_lo[k];
                cnt = pf_hi[k] - start;
            }
            prefetch(b0 + 32u * kWalkAhead, k);
            bool first = has;
            if (HASH) {
                const uint32_t grp = __match_any_sync(0xffffffffu, e.y);
                if (has && (uint32_t)(__ffs(grp) - 1) != (uint32_t)lane) first = false;  // earlier in batch
                bool fresh = false;
                if (first) {
                    if (!spilled) {
                        // shared visited set: keys slot + 1, 0 = free
                        const uint32_t key = e.y + 1u;
                        uint32_t h = (e.y * 0x9E3779B1u) >> (32 - kVisLog2);
                        for (;;) {
                            const uint32_t cur = svis[h];
                            if (cur == 0u) {
                                if (atomicCAS(svis + h, 0u, key) == 0u) {
                                    fresh = true;
                                    break;
                                }
                                continue;
                            }
                            if (cur == key) {
                                first = false;  // visited in an earlier batch
                                break;
                            }
                            h = (h + 1) & (kVis - 1);
                        }
                    } else {
                        const uint32_t key = e.y + 1u;
                        uint32_t h = (e.y * 0x9E3779B1u) >> (32 - ts_log2);
                        for (;;) {
                            const uint32_t cur = hkeys[h];
                            if (cur == 0u) {
                                if (atomicCAS(hkeys + h, 0u, key) == 0u) break;
                                continue;  // lost a race on this entry; re-read it
                            }
                            if (cur == key) {
                                first = false;  // visited in an earlier batch
                                break;
                            }
                            h = (h + 1) & (TS - 1);
                        }
                    }
                }
                nvis += __popc(__ballot_sync(0xffffffffu, fresh));
                if (!spilled && nvis > kVis / 2) {
                    // the shared set is half full: move it to the per-query global
                    // table (sized for the whole budget) and continue there
                    for (uint32_t i = lane; i < TS; i += 32) hkeys[i] = 0u;
                    __syncwarp();
                    for (uint32_t i = lane; i < kVis; i += 32) {
                        const uint32_t v = svis[i];
                        if (v == 0u) continue;
                        uint32_t h = ((v - 1u) * 0x9E3779B1u) >> (32 - ts_log2);
                        while (atomicCAS(hkeys + h, 0u, v) != 0u) h = (h + 1) & (TS - 1);
                    }
                    __syncwarp();
                    spilled = true;
                }
            }
            if (!first) cnt = 0;
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t before = c + (incl - cnt);  // < 2^32: distinct bins hold <= n ids
            const bool emit = first && before < budget;
            const uint32_t em = __ballot_sync(0xffffffffu, emit);
            if (emit) {
                qranges[r + __popc(em & lt)] = make_uint2(start, before);
                maxord = max(maxord, e.x);
            }
            maxord = __reduce_max_sync(0xffffffffu, maxord);
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            r += __popc(em);
            c = (uint64_t)c + tot >= budget ? budget : c + tot;
        }
    }
    st.c = c;
    st.r = r;
    st.maxord = maxord;
    st.nvis = nvis;
    st.spilled = spilled;
}

template <int P, bool HASH, class SYNC>
__device__ __forceinline__ void binsel_fast_body(const DevParams& p, uint64_t q, const uint32_t* __restrict__ l2c_in,
                                                 const float* __restrict__ l2d_in, uint8_t* __restrict__ slope_out,
                                                 uint2* __restrict__ ranges, uint32_t* __restrict__ nranges,
                                                 uint32_t* __restrict__ ncand, uint32_t* __restrict__ ntuples,
                                                 pqtg_query_stats* __restrict__ stats, uint32_t ts_log2,
                                                 uint32_t* __restrict__ ghash, uint32_t W2ab, unsigned char* smem,
                                                 uint32_t tid) {
    const uint32_t W = p.W, PW = P * W;
    const uint32_t H = (uint32_t)p.H;
    const BsLayout lay = bs_layout(PW, W2ab, 0);
    uint32_t* terms = reinterpret_cast<uint32_t*>(smem + lay.terms);
    uint32_t* tA = reinterpret_cast<uint32_t*>(smem + lay.ta);
    uint32_t* tB = reinterpret_cast<uint32_t*>(smem + lay.tb);
    uint2* queue = reinterpret_cast<uint2*>(smem + lay.queue);
    uint32_t* svis = reinterpret_cast<uint32_t*>(smem + lay.svis);
    uint32_t* hkeys = HASH ? ghash + (q << ts_log2) : nullptr;
    __shared__ uint32_t wcnt[2][64];
    __shared__ uint32_t s_nq[2], s_C, s_R, s_maxord;
    const int lane = tid & 31, warp = tid >> 5;
    __shared__ uint32_t s_slope[2];

    // slot terms (flat_part_code · (k1k2)^p) mod H, pqtree.cpp:12-25
    for (uint32_t idx = tid; idx < PW; idx += kBsThreads) {
        const uint32_t code = l2c_in[q * PW + idx];
        const uint64_t flat = (uint64_t)(code >> 16) * p.k2 + (code & 0xFFFFu);
        terms[idx] = (uint32_t)((flat * p.mult[idx / W]) % p.H);
    }
    if (HASH)
        for (uint32_t i = tid; i < kVis; i += kBsThreads) svis[i] = 0u;
    if (tid == 0) {
        s_C = 0;
        s_R = 0;
        s_maxord = 0;
    }
    if ((tid & 31) == 0 && tid < 64) {  // pick_slope_table (binorder.cpp:52-65), one pair per warp
        const uint32_t pr = tid >> 5, t = query_slope(p, l2d_in + q * PW, pr);
        s_slope[pr] = t;
        slope_out[q * 2 + pr] = (uint8_t)t;
    }
    SYNC::sync();
    const uint32_t ta = s_slope[0], tb = s_slope[1];
    if (P == 4 && W2ab) {  // fold each pair stream into per-pair-rank slot terms
        for (uint32_t u = tid; u < W2ab; u += kBsThreads) {
            const uint32_t ea = __ldg(p.pair_streams + (size_t)ta * p.W2 + u);
            const uint32_t eb = __ldg(p.pair_streams + (size_t)tb * p.W2 + u);
            tA[u] = add_mod(terms[ea & 0xFFFFu], terms[W + (ea >> 16)], H);
            tB[u] = add_mod(terms[2 * W + (eb & 0xFFFFu)], terms[3 * W + (eb >> 16)], H);
        }
        SYNC::sync();
    }

    const uint32_t budget = p.budget;
    const uint64_t total = p.total_tuples;
    uint2* qranges = ranges + q * (uint64_t)budget;
    // Warp 0 walks the queue of pass i-1 while warps 1..7 filter pass i (warp
    // specialization): per pass two barriers, and the queue's dependent loads (hash probe,
    // offsets) overlap the next pass's stream/bitmap loads.
    const int fw = warp - 1;                // filter warp index, -1 for warp 0
    const int ft = tid - 32;                // filter thread index
    // stream positions fit 32 bits (BinStream::total is capped at 2^32 - 2 at index build)
    const uint32_t total32 = (uint32_t)total;
    uint32_t base = 0;                      // first stream position of the pass being filtered
    // items per filter thread: 1 on the first pass, then 8; P = 4 streams reach thousands of
    // tuples per query, so they start with full passes
    uint32_t nit = P == 4 ? kMaxItems : 1;
    uint32_t prev_n = 0;                    // queued tuples of the previous pass
    uint32_t nvis = 0;                      // walker: slots inserted in the visited set
    bool spilled = false;                   // walker: visited set moved to global memory
    for (uint32_t pass = 0;; ++pass) {
        const uint32_t buf = pass & 1u;
        uint2* qb = queue + (size_t)buf * kQueueCap;
        uint32_t slot[kMaxItems], ball[kMaxItems];
        if (warp == 0) {
            // ---- queue of the previous pass, in stream order, 32 tuples at a time
            if (pass > 0 && prev_n > 0) {
                const uint2* qp = queue + (size_t)(buf ^ 1u) * kQueueCap;
                WalkState st{s_C, s_R, s_maxord, nvis, spilled};
                walk_queue<HASH>(p, qp, prev_n, st, budget, qranges, svis, hkeys, ts_log2, lane);
                nvis = st.nvis;
                spilled = st.spilled;
                const uint32_t c = st.c, r = st.r, maxord = st.maxord;
                __syncwarp();  // every lane read s_C / s_R / s_maxord above before lane 0 updates them
                if (lane == 0) {
                    s_C = c;
                    s_R = r;
                    s_maxord = maxord;
                }
            }
        } else if (base < total) {
            // ---- filter: slot + non-empty test of this pass's stream positions
            if (nit == 1) filter<P, 1>(p, base, total32, ft, lane, fw, ta, tb, W, H, terms, tA, tB, W2ab, slot, ball, wcnt[buf]);
            else filter<P, kMaxItems>(p, base, total32, ft, lane, fw, ta, tb, W, H, terms, tA, tB, W2ab, slot, ball, wcnt[buf]);
        }
        SYNC::sync();  // B1: counts of pass `pass`; C / R after the previous pass's queue
        // done: budget reached, or the stream ended and its last queue was just walked
        if (s_C >= budget || base >= total) break;
        // ---- order-preserving compaction (every filter warp scans the counts itself)
        uint32_t anyhit = 0;
#pragma unroll
        for (int it = 0; it < kMaxItems; ++it) anyhit |= ball[it];
        if (warp > 0 && (anyhit || warp == 1)) {  // a warp without hits has nothing to place
            const uint32_t n = nit * kFilterWarps;
            const uint32_t v0 = lane < (int)n ? wcnt[buf][lane] : 0;
            const uint32_t v1 = (uint32_t)(lane + 32) < n ? wcnt[buf][lane + 32] : 0;
            uint32_t i0 = v0, i1 = v1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t0 = __shfl_up_sync(0xffffffffu, i0, o);
                const uint32_t t1 = __shfl_up_sync(0xffffffffu, i1, o);
                if (lane >= o) {
                    i0 += t0;
                    i1 += t1;
                }
            }
            const uint32_t carry = __shfl_sync(0xffffffffu, i0, 31);
            const uint32_t ntot = carry + __shfl_sync(0xffffffffu, i1, 31);
            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
            for (int it = 0; it < kMaxItems; ++it) {
                if (it < (int)nit && ball[it]) {  // warp-uniform: most items hold no hit
                    // exclusive prefix of entry e = (item, filter warp) in stream order
                    const uint32_t e = it * kFilterWarps + fw;
                    const uint32_t src = e & 31u;
                    const uint32_t a0 = __shfl_sync(0xffffffffu, i0, src) - __shfl_sync(0xffffffffu, v0, src);
                    const uint32_t a1 = __shfl_sync(0xffffffffu, i1, src) - __shfl_sync(0xffffffffu, v1, src);
                    const uint32_t excl = e < 32 ? a0 : carry + a1;
                    if ((ball[it] >> lane) & 1u) {
                        qb[excl + __popc(ball[it] & lt)] =
                            make_uint2(base + it * kFilterThreads + ft, slot[it]);
                    }
                }
            }
            if (warp == 1 && lane == 0) s_nq[buf] = ntot;
        }
        SYNC::sync();  // B2: queue of pass `pass` complete
        prev_n = s_nq[buf];
        base += nit * kFilterThreads;
        nit = kMaxItems;
    }
    if (tid == 0) {
        const uint32_t C = s_C, R = s_R;
        nranges[q] = R;
        ncand[q] = C;
        ntuples[q] = C >= budget && budget > 0 ? s_maxord + 1 : min(base, total32);
        if (stats) {
            stats[q].bins_visited = R;
            stats[q].candidates = C;
            stats[q].exact_evals = 0;
        }
    }
}


struct BsConfig {
    uint32_t ts_log2, use_hash, W2ab;
    size_t smem;
};

inline BsConfig bs_config(const DevParams& p) {
    BsConfig c{};
    // two tuples can reach one slot only if the positional code space exceeds H
    long double span = 1.0L;
    for (uint32_t i = 0; i < p.P; ++i) span *= (long double)p.k1 * p.k2;
    c.use_hash = span > (long double)p.H ? 1u : 0u;
    c.ts_log2 = 6;
    while ((1ull << c.ts_log2) < ((uint64_t)p.budget + 32) * 3 / 2) ++c.ts_log2;
    // P = 4: the pair streams folded into per-pair-rank slot terms -- whole when W² <= 4096
    // (GIST1M), else their first 256 ranks (SIFT1B's W² = 16384: the merge stream's first few
    // thousand tuples stay below pair rank ~64), past which a tuple loads its pair-stream entries
    c.W2ab = p.P == 4 ? (uint32_t)(p.W2 <= 4096 ? p.W2 : kPartialFold) : 0u;
    c.smem = bs_layout(p.P * p.W, c.W2ab, 0).total;
    return c;
}

// barrier of the whole CTA (the stand-alone kernel)
struct SyncBlock {
    __device__ __forceinline__ static void sync() { __syncthreads(); }
};

// named barrier 1 over the kBsThreads threads of a bin-selection group inside a larger CTA
struct SyncBinselGroup {
    __device__ __forceinline__ static void sync() {
        asm volatile("bar.sync 1, %0;" ::"n"(kBsThreads) : "memory");
    }
};

}  // namespace bsf
}  // namespace pqtg
