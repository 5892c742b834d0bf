// binsel_par.cu — K3 bin selection + gather with every warp working on every pass
// (binorder.cpp:178-283, search.cpp:139-217), for indexes whose slot arithmetic fits 32 bits.
//
// binsel_fast walks each pass's non-empty tuples with ONE warp (32 at a time: dedup, the bins'
// extents, a prefix sum, the budget cut) while the other seven filter the next pass. When most
// probed slots are non-empty but repeat -- P = 4 at H = 2^26, where (k1·k2)^3 ≡ 0 mod H makes the
// fourth part's rank vanish from the slot -- that walk is the whole kernel (SIFT1B: ~860 queued
// tuples per query, 27 serial warp steps). Here a pass of 2048 stream positions is finished by
// all 256 threads together:
//   1. slot + bitmap test per position (bsf::filter),
//   2. (HASH) first occurrence: each non-empty position inserts its slot into a visited set of
//      (slot + 1, smallest position) entries — 2048 in shared memory, moved to the query's
//      global table when 3/4 full — with atomicMin on the position; after a barrier a position
//      is its slot's first occurrence iff the entry holds it (earlier passes hold smaller ones),
//   3. the first occurrences' extents offsets[s], offsets[s + 1], all loads in flight at once,
//   4. one block-wide exclusive scan, in stream order, of (bin size, first flag): the candidate
//      offset of each bin and its range index; the budget cut (search.cpp:209-214) keeps every
//      first occurrence whose offset is below the budget — a prefix, since offsets only grow.
// Output is the same (start position, candidate offset) range list as binsel_fast.
#include <cstdint>

#include "binsel_fast.cuh"

namespace pqtg {

using namespace dev;
using namespace bsf;

namespace bsp {

constexpr int kPItems = 8;
constexpr uint32_t kPassMax = 256 * kPItems;         // stream positions per full pass
constexpr uint32_t kPThreadsMax = 256;                // threads per CTA (filter_blocked's pass width)
constexpr uint32_t kPVisLog2 = 11;
constexpr uint32_t kPVis = 1u << kPVisLog2;          // shared visited-set entries
constexpr uint32_t kPVisMax = kPVis * 3 / 4;         // distinct slots before the set moves to global
constexpr uint32_t kPNone = 0xFFFFFFFFu;

struct Layout {
    size_t terms, ta, tb, vkey, vpos, total;
};

__host__ __device__ inline Layout layout(uint32_t PW, uint32_t W2ab, bool hash) {
    Layout l{};
    size_t o = 0;
    l.terms = o;
    o += ((size_t)PW * 4 + 15) & ~size_t(15);
    l.ta = o;
    o += (size_t)W2ab * 4;
    l.tb = o;
    o += (size_t)W2ab * 4;
    l.vkey = o;
    o += hash ? (size_t)kPVis * 4 : 0;
    l.vpos = o;
    o += hash ? (size_t)kPVis * 4 : 0;
    l.total = o;
    return l;
}

// global visited table per query: 2^ts_log2 keys then 2^ts_log2 positions; it holds every
// distinct non-empty slot seen before the budget is reached (<= budget) plus one pass
__host__ __device__ inline uint32_t ts_log2_for(uint32_t budget) {
    uint32_t lg = 6;
    while ((1ull << lg) < ((uint64_t)budget + kPassMax + 32) * 3 / 2) ++lg;
    return lg;
}

// insert-or-find `key` (slot + 1) and lower its entry's position to `pos`; kPNone when the
// shared set is full (the pass then moves the set to global memory)
__device__ __forceinline__ uint32_t vis_shared(uint32_t* vkey, uint32_t* vpos, uint32_t key, uint32_t pos,
                                               uint32_t* nvis, volatile uint32_t* over) {
    uint32_t h = (key * 0x9E3779B1u) >> (32 - kPVisLog2);
    for (;;) {
        const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(vkey + h);
        if (cur == key) break;
        if (cur == 0u) {
            if (*over) return kPNone;
            const uint32_t prev = atomicCAS(vkey + h, 0u, key);
            if (prev == 0u) {
                if (atomicAdd(nvis, 1u) + 1u >= kPVisMax) *over = 1u;
                break;
            }
            if (prev == key) break;
        }
        h = (h + 1) & (kPVis - 1);
    }
    if (*reinterpret_cast<volatile uint32_t*>(vpos + h) > pos) atomicMin(vpos + h, pos);  // only ever lowers
    return h;
}

__device__ __forceinline__ uint32_t vis_global(uint32_t* gkey, uint32_t* gpos, uint32_t key, uint32_t pos,
                                               uint32_t ts_log2) {
    const uint32_t mask = (1u << ts_log2) - 1u;
    uint32_t h = (key * 0x9E3779B1u) >> (32 - ts_log2);
    for (;;) {
        const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(gkey + h);
        if (cur == key) break;
        if (cur == 0u) {
            const uint32_t prev = atomicCAS(gkey + h, 0u, key);
            if (prev == 0u || prev == key) break;
        }
        h = (h + 1) & mask;
    }
    if (*reinterpret_cast<volatile uint32_t*>(gpos + h) > pos) atomicMin(gpos + h, pos);
    return h;
}

// One filter pass in the blocked arrangement: thread t tests stream positions base + t·NIT + i
// (i < NIT), consecutive in stream order, so a thread's merge / pair-stream entries are one
// contiguous run (16-byte loads on the fast path). Returns the non-empty bits.
template <int P, int NIT>
__device__ __forceinline__ uint32_t filter_blocked(const DevParams& p, uint32_t base, uint32_t total, uint32_t tid,
                                                   uint32_t ta, uint32_t tb, uint32_t W, uint32_t H,
                                                   const uint32_t* terms, const uint32_t* tA, const uint32_t* tB,
                                                   uint32_t W2ab, uint32_t* slot) {
    const uint32_t W2 = (uint32_t)p.W2;
    const uint32_t mcount = (uint32_t)p.merge_count;
    const uint32_t s0 = base + tid * NIT;
    const uint32_t end = base + NIT * kPThreadsMax;
    const bool fast = end <= total &&
                      (P != 4 || (end <= mcount && p.merge16 && (W2ab == W2 || end <= p.merge_fold_end) &&
                                  H < 0x80000000u)) &&
                      (P != 2 || H < 0x80000000u);
    uint32_t word[NIT];
    if (fast) {
        uint32_t e[NIT];
        if constexpr (P == 4 || P == 2) {
            const uint32_t* src = P == 4 ? p.merge16 + s0 : p.pair_streams + (size_t)ta * W2 + s0;
            if (NIT % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
                for (int v = 0; v < NIT / 4; ++v) {
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(src) + v);
                    e[4 * v] = x.x;
                    e[4 * v + 1] = x.y;
                    e[4 * v + 2] = x.z;
                    e[4 * v + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int it = 0; it < NIT; ++it) e[it] = __ldg(src + it);
            }
#pragma unroll
            for (int it = 0; it < NIT; ++it)
                slot[it] = P == 4 ? add_mod_fast(tA[e[it] & 0xFFFFu], tB[e[it] >> 16], H)
                                  : add_mod_fast(terms[e[it] & 0xFFFFu], terms[W + (e[it] >> 16)], H);
        } else {
#pragma unroll
            for (int it = 0; it < NIT; ++it) slot[it] = terms[s0 + it];
        }
        probe_bitmap<NIT>(p, slot, word);
        uint32_t hit = 0;
#pragma unroll
        for (int it = 0; it < NIT; ++it) hit |= ((word[it] >> (slot[it] & 31)) & 1u) << it;
        return hit;
    }
    uint2 ent[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const uint32_t s = s0 + it;
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
    uint32_t hit = 0;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const uint32_t s = s0 + it;
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
    for (int it = 0; it < NIT; ++it) hit |= (uint32_t)(s0 + it < total && ((word[it] >> (slot[it] & 31)) & 1u)) << it;
    return hit;
}

}  // namespace bsp

// NT threads per CTA: 256, four CTAs per SM. (512-thread CTAs, passes twice as long at two CTAs
// per SM, measured slower on every workload: GIST1M 77 -> 82 us, SIFT1M 63 -> 133 us, SIFT1B
// 332 -> 737 us per batch -- most queries need one or two passes, so the longer pass is wasted.)
template <int P, bool HASH, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
    binsel_par_kernel(DevParams p, const uint32_t* __restrict__ l2c_in, const float* __restrict__ l2d_in,
                      uint8_t* __restrict__ slope_out, uint2* __restrict__ ranges, uint32_t* __restrict__ nranges,
                      uint32_t* __restrict__ ncand, uint32_t* __restrict__ ntuples,
                      pqtg_query_stats* __restrict__ stats, uint32_t ts_log2, uint32_t* __restrict__ ghash,
                      uint32_t W2ab) {
    using namespace bsp;
    constexpr int kPThreads = NT, kPWarps = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t q = blockIdx.x;
    if (p.chain) {  // the traversal's lists (a PDL dependent in a chained chunk)
        griddep_wait();
        griddep_launch();
    }
    qt_begin(p, q, 1);
    const uint32_t W = p.W, PW = P * W;
    const uint32_t H = (uint32_t)p.H;
    const Layout lay = layout(PW, W2ab, HASH);
    uint32_t* terms = reinterpret_cast<uint32_t*>(smem + lay.terms);
    uint32_t* tA = reinterpret_cast<uint32_t*>(smem + lay.ta);
    uint32_t* tB = reinterpret_cast<uint32_t*>(smem + lay.tb);
    uint32_t* vkey = reinterpret_cast<uint32_t*>(smem + lay.vkey);
    uint32_t* vpos = reinterpret_cast<uint32_t*>(smem + lay.vpos);
    __shared__ uint32_t s_slope[2];
    __shared__ uint32_t s_nvis, s_over, s_emit, s_maxord;

    // ---- prologue: slot terms (flat_part_code · (k1k2)^p) mod H (pqtree.cpp:12-25), the slope
    // picks (binorder.cpp:52-65) and, for P = 4, the pair streams folded into per-rank terms
    for (uint32_t idx = tid; idx < PW; idx += kPThreads) {
        const uint32_t code = l2c_in[q * PW + idx];
        const uint64_t flat = (uint64_t)(code >> 16) * p.k2 + (code & 0xFFFFu);
        terms[idx] = (uint32_t)((flat * p.mult[idx / W]) % p.H);
    }
    if (HASH)
        for (uint32_t i = tid; i < kPVis; i += kPThreads) {
            vkey[i] = 0u;
            vpos[i] = 0xFFFFFFFFu;
        }
    if (tid == 0) {
        s_nvis = 0;
        s_over = 0;
        s_emit = 0;
        s_maxord = 0;
    }
    if ((tid & 31) == 0 && tid < 64) {
        const uint32_t pr = tid >> 5, t = query_slope(p, l2d_in + q * PW, pr);
        s_slope[pr] = t;
        slope_out[q * 2 + pr] = (uint8_t)t;
    }
    __syncthreads();
    const uint32_t ta = s_slope[0], tb = s_slope[1];
    if (P == 4 && W2ab) {
        for (uint32_t u = tid; u < W2ab; u += kPThreads) {
            const uint32_t ea = __ldg(p.pair_streams + (size_t)ta * p.W2 + u);
            const uint32_t eb = __ldg(p.pair_streams + (size_t)tb * p.W2 + u);
            tA[u] = add_mod(terms[ea & 0xFFFFu], terms[W + (ea >> 16)], H);
            tB[u] = add_mod(terms[2 * W + (eb & 0xFFFFu)], terms[3 * W + (eb >> 16)], H);
        }
        __syncthreads();
    }

    const uint32_t budget = p.budget;
    const uint32_t total32 = (uint32_t)p.total_tuples;  // capped below 2^32 at index build
    uint2* qranges = ranges + q * (uint64_t)budget;
    uint32_t* gkey = HASH ? ghash + (q << (ts_log2 + 1)) : nullptr;
    uint32_t* gpos = HASH ? gkey + (1u << ts_log2) : nullptr;
    uint32_t C = 0, R = 0, base = 0;
    bool done = budget == 0, spilled = false;
    // P = 4 streams run to thousands of tuples: full passes from the start (a first
    // pass of 1024 measured slower even at SIFT1B, whose queries need ~930 tuples: 333 -> 354 us,
    // the pass is latency-bound and the queries past 1024 pay a second one)
    uint32_t nit = P == 4 ? kPItems : 1;
    __shared__ uint32_t s_wtc[2][kPWarps], s_wtf[2][kPWarps];  // per-warp totals (bin sizes, first flags)
    for (uint32_t pass = 0; !done && base < total32; ++pass) {
        const uint32_t pb = pass & 1u;
        // blocked arrangement: thread t owns stream positions base + t·nit .. + nit − 1, so its
        // items are consecutive in stream order and one block scan orders the whole pass
        uint32_t slot[kPItems];
        const uint32_t hit = nit == 1
                                 ? filter_blocked<P, 1>(p, base, total32, tid, ta, tb, W, H, terms, tA, tB, W2ab, slot)
                                 : filter_blocked<P, kPItems>(p, base, total32, tid, ta, tb, W, H, terms, tA, tB, W2ab,
                                                              slot);
        uint32_t first = 0;  // bit i: position base + tid·nit + i is its slot's first occurrence
        if constexpr (HASH) {
            uint32_t hidx[kPItems];
#pragma unroll
            for (int it = 0; it < kPItems; ++it) {
                hidx[it] = kPNone;
                if ((hit >> it) & 1u)
                    hidx[it] = spilled ? vis_global(gkey, gpos, slot[it] + 1u, base + tid * nit + it, ts_log2)
                                       : vis_shared(vkey, vpos, slot[it] + 1u, base + tid * nit + it, &s_nvis, &s_over);
            }
            // a pass without a single non-empty position (most of a sparse stream) ends here
            if (!__syncthreads_or(hit != 0)) {
                base += nit * kPThreads;
                nit = kPItems;
                continue;
            }
            if (!spilled && s_over) {
                // the shared set is 3/4 full: move it to this query's global table and redo
                // this pass's positions there (insert + atomicMin commute, so repeats are harmless)
                const uint32_t TS = 1u << ts_log2;
                for (uint32_t x = tid; x < TS; x += kPThreads) {
                    gkey[x] = 0u;
                    gpos[x] = 0xFFFFFFFFu;
                }
                __syncthreads();
                for (uint32_t x = tid; x < kPVis; x += kPThreads)
                    if (vkey[x]) vis_global(gkey, gpos, vkey[x], vpos[x], ts_log2);
#pragma unroll
                for (int it = 0; it < kPItems; ++it)
                    if ((hit >> it) & 1u)
                        hidx[it] = vis_global(gkey, gpos, slot[it] + 1u, base + tid * nit + it, ts_log2);
                __syncthreads();
                spilled = true;
            }
            const uint32_t* vp = spilled ? gpos : vpos;
#pragma unroll
            for (int it = 0; it < kPItems; ++it)
                if (hidx[it] != kPNone && vp[hidx[it]] == base + tid * nit + it) first |= 1u << it;
        } else {
            if (!__syncthreads_or(hit != 0)) {
                base += nit * kPThreads;
                nit = kPItems;
                continue;
            }
            first = hit;
        }
        // extents of the first occurrences, all loads in flight together
        uint32_t st[kPItems], cn[kPItems];
#pragma unroll
        for (int it = 0; it < kPItems; ++it) {
            st[it] = 0;
            cn[it] = 0;
            if ((first >> it) & 1u) {
                st[it] = __ldg(p.offsets + slot[it]);
                cn[it] = __ldg(p.offsets + slot[it] + 1);
            }
        }
        uint32_t tc = 0;
#pragma unroll
        for (int it = 0; it < kPItems; ++it) {
            cn[it] -= st[it];
            tc += cn[it];  // a pass's bins hold < 2^32 ids
        }
        const uint32_t tf = __popc(first);
        // one block scan of (bin sizes, first flags) over threads = stream order
        uint32_t ic = tc, iff = tf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, ic, o), b = __shfl_up_sync(0xffffffffu, iff, o);
            if (lane >= (uint32_t)o) {
                ic += a;
                iff += b;
            }
        }
        if (lane == 31) {
            s_wtc[pb][warp] = ic;
            s_wtf[pb][warp] = iff;
        }
        __syncthreads();
        uint32_t wc = 0, wf = 0, ctot = 0, ftot = 0;
#pragma unroll
        for (int w = 0; w < kPWarps; ++w) {
            const uint32_t a = s_wtc[pb][w], b = s_wtf[pb][w];
            if ((uint32_t)w < warp) {
                wc += a;
                wf += b;
            }
            ctot += a;
            ftot += b;
        }
        done = (uint64_t)C + ctot >= budget;
        uint64_t before = (uint64_t)C + wc + (ic - tc);
        uint32_t rank = R + wf + (iff - tf), emitted = 0, maxo = 0;
#pragma unroll
        for (int it = 0; it < kPItems; ++it) {
            if ((first >> it) & 1u) {
                if (before < budget) {
                    qranges[rank] = make_uint2(st[it], (uint32_t)before);
                    ++emitted;
                    maxo = base + tid * nit + it + 1u;
                }
                before += cn[it];
                ++rank;
            }
        }
        if (done) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                emitted += __shfl_xor_sync(0xffffffffu, emitted, o);
                maxo = max(maxo, __shfl_xor_sync(0xffffffffu, maxo, o));
            }
            if (lane == 0 && emitted) {
                atomicAdd(&s_emit, emitted);
                atomicMax(&s_maxord, maxo);
            }
        } else {
            C += ctot;
            R += ftot;
        }
        base += nit * kPThreads;
        nit = kPItems;
    }
    __syncthreads();
    if (tid == 0) {
        if (done && budget > 0) {
            R += s_emit;
            C = budget;
        }
        nranges[q] = R;
        ncand[q] = C;
        ntuples[q] = done && budget > 0 ? s_maxord : min(base, total32);
        if (stats) {
            stats[q].bins_visited = R;
            stats[q].candidates = C;
            stats[q].exact_evals = 0;
        }
    }
    qt_end(p, q, 1);
}

namespace {

template <int P, bool HASH, int NT>
void configure_par_nt() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, binsel_par_kernel<P, HASH, NT>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(binsel_par_kernel<P, HASH, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes));
}

template <int P, bool HASH>
void configure_par_one() {
    configure_par_nt<P, HASH, 256>();
}

}  // namespace

uint64_t binsel_par_hash_stride(const DevParams& p) {
    return 2ull << bsp::ts_log2_for(p.budget);
}

void configure_binsel_par() {
    configure_par_one<1, false>();
    configure_par_one<2, false>();
    configure_par_one<2, true>();
    configure_par_one<4, false>();
    configure_par_one<4, true>();
}

void launch_binsel_par(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats, cudaStream_t s) {
    const BsConfig c = bs_config(p);
    const uint32_t lg = bsp::ts_log2_for(p.budget);
    const size_t smem = bsp::layout(p.P * p.W, c.W2ab, c.use_hash).total;
#define PQTG_BP(PP, HH)                                                                                      \
    launch_kernel(p.chain, binsel_par_kernel<PP, HH, 256>, dim3((unsigned)nq), dim3(256), smem, s, p, ws.l2_code, ws.l2_dist, ws.slope, ws.ranges, \
                                                                  ws.nranges, ws.ncand, ws.ntuples, stats, lg,   \
                                                                  ws.hash, c.W2ab)
    if (p.P == 1) {
        PQTG_BP(1, false);
    } else if (p.P == 2) {
        if (c.use_hash) PQTG_BP(2, true); else PQTG_BP(2, false);
    } else {
        if (c.use_hash) PQTG_BP(4, true); else PQTG_BP(4, false);
    }
#undef PQTG_BP
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
