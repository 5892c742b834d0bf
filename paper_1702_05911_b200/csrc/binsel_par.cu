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
    const uint32_t W = p.W, PW = P * W;
    const uint32_t H = (uint32_t)p.H;
    const Layout lay = layout(PW, W2ab, HASH);
    uint32_t* terms = reinterpret_cast<uint32_t*>(smem + lay.terms);
    uint32_t* tA = reinterpret_cast<uint32_t*>(smem + lay.ta);
    uint32_t* tB = reinterpret_cast<uint32_t*>(smem + lay.tb);
    uint32_t* vkey = reinterpret_cast<uint32_t*>(smem + lay.vkey);
    uint32_t* vpos = reinterpret_cast<uint32_t*>(smem + lay.vpos);
    __shared__ uint32_t s_slope[2];
    __shared__ uint32_t s_wc[2][kPItems * kPWarps];                   // hits per (item, warp) (filter)
    __shared__ uint32_t s_cnt[2][kPItems * kPWarps], s_fst[2][kPItems * kPWarps];  // scan partials
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
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t C = 0, R = 0, base = 0;
    bool done = budget == 0, spilled = false;
    // P = 4 streams run to thousands of tuples: full passes from the start (a first
    // pass of 1024 measured slower even at SIFT1B, whose queries need ~930 tuples: 333 -> 354 us,
    // the pass is latency-bound and the queries past 1024 pay a second one)
    uint32_t nit = P == 4 ? kPItems : 1;
    for (uint32_t pass = 0; !done && base < total32; ++pass) {
        const uint32_t pb = pass & 1u;
        uint32_t slot[kPItems], ball[kPItems];
        if (nit == 1)
            filter<P, 1, kPThreads>(p, base, total32, tid, lane, warp, ta, tb, W, H, terms, tA, tB, W2ab, slot, ball,
                                   s_wc[pb]);
        else
            filter<P, kPItems, kPThreads>(p, base, total32, tid, lane, warp, ta, tb, W, H, terms, tA, tB, W2ab, slot,
                                        ball, s_wc[pb]);
        uint32_t first = 0;  // bit it: position base + it·256 + tid is its slot's first occurrence
        if constexpr (HASH) {
            uint32_t hidx[kPItems];
#pragma unroll
            for (int it = 0; it < kPItems; ++it) {
                hidx[it] = kPNone;
                if ((ball[it] >> lane) & 1u) {
                    const uint32_t pos = base + it * kPThreads + tid;
                    hidx[it] = spilled ? vis_global(gkey, gpos, slot[it] + 1u, pos, ts_log2)
                                       : vis_shared(vkey, vpos, slot[it] + 1u, pos, &s_nvis, &s_over);
                }
            }
            __syncthreads();
            // a pass without a single non-empty position (most of a sparse stream) ends here
            uint32_t hits = 0;
            for (uint32_t e = lane; e < nit * kPWarps; e += 32) hits += s_wc[pb][e];
            if (__any_sync(0xffffffffu, hits != 0) == 0) {
                base += nit * kPThreads;
                nit = kPItems;
                continue;
            }
            if (!spilled && s_over) {
                // the shared set is 3/4 full: move it to this query's global table and redo
                // this pass's positions there (insert + atomicMin commute, so repeats are harmless)
                const uint32_t TS = 1u << ts_log2;
                for (uint32_t i = tid; i < TS; i += kPThreads) {
                    gkey[i] = 0u;
                    gpos[i] = 0xFFFFFFFFu;
                }
                __syncthreads();
                for (uint32_t i = tid; i < kPVis; i += kPThreads)
                    if (vkey[i]) vis_global(gkey, gpos, vkey[i], vpos[i], ts_log2);
#pragma unroll
                for (int it = 0; it < kPItems; ++it)
                    if ((ball[it] >> lane) & 1u)
                        hidx[it] = vis_global(gkey, gpos, slot[it] + 1u, base + it * kPThreads + tid, ts_log2);
                __syncthreads();
                spilled = true;
            }
            const uint32_t* vp = spilled ? gpos : vpos;
#pragma unroll
            for (int it = 0; it < kPItems; ++it)
                if (hidx[it] != kPNone && vp[hidx[it]] == base + it * kPThreads + tid) first |= 1u << it;
        } else {
#pragma unroll
            for (int it = 0; it < kPItems; ++it) first |= ((ball[it] >> lane) & 1u) << it;
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
        // warp-level inclusive scans of bin sizes per item; the (item, warp) totals in stream order
        uint32_t inc[kPItems];
#pragma unroll
        for (int it = 0; it < kPItems; ++it) {
            cn[it] -= st[it];
            if (it < (int)nit) {
                const uint32_t fb = __ballot_sync(0xffffffffu, (first >> it) & 1u);
                uint32_t x = 0;
                if (fb) {  // warp-uniform: most (item, warp) groups hold no first occurrence
                    x = cn[it];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= (uint32_t)o) x += t;
                    }
                }
                inc[it] = x;
                if (lane == 31) {
                    s_cnt[pb][it * kPWarps + warp] = x;
                    s_fst[pb][it * kPWarps + warp] = __popc(fb);
                }
            }
        }
        __syncthreads();
        // every warp scans the <= kPItems·kPWarps (item, warp) totals itself: entry r·32 + lane
        // of row r, rows in stream order; xc / xf = exclusive prefixes over all rows
        constexpr int kRows = kPItems * kPWarps / 32;
        const uint32_t ne = nit * kPWarps;
        uint32_t xcr[kRows], xfr[kRows];
        uint32_t ccarry = 0, fcarry = 0;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const uint32_t e = r * 32 + lane;
            const uint32_t cv = e < ne ? s_cnt[pb][e] : 0u, fv = e < ne ? s_fst[pb][e] : 0u;
            uint32_t ic = cv, iff = fv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t a = __shfl_up_sync(0xffffffffu, ic, o), b = __shfl_up_sync(0xffffffffu, iff, o);
                if (lane >= (uint32_t)o) {
                    ic += a;
                    iff += b;
                }
            }
            xcr[r] = ccarry + ic - cv;
            xfr[r] = fcarry + iff - fv;
            ccarry += __shfl_sync(0xffffffffu, ic, 31);  // bins of one pass hold < 2^32 ids
            fcarry += __shfl_sync(0xffffffffu, iff, 31);
        }
        const uint64_t ctot = ccarry;
        const uint32_t ftot = fcarry;
        done = (uint64_t)C + ctot >= budget;
#pragma unroll
        for (int it = 0; it < kPItems; ++it) {
            const bool fst = (first >> it) & 1u;
            const uint32_t fb = __ballot_sync(0xffffffffu, fst);
            if (it < (int)nit && fb) {
                const uint32_t e = it * kPWarps + warp, src = e & 31u, row = e >> 5;  // warp-uniform
                uint32_t sc = 0, sf = 0;
#pragma unroll
                for (int r = 0; r < kRows; ++r)
                    if ((uint32_t)r == row) {
                        sc = xcr[r];
                        sf = xfr[r];
                    }
                const uint64_t ec = __shfl_sync(0xffffffffu, sc, src);
                const uint32_t ef = __shfl_sync(0xffffffffu, sf, src);
                const uint64_t before = (uint64_t)C + ec + (inc[it] - cn[it]);
                const bool emit = fst && before < budget;
                if (emit) qranges[R + ef + __popc(fb & lt)] = make_uint2(st[it], (uint32_t)before);
                if (done) {
                    const uint32_t eb = __ballot_sync(0xffffffffu, emit);
                    const uint32_t mo = __reduce_max_sync(0xffffffffu, emit ? base + it * kPThreads + tid + 1u : 0u);
                    if (lane == 0 && eb) {
                        atomicAdd(&s_emit, __popc(eb));
                        atomicMax(&s_maxord, mo);
                    }
                }
            }
        }
        if (!done) {
            C += (uint32_t)ctot;
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
    binsel_par_kernel<PP, HH, 256><<<(unsigned)nq, 256, smem, s>>>(p, ws.l2_code, ws.l2_dist, ws.slope, ws.ranges, \
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
