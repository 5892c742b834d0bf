// kernels.cu — sm_100a kernels of the PQT online query path.
//
//   K1 traverse_kernel  (north-star kernels 1+2)  pqtree.cpp:74-120 + binorder.cpp:52-65
//   K3 binsel_kernel    (north-star kernels 3+4)  binorder.cpp:69-283 + search.cpp:139-217
//   K5 rerank_kernel    (north-star kernels 5+6)  linequant.cpp:169-182 + search.cpp:221-257
//   merge_topk_kernel   per-shard top-k merge by (dist, id)  (search.cpp:39-41 order)
//
// Exactness contract: every fp32 op is an explicitly rounded
// __fadd_rn/__fsub_rn/__fmul_rn (never contracted to FMA), reductions run in the reference's
// sequential order, and every sort reproduces the reference's total order. Parallelism is
// across (query, centroid, candidate), never inside one sum.
#include <cub/block/block_radix_sort.cuh>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;


// =====================================================================================
// K1 — traversal: exact fine-part LUT, level-1 sort, level-2 distances of the w best
// parents, level-2 sort, slope pick. One CTA per query.
// =====================================================================================
template <int K1T, int K2T>  // compile-time k1 / k2 (0 = runtime): strided loads become immediates
__global__ void __launch_bounds__(kThreads) traverse_kernel(DevParams p, const float* __restrict__ Q,
                                                            float* __restrict__ fine_out,
                                                            float* __restrict__ l2d_out,
                                                            uint32_t* __restrict__ l2c_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t D = p.D, L = p.L, P = p.P, W = p.W, m = p.m, fd = p.fd;
    const uint32_t k1 = K1T ? (uint32_t)K1T : p.k1, k2 = K2T ? (uint32_t)K2T : p.k2;
    float* y = reinterpret_cast<float*>(smem);
    float* fine = y + D;
    float* l1d = fine + L * k1;
    uint32_t* l1o = reinterpret_cast<uint32_t*>(l1d + P * k1);
    float* l2d = reinterpret_cast<float*>(l1o + P * k1);
    uint32_t* l2c = reinterpret_cast<uint32_t*>(l2d + P * W);
    const uint64_t q = blockIdx.x;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    const int tid = threadIdx.x;

    for (uint32_t i = tid; i < D; i += blockDim.x) y[i] = Q[q * D + i];
    __syncthreads();

    // fine_dists[f][i] = l2_sq(y_f, slice(f, i), fd) sequentially (pqtree.cpp:90-93)
    for (uint32_t idx = tid; idx < L * k1; idx += blockDim.x) {
        const uint32_t f = idx / k1, i = idx - f * k1;
        const float* c = p.fine_t + (size_t)f * fd * k1 + i;
        const float* yf = y + f * fd;
        float acc = 0.0f;
        uint32_t t = 0;
        for (; t + 8 <= fd; t += 8, c += 8 * k1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = sq_step(acc, yf[t + u], __ldg(c + u * k1));
        }
        for (; t < fd; ++t, c += k1) acc = sq_step(acc, yf[t], __ldg(c));
        fine[idx] = acc;
        fine_out[q * L * k1 + idx] = acc;
    }
    __syncthreads();

    // level-1 totals: fp32 sum of the part's fine partials in f order (pqtree.cpp:88-96)
    for (uint32_t idx = tid; idx < P * k1; idx += blockDim.x) {
        const uint32_t pp = idx / k1, i = idx - pp * k1;
        float tot = 0.0f;
        for (uint32_t f = pp * p.per_part; f < (pp + 1) * p.per_part; ++f) tot = __fadd_rn(tot, fine[f * k1 + i]);
        l1d[idx] = tot;
    }
    __syncthreads();

    // sort each part's k1 entries by (dist, id) (pqtree.cpp:98-100): rank = #smaller keys
    for (uint32_t idx = tid; idx < P * k1; idx += blockDim.x) {
        const uint32_t pp = idx / k1, i = idx - pp * k1;
        const float d = l1d[idx];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[pp * k1 + j];
            rank += (dj < d) || (dj == d && j < i);
        }
        l1o[pp * k1 + rank] = i;
    }
    __syncthreads();

    // level-2: k2 children of each of the w best parents, l2_sq over m (pqtree.cpp:102-111)
    const uint32_t per = p.w * k2;
    for (uint32_t idx = tid; idx < P * per; idx += blockDim.x) {
        const uint32_t pp = idx / per, rem = idx - pp * per, r = rem / k2, c = rem - r * k2;
        const uint32_t parent = l1o[pp * k1 + r];
        const float* yp = y + pp * m;
        const float* cb = p.l2_t + ((size_t)(pp * k1 + parent) * m) * k2 + c;
        float acc = 0.0f;
        uint32_t t = 0;
        for (; t + 16 <= m; t += 16, cb += 16 * k2) {
            float cv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) cv[u] = __ldg(cb + u * k2);
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = sq_step(acc, yp[t + u], cv[u]);
        }
        for (; t < m; ++t, cb += k2) acc = sq_step(acc, yp[t], __ldg(cb));
        l2d[idx] = acc;
        l2c[idx] = (parent << 16) | c;
    }
    __syncthreads();

    // sort each part's W entries by (dist, parent, child) (pqtree.cpp:112-117)
    for (uint32_t idx = tid; idx < P * W; idx += blockDim.x) {
        const uint32_t pp = idx / W;
        const float d = l2d[idx];
        const uint32_t code = l2c[idx];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < W; ++j) {
            const float dj = l2d[pp * W + j];
            const uint32_t cj = l2c[pp * W + j];
            rank += (dj < d) || (dj == d && cj < code);
        }
        const size_t o = q * P * W + pp * W + rank;
        l2d_out[o] = d;
        l2c_out[o] = code;
    }
    qt_end(p, q, 0);
}

size_t traverse_smem(const DevParams& p) {
    return sizeof(float) * ((size_t)p.D + (size_t)p.L * p.k1 + 2ull * p.P * p.k1 + 2ull * p.P * p.W);
}

void launch_traverse(const DevParams& p, const float* queries, uint64_t nq, const WsSlice& ws,
                     cudaStream_t s) {
    if (kernel_variant() == 2 && ws.scr && screen_ok(p)) {
        // north-star kernel (1): tcgen05 screen of every child, exact residual check per part
        // (opt-in: at the benchmark shapes the all-exact per-part traversal is faster)
        launch_screen_gemm(p, queries, nq, ws.scr, s);
        launch_traverse_screen(p, queries, nq, ws.scr, ws, s);
        return;
    }
    if (kernel_variant() != 1 && traverse_part_ok(p)) {
        launch_traverse_part(p, queries, nq, ws, s);
        return;
    }
    // one thread per level-2 distance (P·w·k2 of them) keeps every thread busy in the long
    // sequential m-loop; 64..256 threads
    const uint32_t jobs = p.P * p.w * p.k2;
    const unsigned bs = jobs >= 256 ? 256u : (jobs <= 64 ? 64u : (unsigned)((jobs + 31) / 32 * 32));
#define PQTG_TRAV(A, B)                                                                       \
    traverse_kernel<A, B><<<(unsigned)nq, bs, traverse_smem(p), s>>>(p, queries, ws.fine, ws.l2_dist, \
                                                                     ws.l2_code)
    if (p.k1 == 16 && p.k2 == 8) PQTG_TRAV(16, 8);
    else if (p.k1 == 32 && p.k2 == 16) PQTG_TRAV(32, 16);
    else if (p.k1 == 16 && p.k2 == 16) PQTG_TRAV(16, 16);
    else PQTG_TRAV(0, 0);
#undef PQTG_TRAV
    PQTG_CUDA_CHECK(cudaGetLastError());
}

// =====================================================================================
// K3 — bin selection + gather: walk the heuristic rank-tuple stream in chunks, hash each
// tuple to its slot, drop empty slots with the bitmap, keep the first occurrence of every
// non-empty slot (shared-memory hash set keyed by slot, atomicMin of processing rank), and
// cut at the candidate budget with a block prefix sum. Emits one range per visited bin.
// =====================================================================================
namespace {

struct BinselSmem {
    uint32_t ts_mask;
    uint32_t ts_shift;
};

__device__ __forceinline__ uint32_t hash_slot(uint32_t slot, uint32_t shift) {
    return (slot * 0x9E3779B1u) >> shift;
}

// The slot of a rank tuple (pqtree.cpp:12-25): the positional code sum (u64 wrap) mod H, from
// the per-part terms (flat code · (k1k2)^p, reduced mod H when mod_fast).
__device__ __forceinline__ uint64_t slot_of_ranks(const DevParams& p, const uint32_t* r, const uint64_t* terms) {
    uint64_t code = 0;
    for (uint32_t q = 0; q < p.P; ++q) code += terms[q * p.W + r[q]];
    if (p.h_pow2) return code & (p.H - 1);
    if (p.mod_fast) {  // terms already reduced mod H, sum < P*H
        while (code >= p.H) code -= p.H;
        return code;
    }
    return code % p.H;
}

// ---- exact order (binorder.cpp:114-167): every tuple in ascending (fp64 sum of its list
// distances, tuple) order. A min-heap in shared memory on one thread; each tuple is pushed once,
// by its canonical parent (the tuple minus one at its last non-zero rank: its sum is not larger
// and it is lexicographically smaller, so it pops first), which emits the reference's sequence
// without its visited set. Tuples are packed big-endian, tuple_bits per rank, so u64 order is
// the lexicographic order.
struct ExactHeap {
    double* sum;
    uint64_t* tup;
    uint32_t cap;
};

__device__ __forceinline__ bool exact_less(const ExactHeap& h, uint32_t a, uint32_t b) {
    return h.sum[a] < h.sum[b] || (h.sum[a] == h.sum[b] && h.tup[a] < h.tup[b]);
}

__device__ __forceinline__ double exact_sum(const DevParams& p, uint64_t t, const float* dl) {
    const uint32_t B = p.tuple_bits, mask = (1u << B) - 1u;
    double s = 0.0;  // BinStream's sum_of: fp64, parts in order
    for (uint32_t q = 0; q < p.P; ++q) {
        const uint32_t r = (uint32_t)(t >> ((p.P - 1 - q) * B)) & mask;
        s = __dadd_rn(s, (double)dl[q * p.W + r]);
    }
    return s;
}

// push; false when the heap is full
__device__ __forceinline__ bool exact_push(ExactHeap& h, uint32_t& n, double sum, uint64_t t) {
    if (n >= h.cap) return false;
    uint32_t i = n++;
    h.sum[i] = sum;
    h.tup[i] = t;
    while (i > 0) {
        const uint32_t par = (i - 1) >> 1;
        if (!exact_less(h, i, par)) break;
        const double ds = h.sum[i];
        const uint64_t dt = h.tup[i];
        h.sum[i] = h.sum[par];
        h.tup[i] = h.tup[par];
        h.sum[par] = ds;
        h.tup[par] = dt;
        i = par;
    }
    return true;
}

// the next `want` tuples of the exact order into out; returns how many (fewer at the end of the
// stream or, with *overflow set, when the heap is full)
__device__ uint32_t exact_fill(const DevParams& p, ExactHeap& h, uint32_t& n, const float* dl, uint64_t* out,
                               uint32_t want, uint32_t* overflow) {
    const uint32_t B = p.tuple_bits, mask = (1u << B) - 1u, P = p.P;
    uint32_t got = 0;
    while (got < want && n > 0) {
        const uint64_t t = h.tup[0];
        out[got++] = t;
        // pop
        --n;
        h.sum[0] = h.sum[n];
        h.tup[0] = h.tup[n];
        for (uint32_t i = 0;;) {
            const uint32_t l = 2 * i + 1, r = l + 1;
            uint32_t m = i;
            if (l < n && exact_less(h, l, m)) m = l;
            if (r < n && exact_less(h, r, m)) m = r;
            if (m == i) break;
            const double ds = h.sum[i];
            const uint64_t dt = h.tup[i];
            h.sum[i] = h.sum[m];
            h.tup[i] = h.tup[m];
            h.sum[m] = ds;
            h.tup[m] = dt;
            i = m;
        }
        // children: +1 at every part from the last non-zero rank on
        uint32_t j = 0;
        for (uint32_t q = 0; q < P; ++q)
            if ((t >> ((P - 1 - q) * B)) & mask) j = q;
        for (uint32_t q = j; q < P; ++q) {
            const uint32_t sh = (P - 1 - q) * B;
            if (((t >> sh) & mask) + 1 < p.W) {
                const uint64_t c = t + (1ull << sh);
                if (!exact_push(h, n, exact_sum(p, c, dl), c)) {
                    *overflow = 1;
                    return got;
                }
            }
        }
    }
    return got;
}

__device__ __forceinline__ void exact_ranks(const DevParams& p, uint64_t t, uint32_t* r) {
    const uint32_t B = p.tuple_bits, mask = (1u << B) - 1u;
    for (uint32_t q = 0; q < p.P; ++q) r[q] = (uint32_t)(t >> ((p.P - 1 - q) * B)) & mask;
}

// Stream tuple at position s -> the slot it addresses (binorder.cpp:251-283, pqtree.cpp:12-25).
__device__ __forceinline__ uint64_t tuple_slot(const DevParams& p, uint64_t s, uint32_t ta, uint32_t tb,
                                               const uint64_t* terms) {
    uint32_t r0, r1 = 0, r2 = 0, r3 = 0;
    if (p.P == 1) {
        r0 = (uint32_t)s;
    } else if (p.P == 2) {
        const uint32_t e = __ldg(p.pair_streams + (size_t)ta * p.W2 + s);
        r0 = e & 0xFFFFu;
        r1 = e >> 16;
    } else {
        uint64_t u, v;
        if (s < p.merge_count) {
            const uint2 uv = __ldg(p.merge + s);
            u = uv.x;
            v = uv.y;
        } else {
            const uint64_t j = s - p.merge_count;
            u = p.merge_row0 + j / p.W2;
            v = j - (u - p.merge_row0) * p.W2;
        }
        const uint32_t ea = __ldg(p.pair_streams + (size_t)ta * p.W2 + u);
        const uint32_t eb = __ldg(p.pair_streams + (size_t)tb * p.W2 + v);
        r0 = ea & 0xFFFFu;
        r1 = ea >> 16;
        r2 = eb & 0xFFFFu;
        r3 = eb >> 16;
    }
    const uint32_t W = p.W;
    uint64_t code = terms[r0];
    if (p.P >= 2) code += terms[W + r1];
    if (p.P == 4) code += terms[2 * W + r2] + terms[3 * W + r3];
    if (p.h_pow2) return code & (p.H - 1);
    if (p.mod_fast) {  // terms already reduced mod H, sum < P*H
        while (code >= p.H) code -= p.H;
        return code;
    }
    return code % p.H;
}

}  // namespace

template <int ITEMS, bool RESORT, bool EXACT>
__global__ void __launch_bounds__(kThreads) binsel_kernel(DevParams p, const float* __restrict__ l2d_in,
                                                          const uint32_t* __restrict__ l2c_in,
                                                          uint8_t* __restrict__ slope_out,
                                                          uint2* __restrict__ ranges,
                                                          uint32_t* __restrict__ nranges,
                                                          uint32_t* __restrict__ ncand,
                                                          uint32_t* __restrict__ ntuples,
                                                          pqtg_query_stats* __restrict__ stats,
                                                          uint32_t ts_log2, uint32_t heap_cap,
                                                          uint32_t* __restrict__ err,
                                                          uint64_t* __restrict__ gscr, uint64_t gscr_stride) {
    using Sort = cub::BlockRadixSort<uint32_t, kThreads, ITEMS, uint32_t>;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t PW_ = p.P * p.W;
    const uint32_t TS = 1u << ts_log2;
    const uint32_t shift = 32 - ts_log2;
    const uint64_t q = blockIdx.x;
    // gscr (large budgets): this query's scratch in the workspace -- the visited set [TS] (u32
    // keys, u32 first positions) and, for resort batches longer than one chunk, two sort buffers
    // and the exact order's batch of tuples, [budget] u64 each
    uint64_t* gq = gscr ? gscr + q * gscr_stride : nullptr;
    uint64_t* terms = reinterpret_cast<uint64_t*>(smem);
    uint64_t* warp_sums = terms + PW_;
    float* dl = reinterpret_cast<float*>(warp_sums + 32);
    uint32_t* hkeys = gq ? reinterpret_cast<uint32_t*>(gq) : reinterpret_cast<uint32_t*>(dl + PW_);
    uint32_t* hvals = hkeys + TS;
    // EXACT: this chunk's tuples, then the heap (8-byte aligned after the u32 tables)
    unsigned char* after = reinterpret_cast<unsigned char*>(gq ? reinterpret_cast<uint32_t*>(dl + PW_) : hvals + TS);
    uint64_t* tbuf = reinterpret_cast<uint64_t*>(smem + (((size_t)(after - smem) + 7) & ~size_t(7)));
    ExactHeap heap{reinterpret_cast<double*>(tbuf + kThreads * ITEMS), nullptr, heap_cap};
    heap.tup = reinterpret_cast<uint64_t*>(heap.sum + heap_cap);
    __shared__ uint32_t s_emitted, s_maxord, s_got, s_overflow, s_heap_n;
    __shared__ typename Sort::TempStorage sort_tmp;

    if (p.chain) {  // the traversal's lists (a PDL dependent in a chained chunk)
        griddep_wait();
        griddep_launch();
    }
    qt_begin(p, q, 1);
    const int tid = threadIdx.x;

    for (uint32_t idx = tid; idx < PW_; idx += blockDim.x) {
        const uint32_t code = l2c_in[q * PW_ + idx];
        const uint32_t pp = idx / p.W;
        const uint64_t flat = (uint64_t)(code >> 16) * p.k2 + (code & 0xFFFFu);  // flat_part_code
        uint64_t t = flat * p.mult[pp];                                          // u64 wrap
        if (p.mod_fast) t %= p.H;
        terms[idx] = t;
        dl[idx] = l2d_in[q * PW_ + idx];
    }
    for (uint32_t i = tid; i < TS; i += blockDim.x) {
        hkeys[i] = kEmptyKey;
        hvals[i] = 0xFFFFFFFFu;
    }
    __shared__ uint32_t s_slope[2];
    if (tid == 0) {
        s_maxord = 0;
        s_overflow = 0;
        s_heap_n = 0;
    }
    if ((tid & 31) == 0 && tid < 64) {  // pick_slope_table (binorder.cpp:52-65), one pair per warp
        const uint32_t pr = tid >> 5, t = query_slope(p, l2d_in + q * PW_, pr);
        s_slope[pr] = t;
        slope_out[q * 2 + pr] = (uint8_t)t;
    }
    __syncthreads();
    const uint32_t ta = s_slope[0], tb = s_slope[1];

    const uint32_t budget = p.budget;
    uint64_t total = p.total_tuples;
    const uint32_t CH = kThreads * ITEMS;
    uint2* qranges = ranges + q * (uint64_t)budget;
    uint32_t C = 0, R = 0;
    uint64_t base = 0;
    if (EXACT && tid == 0) {  // the all-zero tuple starts the exact order
        uint32_t n0 = 0;
        exact_push(heap, n0, exact_sum(p, 0, dl), 0);
        s_heap_n = n0;
    }

    // a resort batch longer than one chunk sorts through the workspace (RESORT implies gq then)
    uint64_t* srt_a = gq ? gq + TS : nullptr;
    uint64_t* srt_b = srt_a ? srt_a + budget : nullptr;
    uint64_t* tup = tbuf;  // the exact order's tuples of this chunk / batch
    if (EXACT && RESORT && gq && budget > CH) tup = srt_b + budget;
    while (C < budget && base < total) {
        if constexpr (EXACT) {
            // this chunk's (or resort batch's) tuples, in order, from the heap
            const uint32_t want = RESORT ? (uint32_t)min((uint64_t)budget, total - base) : CH;
            __syncthreads();
            if (tid == 0) {
                uint32_t n = s_heap_n;
                s_got = exact_fill(p, heap, n, dl, tup, want, &s_overflow);
                s_heap_n = n;
            }
            __syncthreads();
            if (s_got < want) total = base + s_got;  // the stream (or the heap) ends in this chunk
            if (s_got == 0) break;
        }
        uint64_t spos[ITEMS];
        bool inb[ITEMS];
        uint64_t step;
        uint32_t nsub = 1;             // chunks of CH tuples this batch is processed in
        const uint64_t* srt = nullptr;  // a long resort batch in order: (key << 32 | batch index)
        uint64_t bs = 0;
        if (RESORT) {
            // one batch = the next `budget` tuples (search.cpp:153), stable-sorted by the
            // fp32 sum of their part distances (search.cpp:179-190)
            bs = min((uint64_t)budget, total - base);
            if (bs > CH) nsub = (uint32_t)((bs + CH - 1) / CH);
            for (uint32_t sc = 0; sc < nsub; ++sc) {
            uint32_t keys[ITEMS], vals[ITEMS];
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                const uint32_t o = sc * CH + tid * ITEMS + it;
                vals[it] = o;
                keys[it] = 0xFFFFFFFFu;
                if (o < bs) {
                    const uint64_t s = base + o;
                    // ranks of tuple s (recomputed; resort batches are budget-sized)
                    uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (EXACT) {
                        exact_ranks(p, tup[o], r);
                    } else if (p.P == 1) {
                        r[0] = (uint32_t)s;
                    } else if (p.P == 2) {
                        const uint32_t e = p.pair_streams[(size_t)ta * p.W2 + s];
                        r[0] = e & 0xFFFFu;
                        r[1] = e >> 16;
                    } else {
                        uint64_t u, v;
                        if (s < p.merge_count) {
                            u = p.merge[s].x;
                            v = p.merge[s].y;
                        } else {
                            const uint64_t j = s - p.merge_count;
                            u = p.merge_row0 + j / p.W2;
                            v = j - (u - p.merge_row0) * p.W2;
                        }
                        const uint32_t ea = p.pair_streams[(size_t)ta * p.W2 + u];
                        const uint32_t eb = p.pair_streams[(size_t)tb * p.W2 + v];
                        r[0] = ea & 0xFFFFu;
                        r[1] = ea >> 16;
                        r[2] = eb & 0xFFFFu;
                        r[3] = eb >> 16;
                    }
                    float agg = 0.0f;
                    for (uint32_t pp = 0; pp < p.P; ++pp) agg = __fadd_rn(agg, dl[pp * p.W + r[pp]]);
                    keys[it] = orderable(agg);
                }
            }
            Sort(sort_tmp).Sort(keys, vals);  // stable LSD radix sort, blocked arrangement
            __syncthreads();
            if (nsub == 1) {
#pragma unroll
                for (int it = 0; it < ITEMS; ++it) {
                    const uint32_t o = tid * ITEMS + it;
                    inb[it] = o < bs;
                    spos[it] = base + vals[it];
                }
            } else {  // the chunk's sorted run (its valid keys first: sentinels sort last, stably)
#pragma unroll
                for (int it = 0; it < ITEMS; ++it) {
                    const uint32_t o = sc * CH + tid * ITEMS + it;
                    if (o < bs) srt_a[o] = (uint64_t)keys[it] << 32 | vals[it];
                }
            }
            }
            if (nsub > 1) {
                // merge the sorted runs pairwise: (key, batch index) pairs are distinct, so an
                // element's place is its index in its run plus the count of smaller elements in
                // the partner run (the stable sort's order)
                __syncthreads();
                uint64_t* src = srt_a;
                uint64_t* dst = srt_b;
                for (uint64_t w = CH; w < bs; w *= 2) {
                    for (uint32_t e = tid; e < bs; e += kThreads) {
                        const uint64_t key = src[e];
                        const uint64_t r = e / w, lo = e - r * w, pb = (r ^ 1) * w;
                        uint64_t a = pb, b = pb < bs ? min(pb + w, bs) : pb;
                        while (a < b) {
                            const uint64_t m = (a + b) >> 1;
                            if (src[m] < key) a = m + 1;
                            else b = m;
                        }
                        dst[(r & ~1ull) * w + lo + (a - pb)] = key;
                    }
                    __syncthreads();
                    uint64_t* t = src;
                    src = dst;
                    dst = t;
                }
                srt = src;
            }
            step = bs;
        } else {
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                spos[it] = base + (uint64_t)(tid * ITEMS + it);
                inb[it] = spos[it] < total;
            }
            step = CH;
        }

        for (uint32_t sc = 0; sc < nsub && C < budget; ++sc) {
        const uint64_t obase = base + (uint64_t)sc * CH;  // processing-order position of the chunk
        if (srt) {
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                const uint64_t o = (uint64_t)sc * CH + tid * ITEMS + it;
                inb[it] = o < bs;
                spos[it] = base + (inb[it] ? (uint32_t)srt[o] : 0u);
            }
        }
        // slot, emptiness and first-occurrence bookkeeping
        uint32_t slot[ITEMS], hidx[ITEMS];
        bool ne[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            ne[it] = false;
            hidx[it] = 0;
            slot[it] = 0;
            if (inb[it]) {
                uint64_t sl;
                if constexpr (EXACT) {
                    uint32_t r[8];
                    exact_ranks(p, tup[spos[it] - base], r);
                    sl = slot_of_ranks(p, r, terms);
                } else {
                    sl = tuple_slot(p, spos[it], ta, tb, terms);
                }
                slot[it] = (uint32_t)sl;
                ne[it] = (__ldg(p.bitmap + (sl >> 5)) >> (sl & 31)) & 1u;
            }
            if (ne[it]) {
                // Empty slots need no dedup: a repeat of an empty slot is empty again.
                const uint32_t ord = (uint32_t)(obase + tid * ITEMS + it);
                uint32_t h = hash_slot(slot[it], shift);
                for (;;) {
                    const uint32_t prev = atomicCAS(hkeys + h, kEmptyKey, slot[it]);
                    if (prev == kEmptyKey || prev == slot[it]) {
                        atomicMin(hvals + h, ord);
                        break;
                    }
                    h = (h + 1) & (TS - 1);
                }
                hidx[it] = h;
            }
        }
        __syncthreads();

        uint32_t cnt[ITEMS], start[ITEMS];
        uint64_t local = 0;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            cnt[it] = 0;
            start[it] = 0;
            if (ne[it]) {
                const uint32_t ord = (uint32_t)(obase + tid * ITEMS + it);
                const uint32_t first = gq ? __ldcg(hvals + hidx[it]) : hvals[hidx[it]];  // global: its atomics live in L2
                if (first == ord) {  // first occurrence in processing order
                    start[it] = __ldg(p.offsets + slot[it]);
                    cnt[it] = __ldg(p.offsets + slot[it] + 1) - start[it];
                }
            }
            local += ((uint64_t)cnt[it] << 32) | (cnt[it] ? 1u : 0u);
        }
        if (tid == 0) s_emitted = 0;
        uint64_t tot;
        uint64_t excl = block_excl_scan(local, warp_sums, &tot);
        uint32_t emitted = 0, maxord = 0;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (cnt[it]) {
                const uint64_t before_c = (uint64_t)C + (excl >> 32);
                if (before_c < budget) {
                    const uint32_t r = R + (uint32_t)(excl & 0xFFFFFFFFu);
                    qranges[r] = make_uint2(start[it], (uint32_t)before_c);
                    ++emitted;
                    maxord = max(maxord, (uint32_t)(obase + tid * ITEMS + it));
                }
                excl += ((uint64_t)cnt[it] << 32) | 1u;
            }
        }
        if (emitted) {
            atomicAdd(&s_emitted, emitted);
            atomicMax(&s_maxord, maxord);
        }
        __syncthreads();
        R += s_emitted;
        const uint64_t newc = (uint64_t)C + (tot >> 32);
        C = newc < budget ? (uint32_t)newc : budget;
        __syncthreads();
        }
        base += step;
    }
    if (tid == 0) {
        nranges[q] = R;
        ncand[q] = C;
        // tuples the reference's gather loop consumes: up to the one that filled the budget,
        // or the whole stream (search.cpp:166-217)
        ntuples[q] = C >= budget && budget > 0 ? s_maxord + 1 : (uint32_t)min(base, total);
        if (EXACT && s_overflow) {  // the heap overflowed: reported by the host API
            ntuples[q] = 0xFFFFFFFFu;
            atomicOr(err, PQTG_WS_ERR_HEAP);
        }
        if (stats) {
            stats[q].bins_visited = R;
            stats[q].candidates = C;
            stats[q].exact_evals = 0;
        }
    }
    qt_end(p, q, 1);
}

namespace {
uint32_t ts_log2_for(const DevParams& p) {
    const uint64_t ch = p.resort ? 4096 : (uint64_t)kThreads * 4;
    const uint64_t need = ((uint64_t)p.budget + ch) * 3 / 2 + 64;
    uint32_t lg = 6;
    while ((1ull << lg) < need) ++lg;
    return lg;
}
}  // namespace

size_t binsel_smem(const DevParams& p, bool global_visited) {
    const uint64_t TS = global_visited ? 0 : 1ull << ts_log2_for(p);
    return (size_t)p.P * p.W * (8 + 4) + TS * 8 + 32 * 8;
}

// u64 words of workspace scratch per query for the generic bin selection (0: none): the visited
// set when it does not fit shared memory, plus the sort buffers of resort batches longer than
// one chunk (budget > 4096) -- see binsel_kernel
uint64_t binsel_scratch_stride(const DevParams& p) {
    if (binsel_fast_ok(p)) return 0;
    const bool big_resort = p.resort && p.budget > 16u * kThreads;
    if (!big_resort && binsel_smem(p, false) + 2048 <= (size_t)optin_bytes()) return 0;
    return (1ull << ts_log2_for(p)) + (big_resort ? 3ull * p.budget : 0ull);
}

void launch_binsel(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats,
                   cudaStream_t s) {
    if (kernel_variant() != 1 && binsel_fast_ok(p)) {
        // all-warp passes (binsel_par) unless the stream is the folded P = 4 one (W·W <= 4096,
        // e.g. GIST1M), whose sparse hits favour overlapping the filter with a walker warp
        // (measured); variants 3 / 4 force either design
        const int v = kernel_variant();
        const bool walker = v == 3 || (v != 4 && binsel_prefers_walker(p));
        if (walker) launch_binsel_fast(p, nq, ws, stats, s);
        else launch_binsel_par(p, nq, ws, stats, s);
        return;
    }
    const uint32_t lg = ts_log2_for(p);
    const uint64_t gstride = binsel_scratch_stride(p);
    if (gstride && !ws.bscr) throw Error{PQTG_ERR_ARG, "bin selection scratch missing from the workspace"};
    uint64_t* gscr = gstride ? ws.bscr : nullptr;
    const size_t sm = binsel_smem(p, gstride != 0);
    if (p.exact_order) {
        // the exact order's heap takes the rest of the opt-in shared memory (<= 64 Ki entries)
        const uint32_t ch = (p.resort ? 16u : 4u) * kThreads;
        const size_t fixed = ((sm + 7) & ~size_t(7)) + (size_t)ch * 8;
        int dev = 0, optin = 0;
        PQTG_CUDA_CHECK(cudaGetDevice(&dev));
        PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        cudaFuncAttributes a{};
        if (p.resort) PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, binsel_kernel<16, true, true>));
        else PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, binsel_kernel<4, false, true>));
        const size_t avail = (size_t)optin - a.sharedSizeBytes;
        if (avail < fixed + 64 * 16) throw Error{PQTG_ERR_UNSUPPORTED, "exact bin order: no shared memory for its heap"};
        const uint32_t cap = (uint32_t)std::min<size_t>((avail - fixed) / 16, 65536);
        const size_t smx = fixed + (size_t)cap * 16;
        if (p.resort)
            launch_kernel(p.chain, binsel_kernel<16, true, true>, dim3((unsigned)nq), dim3(kThreads), smx, s, 
                p, ws.l2_dist, ws.l2_code, ws.slope, ws.ranges, ws.nranges, ws.ncand, ws.ntuples, stats, lg, cap, ws.err, gscr, gstride);
        else
            launch_kernel(p.chain, binsel_kernel<4, false, true>, dim3((unsigned)nq), dim3(kThreads), smx, s, 
                p, ws.l2_dist, ws.l2_code, ws.slope, ws.ranges, ws.nranges, ws.ncand, ws.ntuples, stats, lg, cap, ws.err, gscr, gstride);
    } else if (p.resort) {
        launch_kernel(p.chain, binsel_kernel<16, true, false>, dim3((unsigned)nq), dim3(kThreads), sm, s, 
            p, ws.l2_dist, ws.l2_code, ws.slope, ws.ranges, ws.nranges, ws.ncand, ws.ntuples, stats, lg, 0, ws.err, gscr, gstride);
    } else {
        launch_kernel(p.chain, binsel_kernel<4, false, false>, dim3((unsigned)nq), dim3(kThreads), sm, s, 
            p, ws.l2_dist, ws.l2_code, ws.slope, ws.ranges, ws.nranges, ws.ncand, ws.ntuples, stats, lg, 0, ws.err, gscr, gstride);
    }
    PQTG_CUDA_CHECK(cudaGetLastError());
}

// =====================================================================================
// K5 — line-quantized re-rank + top-k. One CTA per query; per-query LUT (fine dists) and
// the pair tables in shared memory; one thread per candidate walks its code row; then an
// 8-bit radix select finds the k-th (dist, id) key and a bitonic sort orders the top k.
// =====================================================================================
namespace {

// part contribution (linequant.hpp:83-85 in linequant.cpp:171-181's order) for stored byte
// `b` (a pair id, or i << 4 | ((i + j) & 15) when the index re-encoded pairs); c2 rows are [f][npairs] or,
// for (i, j) codes, [f][256].
__device__ __forceinline__ void pair_terms(uint32_t b, uint32_t f, bool ij, const float* fine, const float* c2,
                                           const uint32_t* pairs, uint32_t k1, uint32_t npairs, float& b2,
                                           float& a2, float& cc, const uint8_t* __restrict__ jt,
                                           const float* __restrict__ c2v) {
    if (ij) {  // b = i << 4 | n: n = (i + j) & 15, or the per-part bank map's (jt: j of b)
        b2 = fine[f * k1 + (b >> 4)];
        a2 = fine[f * k1 + (jt ? (uint32_t)__ldg(jt + f * 256 + b) : (((b & 15u) - (b >> 4)) & 15u))];
        cc = c2[f * 256 + b];
    } else if (c2v) {  // code_j: b = i | j << 5 (index_prep.cpp, DIRECT shards)
        b2 = fine[f * k1 + (b & 31u)];
        a2 = fine[f * k1 + ((b >> 5) & 31u)];
        cc = __ldg(c2v + f * 1024 + (b & 0x3FFu));
    } else {
        const uint32_t pr = pairs[b];
        b2 = fine[f * k1 + (pr & 0xFFFFu)];
        a2 = fine[f * k1 + (pr >> 16)];
        cc = c2[f * npairs + b];
    }
}

template <int LT, int PW>
__device__ __forceinline__ float line_distance_row(const uint8_t* __restrict__ row, const float* fine,
                                                   const float* c2, const uint32_t* pairs, uint32_t L,
                                                   uint32_t k1, uint32_t npairs, bool ij, uint32_t pid_mask,
                                                   const uint8_t* __restrict__ jt, const float* __restrict__ c2v) {
    const float inv255 = __uint_as_float(0x3B808081u);  // 1.0f / 255.0f (linequant.cpp:175)
    float total = 0.0f;
    if constexpr (LT > 0) {
        constexpr int kBytes = LT * (1 + PW);
        constexpr int kVec = (kBytes + 15) / 16;
        uint4 v[kVec];
        const uint4* r4 = reinterpret_cast<const uint4*>(row);
#pragma unroll
        for (int i = 0; i < kVec; ++i) v[i] = __ldg(r4 + i);
        const uint32_t* wds = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
        for (int f = 0; f < LT; ++f) {
            uint32_t lq, pid;
            if constexpr (PW == 1) {
                const int bl = 2 * f, bp = 2 * f + 1;
                lq = (wds[bl >> 2] >> ((bl & 3) * 8)) & 0xFFu;
                pid = (wds[bp >> 2] >> ((bp & 3) * 8)) & 0xFFu;
            } else {
                lq = (wds[f >> 2] >> ((f & 3) * 8)) & 0xFFu;
                const int b0 = LT + 2 * f, b1 = b0 + 1;
                pid = ((wds[b0 >> 2] >> ((b0 & 3) * 8)) & 0xFFu) | (((wds[b1 >> 2] >> ((b1 & 3) * 8)) & 0xFFu) << 8);
                pid &= pid_mask;  // code_pi rows carry the first centroid in bits 9..13 (code_j: i | j << 5)
            }
            float b2, a2, cc;
            pair_terms(pid, f, ij, fine, c2, pairs, k1, npairs, b2, a2, cc, jt, c2v);
            const float lam = __fmul_rn((float)lq, inv255);
            const float part = __fadd_rn(__fadd_rn(b2, __fmul_rn(__fmul_rn(lam, lam), cc)),
                                         __fmul_rn(lam, __fsub_rn(__fsub_rn(a2, b2), cc)));
            total = __fadd_rn(total, part);
        }
    } else {
        for (uint32_t f = 0; f < L; ++f) {
            uint32_t lq, pid;
            if (PW == 1) {
                lq = __ldg(row + 2 * f);
                pid = __ldg(row + 2 * f + 1);
            } else {
                lq = __ldg(row + f);
                pid = ((uint32_t)__ldg(row + L + 2 * f) | ((uint32_t)__ldg(row + L + 2 * f + 1) << 8)) & pid_mask;
            }
            float b2, a2, cc;
            pair_terms(pid, f, ij, fine, c2, pairs, k1, npairs, b2, a2, cc, jt, c2v);
            const float lam = __fmul_rn((float)lq, inv255);
            const float part = __fadd_rn(__fadd_rn(b2, __fmul_rn(__fmul_rn(lam, lam), cc)),
                                         __fmul_rn(lam, __fsub_rn(__fsub_rn(a2, b2), cc)));
            total = __fadd_rn(total, part);
        }
    }
    return total;
}

uint32_t next_pow2(uint32_t x) {
    uint32_t r = 1;
    while (r < x) r <<= 1;
    return r;
}

}  // namespace

template <int LT, int PW>
__global__ void __launch_bounds__(kThreads) rerank_kernel(DevParams p, uint32_t k, uint32_t sel_cap,
                                                          const float* __restrict__ fine_in,
                                                          const uint2* __restrict__ ranges,
                                                          const uint32_t* __restrict__ nranges,
                                                          const uint32_t* __restrict__ ncand,
                                                          uint32_t* __restrict__ out_ids,
                                                          float* __restrict__ out_dists,
                                                          uint32_t* __restrict__ out_counts,
                                                          uint64_t* __restrict__ gkeys) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t L = p.L, k1 = p.k1, npairs = p.npairs, budget = p.budget;
    // keys: shared memory, or this query's row of the workspace buffer for large budgets
    uint64_t* keys = gkeys ? gkeys + blockIdx.x * (uint64_t)budget : reinterpret_cast<uint64_t*>(smem);
    uint64_t* sel = gkeys ? reinterpret_cast<uint64_t*>(smem) : keys + budget;  // sel_cap
    float* fine = reinterpret_cast<float*>(sel + sel_cap);        // L*k1
    float* c2 = fine + L * k1;                                    // L*npairs
    uint32_t* pairs = reinterpret_cast<uint32_t*>(c2 + L * (p.code_ij ? 256u : npairs));  // npairs
    uint32_t* coff = pairs + npairs;                              // budget
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_count;
    __shared__ TopkShared s_sel;

    const uint64_t q = blockIdx.x;
    if (p.chain) {  // the bin selection's ranges (a PDL dependent in a chained chunk)
        griddep_wait();
        griddep_launch();
    }
    qt_begin(p, q, 2);
    const int tid = threadIdx.x;
    const uint32_t R = nranges[q], C = ncand[q];
    const uint2* qr = ranges + q * (uint64_t)budget;

    for (uint32_t i = tid; i < L * k1; i += blockDim.x) fine[i] = fine_in[q * L * k1 + i];
    const bool ij = p.code_ij != 0;
    const uint32_t c2n = ij ? L * 256 : L * npairs;
    for (uint32_t i = tid; i < c2n; i += blockDim.x) c2[i] = __ldg((ij ? p.c2ij : p.c2) + i);
    for (uint32_t i = tid; i < npairs; i += blockDim.x) pairs[i] = __ldg(p.pairs + i);
    for (uint32_t r = tid; r < R; r += blockDim.x) coff[r] = qr[r].y;
    if (tid == 0) s_count = 0;
    __syncthreads();

    // every index is a position range: [0, n) unsharded, possibly empty on a shard
    constexpr bool sharded = true;
    uint32_t mine = 0;
    for (uint32_t j = tid; j < C; j += blockDim.x) {
        // range containing candidate j: last r with coff[r] <= j
        uint32_t lo = 0, hi = R - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (coff[mid] <= j) lo = mid; else hi = mid - 1;
        }
        const uint64_t pos = (uint64_t)__ldg(&qr[lo].x) + (j - coff[lo]);
        uint64_t key = kSentinel;
        if (!sharded || (pos >= p.shard_lo && pos < p.shard_hi)) {
            const uint64_t lp = pos - p.shard_lo;
            const uint32_t id = __ldg(p.ids + lp);
            const float d = line_distance_row<LT, PW>(p.codes + lp * p.row_bytes, fine, c2, pairs, L, k1, npairs, ij,
                                                      p.code_j ? 0x3FFu : p.code_pi ? 0x1FFu : 0xFFFFu, p.jt_ij,
                                                      p.code_j ? p.c2v : nullptr);
            key = ((uint64_t)orderable(d) << 32) | id;
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
    qt_end(p, q, 2);
}

namespace {
uint32_t sel_cap_for(const DevParams& p, uint32_t k) {
    const uint32_t kk = k < p.budget ? k : p.budget;
    return next_pow2(kk > 0 ? kk : 1);
}

// Opt in to the largest dynamic shared memory the kernel can take next to its static part.
template <class K>
void allow_max_smem(K kernel) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, kernel));
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

template <int LT, int PW>
void set_rerank_attr() {
    allow_max_smem(rerank_kernel<LT, PW>);
}
}  // namespace

size_t rerank_smem(const DevParams& p, uint32_t k, bool gkeys) {
    return (gkeys ? 0ull : 8ull * p.budget) + 8ull * sel_cap_for(p, k) + 4ull * p.L * p.k1 +
           4ull * p.L * (p.code_ij ? 256u : p.npairs) + 4ull * p.npairs + 4ull * p.budget;
}

int optin_bytes() {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return optin;
}

namespace {
bool generic_gkeys(const DevParams& p, uint32_t k) { return rerank_smem(p, k) + 2048 > (size_t)optin_bytes(); }
}  // namespace

bool rerank_needs_gkeys(const DevParams& p, uint32_t k) {
    if (kernel_variant() != 1 && rerank_ij_ok(p, k)) return rerank_ij_gkeys(p, k);
    return generic_gkeys(p, k);
}

void launch_rerank(const DevParams& p, uint64_t nq, uint32_t k, const WsSlice& ws, uint32_t* ids,
                   float* dists, uint32_t* counts, cudaStream_t s) {
    if (kernel_variant() != 1 && rerank_ij_ok(p, k)) {
        launch_rerank_ij(p, nq, k, ws, ids, dists, counts, s);
        return;
    }
    const bool gk = generic_gkeys(p, k);
    if (gk && !ws.keys) throw Error{PQTG_ERR_ARG, "workspace has no candidate-key buffer for this budget"};
    const size_t sm = rerank_smem(p, k, gk);
    if (sm + 2048 > (size_t)optin_bytes())
        throw Error{PQTG_ERR_UNSUPPORTED, "re-rank tables and selection do not fit shared memory at this budget"};
    const uint32_t cap = sel_cap_for(p, k);
    uint64_t* gkeys = gk ? ws.keys : nullptr;
#define PQTG_RERANK(LT, PW)                                                                          \
    launch_kernel(p.chain, rerank_kernel<LT, PW>, dim3((unsigned)nq), dim3(kThreads), sm, s, p, k, cap, ws.fine, ws.ranges, ws.nranges, \
                                                             ws.ncand, ids, dists, counts, gkeys)
    if (p.pw == 1) {
        switch (p.L) {
        case 16: PQTG_RERANK(16, 1); break;
        case 32: PQTG_RERANK(32, 1); break;
        case 64: PQTG_RERANK(64, 1); break;
        case 120: PQTG_RERANK(120, 1); break;
        default: PQTG_RERANK(0, 1); break;
        }
    } else {
        switch (p.L) {
        case 32: PQTG_RERANK(32, 2); break;
        default: PQTG_RERANK(0, 2); break;
        }
    }
#undef PQTG_RERANK
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void configure_kernels(const DevParams& p, uint32_t) {
    // function attributes are per device: configure each device once
    static std::once_flag once[64];
    int dev = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    std::call_once(once[dev & 63], [] {
        allow_max_smem(traverse_kernel<16, 8>);
        allow_max_smem(traverse_kernel<32, 16>);
        allow_max_smem(traverse_kernel<16, 16>);
        allow_max_smem(traverse_kernel<0, 0>);
        allow_max_smem(binsel_kernel<4, false, false>);
        allow_max_smem(binsel_kernel<16, true, false>);
        allow_max_smem(binsel_kernel<4, false, true>);
        allow_max_smem(binsel_kernel<16, true, true>);
        set_rerank_attr<16, 1>();
        set_rerank_attr<32, 1>();
        set_rerank_attr<64, 1>();
        set_rerank_attr<120, 1>();
        set_rerank_attr<0, 1>();
        set_rerank_attr<32, 2>();
        set_rerank_attr<0, 2>();
        configure_rerank_ij();
        configure_binsel_fast();
        configure_binsel_par();
        configure_traverse_part();
        configure_exact();
        configure_screen();
    });
    (void)p;
}

// =====================================================================================
// Per-shard top-k merge: G sorted lists per query -> global top-k by (dist, id).
// =====================================================================================
__global__ void merge_topk_kernel(uint32_t G, uint64_t nq, uint32_t k, const uint32_t* __restrict__ ids,
                                  const float* __restrict__ dists, const uint32_t* __restrict__ counts,
                                  uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                                  uint32_t* __restrict__ out_counts) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    uint32_t cur[16];
    for (uint32_t g = 0; g < G; ++g) cur[g] = 0;
    uint32_t out = 0;
    while (out < k) {
        int best = -1;
        uint64_t bk = kSentinel;
        for (uint32_t g = 0; g < G; ++g) {
            if (cur[g] < counts[g * nq + q]) {
                const uint64_t off = ((uint64_t)g * nq + q) * k + cur[g];
                const uint64_t key = ((uint64_t)orderable(dists[off]) << 32) | ids[off];
                if (best < 0 || key < bk) {
                    best = (int)g;
                    bk = key;
                }
            }
        }
        if (best < 0) break;
        const uint64_t off = ((uint64_t)best * nq + q) * k + cur[best];
        out_ids[q * k + out] = ids[off];
        out_dists[q * k + out] = dists[off];
        ++cur[best];
        ++out;
    }
    for (uint32_t i = out; i < k; ++i) {
        out_ids[q * k + i] = 0xFFFFFFFFu;
        out_dists[q * k + i] = __uint_as_float(0x7F800000u);
    }
    out_counts[q] = out;
}

// Parallel merge of G sorted lists per query (one CTA per query). For G <= 32: every list is cut
// at M, the largest of the lists' ceil(kk/G)-th keys (the lists' first ceil(kk/G) keys, >= kk in
// all, lie at or below M, so the top kk of the union do too), the kept keys are compacted and
// each is written at its rank among them -- its rank in the union -- found by counting (keys are
// (dist, id) with distinct ids, so ranks are distinct). Otherwise each element's rank is its index
// in its own list plus, per other list, a binary search. Elements of rank < kk are written at
// their rank.
constexpr int kMergeThreads = 256;
constexpr uint32_t kMergeMaxLists = 64;

__global__ void __launch_bounds__(kMergeThreads) merge_ranked_kernel(uint32_t G, uint64_t nq, uint32_t k,
                                                                     const uint32_t* __restrict__ ids,
                                                                     const float* __restrict__ dists,
                                                                     const uint32_t* __restrict__ counts,
                                                                     uint32_t* __restrict__ out_ids,
                                                                     float* __restrict__ out_dists,
                                                                     uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);  // [G][k], then the kept keys (G <= 32)
    __shared__ uint32_t cnt[kMergeMaxLists], s_len[32], s_off[33];
    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    if (tid < G) cnt[tid] = min(counts[(uint64_t)tid * nq + q], k);
    __syncthreads();
    for (uint32_t e = tid; e < G * k; e += blockDim.x) {
        const uint32_t g = e / k, i = e - g * k;
        if (i < cnt[g]) {
            const uint64_t off = ((uint64_t)g * nq + q) * k + i;
            keys[e] = ((uint64_t)orderable(dists[off]) << 32) | ids[off];
        }
    }
    __syncthreads();
    uint32_t total = 0;
    for (uint32_t g = 0; g < G; ++g) total += cnt[g];
    const uint32_t kk = total < k ? total : k;
    if (G <= 32) {
        if (tid < 32) {
            const uint32_t n = tid < G ? cnt[tid] : 0u;
            const uint32_t c = (kk + G - 1) / G;
            uint32_t have = n < c ? n : c;
            uint64_t mx = have ? keys[tid * k + have - 1] : 0ull;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                const uint64_t o = __shfl_xor_sync(0xffffffffu, mx, d);
                mx = o > mx ? o : mx;
                have += __shfl_xor_sync(0xffffffffu, have, d);
            }
            const uint64_t thr = have >= kk ? mx : ~0ull;
            uint32_t len = 0;  // list keys <= thr
            if (tid < G) {
                const uint64_t* l = keys + tid * k;
                uint32_t lo = 0, hi = n;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (l[mid] <= thr) lo = mid + 1; else hi = mid;
                }
                len = lo;
            }
            uint32_t incl = len;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                if (tid >= (uint32_t)d) incl += v;
            }
            if (tid < G) s_len[tid] = len;
            if (tid <= G) s_off[tid] = incl - len;
        }
        __syncthreads();
        const uint32_t E = s_off[G];
        uint64_t* kept = keys + (uint64_t)G * k;
        for (uint32_t e = tid; e < G * k; e += blockDim.x) {
            const uint32_t g = e / k, i = e - g * k;
            if (i < s_len[g]) kept[s_off[g] + i] = keys[e];
        }
        __syncthreads();
        for (uint32_t e = tid; e < E; e += blockDim.x) {
            const uint64_t key = kept[e];
            uint32_t rank = 0, j = 0;
            for (; j + 4 <= E; j += 4)  // broadcast reads, four in flight
                rank += (uint32_t)(kept[j] < key) + (uint32_t)(kept[j + 1] < key) + (uint32_t)(kept[j + 2] < key) +
                        (uint32_t)(kept[j + 3] < key);
            for (; j < E; ++j) rank += kept[j] < key;
            if (rank < kk) {
                out_ids[q * k + rank] = (uint32_t)(key & 0xFFFFFFFFu);
                out_dists[q * k + rank] = unorderable((uint32_t)(key >> 32));
            }
        }
    } else {
        for (uint32_t e = tid; e < G * k; e += blockDim.x) {
            const uint32_t g = e / k, i = e - g * k;
            if (i >= cnt[g] || i >= kk) continue;  // an element at index >= kk of its list ranks >= kk
            const uint64_t key = keys[e];
            uint32_t rank = i;
            for (uint32_t h = 0; h < G && rank < kk; ++h) {
                if (h == g) continue;
                const uint64_t* l = keys + (uint64_t)h * k;
                uint32_t lo = 0, hi = cnt[h];  // keys of list h below `key`
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (l[mid] < key) lo = mid + 1; else hi = mid;
                }
                rank += lo;
            }
            if (rank < kk) {
                out_ids[q * k + rank] = (uint32_t)(key & 0xFFFFFFFFu);
                out_dists[q * k + rank] = unorderable((uint32_t)(key >> 32));
            }
        }
    }
    for (uint32_t i = kk + tid; i < k; i += blockDim.x) {
        out_ids[q * k + i] = 0xFFFFFFFFu;
        out_dists[q * k + i] = __uint_as_float(0x7F800000u);
    }
    if (tid == 0) out_counts[q] = kk;
}

void launch_merge(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* ids, const float* dists,
                  const uint32_t* counts, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                  cudaStream_t s) {
    if (nq == 0) return;
    const size_t sm = (size_t)shards * k * 8 * (shards <= 32 ? 2 : 1);  // lists (+ kept keys)
    if (k > 0 && shards <= kMergeMaxLists && sm + 1024 <= (size_t)optin_bytes()) {
        static std::once_flag once[64];
        int dev = 0;
        PQTG_CUDA_CHECK(cudaGetDevice(&dev));
        std::call_once(once[dev & 63], [] { allow_max_smem(merge_ranked_kernel); });
        merge_ranked_kernel<<<(unsigned)nq, kMergeThreads, sm, s>>>(shards, nq, k, ids, dists, counts, out_ids,
                                                                    out_dists, out_counts);
    } else {
        const unsigned blocks = (unsigned)((nq + 127) / 128);
        merge_topk_kernel<<<blocks, 128, 0, s>>>(shards, nq, k, ids, dists, counts, out_ids, out_dists, out_counts);
    }
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
