// traverse.cu — K1 fast path: tree traversal (pqtree.cpp:74-120) with one CTA per
// (query, tree part) instead of one per query.
//
// A part's work is independent of the other parts' until bin selection: its fine-part LUT
// entries (pqtree.cpp:84-93), its level-1 totals and order (:88-100), and the level-2
// distances of its w best parents' children (:102-117). Splitting a query over P CTAs gives
// P times the parallelism of the latency-bound chains, and each CTA streams its w parents'
// level-2 codebook blocks ([m][k2] f32, contiguous) into shared memory with TMA bulk copies
// (cp.async.bulk → UBLKCP) in t-chunks through two mbarrier-tracked buffers, so the next chunk
// is in flight while the chains run over the current one and a CTA needs only ~18 KB of shared
// memory (about 12 resident per SM). The level-2 chains read shared memory.
// pick_slope_table (binorder.cpp:52-65) needs two parts' lists; bin selection computes it.
//
// Exactness: every sum is the reference's sequential fp32 chain (common.cuh sq_step,
// explicit __f*_rn), every sort reproduces its total order.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kTpThreads = 128;

struct TpLayout {
    size_t blk, y, fine, l1d, l1o, keys, total;
    uint32_t rows;        // t-rows of the parent blocks staged per chunk (multiple of 4)
    uint32_t blk_stride;  // floats per staged parent piece (padded; 16-byte multiple)
};

// The w best parents' blocks L2[part][parent][m][k2] are staged in chunks of `rows` t-rows
// through two buffers (~16 KB together), so a CTA needs little shared memory and many CTAs
// (query parts) are resident per SM.
__host__ __device__ inline TpLayout tp_layout(const DevParams& p) {
    TpLayout l{};
    uint32_t rows = (16u * 1024u) / (2u * p.w * p.k2 * 4u);
    rows = rows / 4 * 4;
    if (rows < 4) rows = 4;
    if (rows > (p.m + 3) / 4 * 4) rows = (p.m + 3) / 4 * 4;
    l.rows = rows;
    const uint32_t mk = rows * p.k2;
    // pad so consecutive parents' pieces start k2 banks apart: the lanes (parent r, child c)
    // of a warp then read distinct banks at every t
    uint32_t pad = 0;
    while (((mk + pad) % 32 != p.k2 % 32 || pad % 4) && pad < 128) ++pad;
    if (pad >= 128) pad = (4 - mk % 4) % 4;
    l.blk_stride = mk + pad;
    size_t o = 0;
    l.blk = o;
    o += 2ull * p.w * l.blk_stride * 4;
    l.y = o;
    o += (size_t)p.m * 4;
    l.fine = o;
    o += (size_t)p.per_part * p.k1 * 4;
    l.l1d = o;
    o += (size_t)p.k1 * 4;
    l.l1o = o;
    o += (size_t)p.k1 * 4;
    l.keys = (o + 7) & ~size_t(7);  // level-2 sort exchange: one u64 per power-of-two slot
    uint32_t n2 = 1;
    while (n2 < p.W) n2 <<= 1;
    o = l.keys + (size_t)n2 * 8;
    l.total = (o + 15) & ~size_t(15);
    return l;
}

// Ascending bitonic sort of N u64 keys, thread t holding key t (t < N; N <= blockDim): the
// network fully unrolled, partner exchange by shuffle within a warp and through `buf` (N
// slots) across warps. Every thread of the block calls it when N > 32.
template <int N>
__device__ __forceinline__ uint64_t bitonic_block(uint64_t key, uint32_t tid, uint64_t* buf) {
#pragma unroll
    for (uint32_t kk = 2; kk <= (uint32_t)N; kk <<= 1) {
#pragma unroll
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
            uint64_t other;
            if (jj >= 32) {
                __syncthreads();
                if (tid < (uint32_t)N) buf[tid] = key;
                __syncthreads();
                other = tid < (uint32_t)N ? buf[tid ^ jj] : ~0ull;
            } else {
                other = __shfl_xor_sync(0xffffffffu, key, jj);
            }
            const uint32_t take_min = ((tid & kk) == 0) == ((tid & jj) == 0), lt = other < key, gt = other > key;
            key = ((take_min & lt) | (~take_min & 1u & gt)) ? other : key;  // branch-free
        }
    }
    return key;
}

}  // namespace

// FB: fine-part codebook values loaded per thread per batch (8 when fd <= 8, else 32)
template <int K1T, int K2T, int FB>
__global__ void __launch_bounds__(kTpThreads) traverse_part_kernel(DevParams p, const float* __restrict__ Q,
                                                                   float* __restrict__ fine_out,
                                                                   float* __restrict__ l2d_out,
                                                                   uint32_t* __restrict__ l2c_out, uint32_t bulk,
                                                                   const TpLayout lay) {  // tp_layout(p), host-made
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar[2];
    const uint32_t k1 = K1T ? (uint32_t)K1T : p.k1, k2 = K2T ? (uint32_t)K2T : p.k2;
    const uint32_t P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W, w = p.w;
    float* blk = reinterpret_cast<float*>(smem + lay.blk);
    float* y = reinterpret_cast<float*>(smem + lay.y);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    float* l1d = reinterpret_cast<float*>(smem + lay.l1d);
    uint32_t* l1o = reinterpret_cast<uint32_t*>(smem + lay.l1o);

    const uint64_t q = blockIdx.x / P;
    const uint32_t part = blockIdx.x - (uint32_t)q * P;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    const uint32_t tid = threadIdx.x;
    const uint32_t jobs = pp * k1;  // this part's fine LUT entries (f, i)
    const uint32_t f0 = part * pp;

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
    }
    const float* yq = Q + q * p.D + (uint64_t)part * m;
    for (uint32_t t = tid; t < m; t += blockDim.x) y[t] = __ldg(yq + t);
    // first batch of this thread's first fine job, in flight across the barrier
    float cv[FB];
    auto load_batch = [&](uint32_t idx, uint32_t t0) {
        const uint32_t f = f0 + idx / k1, i = idx - (idx / k1) * k1;
        const float* c = p.fine_t + ((size_t)f * fd + t0) * k1 + i;
#pragma unroll
        for (int u = 0; u < FB; ++u) cv[u] = t0 + u < fd ? __ldg(c + (size_t)u * k1) : 0.0f;
    };
    if (tid < jobs) load_batch(tid, 0);
    __syncthreads();

    // fine_dists[f][i] = l2_sq(y_f, slice(f, i), fd), sequential (pqtree.cpp:90-93)
    for (uint32_t idx = tid; idx < jobs; idx += blockDim.x) {
        const uint32_t lf = idx / k1, i = idx - lf * k1;
        const float* yf = y + lf * fd;
        float acc = 0.0f;
        for (uint32_t t0 = 0;;) {
#pragma unroll
            for (int u = 0; u < FB; ++u)
                if (t0 + u < fd) acc = sq_step(acc, yf[t0 + u], cv[u]);
            t0 += FB;
            if (t0 >= fd) break;
            load_batch(idx, t0);
        }
        fine[idx] = acc;
        fine_out[(q * p.L + f0 + lf) * k1 + i] = acc;
        if (idx + blockDim.x < jobs) load_batch(idx + blockDim.x, 0);
    }
    __syncthreads();

    // level-1 totals: the part's fine partials summed in f order (pqtree.cpp:88-96), then
    // ranked by (dist, id) (:98-100)
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        float tot = 0.0f;
        for (uint32_t lf = 0; lf < pp; ++lf) tot = __fadd_rn(tot, fine[lf * k1 + i]);
        l1d[i] = tot;
    }
    __syncthreads();
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        const float d = l1d[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[j];
            rank += (dj < d) || (dj == d && j < i);
        }
        l1o[rank] = i;
    }
    __syncthreads();

    // level-2: l2_sq(y_p, L2[part][parent][c], m) sequentially over m (pqtree.cpp:102-111), the
    // parents' blocks streamed in t-chunks through two buffers (TMA bulk copies on one mbarrier
    // per buffer; chunk c + 2 is issued as soon as chunk c's buffer is free)
    const uint32_t mk = m * k2, bs = lay.blk_stride, rows = lay.rows;
    const uint32_t nch = (m + rows - 1) / rows;
    auto stage = [&](uint32_t c) {  // thread 0 (bulk) / every thread (plain loads)
        const uint32_t t0 = c * rows, nr = m - t0 < rows ? m - t0 : rows, b = c & 1u;
        float* dst = blk + (size_t)b * w * bs;
        if (bulk) {
            if (tid == 0) {
                mbar_expect_tx(&mbar[b], w * nr * k2 * 4);
                for (uint32_t r = 0; r < w; ++r)
                    bulk_g2s(dst + r * bs, p.l2_t + ((size_t)part * k1 + l1o[r]) * mk + (size_t)t0 * k2, nr * k2 * 4,
                             &mbar[b]);
            }
        } else {
            for (uint32_t e = tid; e < w * nr * k2; e += blockDim.x) {
                const uint32_t r = e / (nr * k2), o = e - r * nr * k2;
                dst[r * bs + o] = __ldg(p.l2_t + ((size_t)part * k1 + l1o[r]) * mk + (size_t)t0 * k2 + o);
            }
        }
    };
    stage(0);
    if (nch > 1) stage(1);
    const uint32_t j = tid;  // W <= blockDim (traverse_part_ok)
    const uint32_t r = j / k2, c = j - r * k2;
    float acc = 0.0f;
    uint32_t phases = 0u;  // bit b: buffer b's mbarrier parity
    for (uint32_t ch = 0; ch < nch; ++ch) {
        const uint32_t b = ch & 1u, t0 = ch * rows, nr = m - t0 < rows ? m - t0 : rows;
        if (bulk) {
            mbar_wait(&mbar[b], (phases >> b) & 1u);
            phases ^= 1u << b;
        } else {
            __syncthreads();
        }
        if (j < W) {
            const float* bp = blk + (size_t)b * w * bs + r * bs + c;
            const float* yt = y + t0;
            uint32_t t = 0;
            // y four at a time (16-byte aligned: t0 and the y block are multiples of 4 floats)
            const float4* y4 = reinterpret_cast<const float4*>(yt);
            for (; t + 16 <= nr; t += 16) {
#pragma unroll
                for (int u = 0; u < 16; u += 4) {
                    const float4 yv = y4[(t + u) >> 2];
                    acc = sq_step(acc, yv.x, bp[(t + u + 0) * k2]);
                    acc = sq_step(acc, yv.y, bp[(t + u + 1) * k2]);
                    acc = sq_step(acc, yv.z, bp[(t + u + 2) * k2]);
                    acc = sq_step(acc, yv.w, bp[(t + u + 3) * k2]);
                }
            }
            for (; t < nr; ++t) acc = sq_step(acc, yt[t], bp[t * k2]);
        }
        __syncthreads();  // buffer b is free
        if (ch + 2 < nch) stage(ch + 2);
    }
    // order by (dist, parent, child) (pqtree.cpp:112-117): the keys (orderable(dist) << 32 |
    // parent << 16 | child) -- distances are sums of squares, never -0 or NaN, so the u64 order
    // is the reference's -- bitonic-sorted across the block (shuffles below 32, shared memory
    // above), thread t ends holding rank t
    uint64_t key = ~0ull;
    if (j < W) key = ((uint64_t)orderable(acc) << 32) | ((l1o[r] << 16) | c);
    uint64_t* kbuf = reinterpret_cast<uint64_t*>(smem + lay.keys);  // used when W > 32
    if (W <= 32) {
        if (tid < 32) key = bitonic_block<32>(key, tid, kbuf);  // warp 0 alone, shuffles only
    } else if (W <= 64) {
        key = bitonic_block<64>(key, tid, kbuf);
    } else {
        key = bitonic_block<128>(key, tid, kbuf);
    }
    if (j < W) {
        const size_t out = (q * P + part) * W + j;
        l2d_out[out] = unorderable((uint32_t)(key >> 32));
        l2c_out[out] = (uint32_t)key;
    }
    qt_end(p, q, 0);
}

// Small trees (W = w·k2 <= 32, k1 <= 32, P <= 4): one CTA per query, one warp per part, no
// block barrier after the query is staged. In traverse_part_kernel three of its four warps wait
// at a barrier while one warp runs the W level-2 chains; here every warp runs its own part's
// chains, reading the parents' [m][k2] blocks straight from L2 (the level-2 codebooks are
// shared by all queries) with eight loads in flight, and sorts them with a one-warp network.
template <int K1T, int K2T, int FB>
__global__ void __launch_bounds__(128) traverse_warp_kernel(DevParams p, const float* __restrict__ Q,
                                                            float* __restrict__ fine_out, float* __restrict__ l2d_out,
                                                            uint32_t* __restrict__ l2c_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k1 = K1T ? (uint32_t)K1T : p.k1, k2 = K2T ? (uint32_t)K2T : p.k2;
    const uint32_t P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W;
    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x, lane = tid & 31, part = tid >> 5;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    float* y = reinterpret_cast<float*>(smem);                        // [D]
    float* fine = y + ((p.D + 3) & ~3u) + part * pp * 32;             // [P][pp][<= 32]
    float* l1d = y + ((p.D + 3) & ~3u) + P * pp * 32 + part * 32;     // [P][32]
    uint32_t* l1o = reinterpret_cast<uint32_t*>(y + ((p.D + 3) & ~3u) + P * pp * 32 + P * 32) + part * 32;
    for (uint32_t t = tid; t < p.D; t += blockDim.x) y[t] = __ldg(Q + q * p.D + t);
    __syncthreads();
    if (part >= P) return;
    const uint32_t f0 = part * pp, jobs = pp * k1;
    // fine_dists[f][i] = l2_sq(y_f, slice(f, i), fd), sequential (pqtree.cpp:90-93)
    for (uint32_t idx = lane; idx < jobs; idx += 32) {
        const uint32_t lf = idx / k1, i = idx - lf * k1;
        const float* yf = y + (f0 + lf) * fd;
        const float* c = p.fine_t + (size_t)(f0 + lf) * fd * k1 + i;
        float acc = 0.0f;
        for (uint32_t t0 = 0; t0 < fd; t0 += FB) {
            float cv[FB];
#pragma unroll
            for (int u = 0; u < FB; ++u) cv[u] = t0 + u < fd ? __ldg(c + (size_t)(t0 + u) * k1) : 0.0f;
#pragma unroll
            for (int u = 0; u < FB; ++u)
                if (t0 + u < fd) acc = sq_step(acc, yf[t0 + u], cv[u]);
        }
        fine[lf * k1 + i] = acc;
        fine_out[(q * p.L + f0 + lf) * k1 + i] = acc;
    }
    __syncwarp();
    // level-1 totals in f order (pqtree.cpp:88-96), ranked by (dist, id) (:98-100)
    if (lane < k1) {
        float tot = 0.0f;
        for (uint32_t lf = 0; lf < pp; ++lf) tot = __fadd_rn(tot, fine[lf * k1 + lane]);
        l1d[lane] = tot;
    }
    __syncwarp();
    if (lane < k1) {
        const float d = l1d[lane];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[j];
            rank += (dj < d) || (dj == d && j < lane);
        }
        l1o[rank] = lane;
    }
    __syncwarp();
    // level-2: l2_sq(y_p, L2[part][parent][c], m), sequential over m (pqtree.cpp:102-111)
    uint64_t key = ~0ull;
    if (lane < W) {
        const uint32_t r = lane / k2, c = lane - r * k2, parent = l1o[r];
        const float* cb = p.l2_t + ((size_t)part * k1 + parent) * m * k2 + c;
        const float* yp = y + part * m;
        float acc = 0.0f;
        uint32_t t = 0;
        for (; t + 8 <= m; t += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(cb + (size_t)(t + u) * k2);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = sq_step(acc, yp[t + u], v[u]);
        }
        for (; t < m; ++t) acc = sq_step(acc, yp[t], __ldg(cb + (size_t)t * k2));
        key = ((uint64_t)orderable(acc) << 32) | ((parent << 16) | c);
    }
    key = bitonic_block<32>(key, lane, nullptr);  // (dist, parent, child) (pqtree.cpp:112-117)
    if (lane < W) {
        const size_t out = (q * P + part) * W + lane;
        l2d_out[out] = unorderable((uint32_t)(key >> 32));
        l2c_out[out] = (uint32_t)key;
    }
    qt_end(p, q, 0);
}

// Ascending bitonic sort of 32·EPT u64 keys held by one warp in registers, lane l holding keys
// l·EPT + i: exchanges below distance EPT stay in the lane (one thread does both sides), the
// others go through shuffles.
template <int EPT>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&e)[EPT], uint32_t lane) {
    constexpr uint32_t N = 32 * EPT;
#pragma unroll
    for (uint32_t kk = 2; kk <= N; kk <<= 1) {
#pragma unroll
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
            if (jj < (uint32_t)EPT) {
#pragma unroll
                for (uint32_t i = 0; i < (uint32_t)EPT; ++i) {
                    if (i & jj) continue;
                    const uint32_t n = lane * EPT + i;
                    const uint64_t a = e[i], b = e[i ^ jj];
                    // branch-free (the direction is lane-dependent: a ternary here compiled to
                    // divergent branches with reconvergence around every exchange)
                    const uint32_t up = (n & kk) == 0, lt = b < a, gt = a < b;
                    const bool sw = (up & lt) | (~up & 1u & gt);
                    e[i] = sw ? b : a;
                    e[i ^ jj] = sw ? a : b;
                }
            } else {
#pragma unroll
                for (uint32_t i = 0; i < (uint32_t)EPT; ++i) {
                    const uint32_t n = lane * EPT + i;
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, e[i], jj / EPT);
                    const uint32_t take_min = ((n & kk) == 0) == ((n & jj) == 0), lt = o < e[i], gt = o > e[i];
                    e[i] = ((take_min & lt) | (~take_min & 1u & gt)) ? o : e[i];
                }
            }
        }
    }
}

// The warp-per-part traversal for W = 32·EPT > 32 (the SIFT1B tree: W = 128, k2 = 16): lane l
// owns children l·EPT .. l·EPT + EPT − 1 — consecutive children of one parent when k2 % EPT == 0,
// read as one 16-byte load per t — and sorts the part's W keys held in registers.
template <int K1T, int K2T, int EPT>
__global__ void __launch_bounds__(128) traverse_warp_wide_kernel(DevParams p, const float* __restrict__ Q,
                                                                 float* __restrict__ fine_out,
                                                                 float* __restrict__ l2d_out,
                                                                 uint32_t* __restrict__ l2c_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr uint32_t k1 = K1T, k2 = K2T;
    const uint32_t P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W;
    const uint64_t q = blockIdx.x;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    const uint32_t tid = threadIdx.x, lane = tid & 31, part = tid >> 5;
    float* y = reinterpret_cast<float*>(smem);
    float* fine = y + ((p.D + 3) & ~3u) + part * pp * 32;
    float* l1d = y + ((p.D + 3) & ~3u) + P * pp * 32 + part * 32;
    uint32_t* l1o = reinterpret_cast<uint32_t*>(y + ((p.D + 3) & ~3u) + P * pp * 32 + P * 32) + part * 32;
    for (uint32_t t = tid; t < p.D; t += blockDim.x) y[t] = __ldg(Q + q * p.D + t);
    __syncthreads();
    if (part >= P) return;
    const uint32_t f0 = part * pp, jobs = pp * k1;
    // fine LUT (pqtree.cpp:90-93): jobs / 32 independent sequential chains per lane
    for (uint32_t idx = lane; idx < jobs; idx += 32) {
        const uint32_t lf = idx / k1, i = idx - lf * k1;
        const float* yf = y + (f0 + lf) * fd;
        const float* c = p.fine_t + (size_t)(f0 + lf) * fd * k1 + i;
        float acc = 0.0f;
        for (uint32_t t = 0; t < fd; ++t) acc = sq_step(acc, yf[t], __ldg(c + (size_t)t * k1));
        fine[lf * k1 + i] = acc;
        fine_out[(q * p.L + f0 + lf) * k1 + i] = acc;
    }
    __syncwarp();
    if (lane < k1) {
        float tot = 0.0f;
        for (uint32_t lf = 0; lf < pp; ++lf) tot = __fadd_rn(tot, fine[lf * k1 + lane]);
        l1d[lane] = tot;
    }
    __syncwarp();
    if (lane < k1) {
        const float d = l1d[lane];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[j];
            rank += (dj < d) || (dj == d && j < lane);
        }
        l1o[rank] = lane;
    }
    __syncwarp();
    // level-2 chains (pqtree.cpp:102-111): EPT children of one parent per lane
    uint64_t key[EPT];
    const uint32_t j0 = lane * EPT, r = j0 / k2, c0 = j0 - r * k2;
    const bool live = j0 < W;
    const uint32_t parent = live ? l1o[r] : 0u;
    const float* cb = p.l2_t + ((size_t)part * k1 + parent) * m * k2 + c0;
    const float* yp = y + part * m;
    float acc[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) acc[e] = 0.0f;
    if (live) {
        for (uint32_t t = 0; t < m; t += 4) {
            float4 v[4][EPT / 4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int e4 = 0; e4 < EPT / 4; ++e4)
                    v[u][e4] = t + u < m ? __ldg(reinterpret_cast<const float4*>(cb + (size_t)(t + u) * k2) + e4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t + u >= m) break;
                const float yv = yp[t + u];
#pragma unroll
                for (int e4 = 0; e4 < EPT / 4; ++e4) {
                    acc[4 * e4 + 0] = sq_step(acc[4 * e4 + 0], yv, v[u][e4].x);
                    acc[4 * e4 + 1] = sq_step(acc[4 * e4 + 1], yv, v[u][e4].y);
                    acc[4 * e4 + 2] = sq_step(acc[4 * e4 + 2], yv, v[u][e4].z);
                    acc[4 * e4 + 3] = sq_step(acc[4 * e4 + 3], yv, v[u][e4].w);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e)
        key[e] = live ? ((uint64_t)orderable(acc[e]) << 32) | ((parent << 16) | (c0 + e)) : ~0ull;
    warp_sort_regs<EPT>(key, lane);  // (dist, parent, child) (pqtree.cpp:112-117)
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const uint32_t o = lane * EPT + e;
        if (o < W) {
            l2d_out[(q * P + part) * W + o] = unorderable((uint32_t)(key[e] >> 32));
            l2c_out[(q * P + part) * W + o] = (uint32_t)key[e];
        }
    }
    qt_end(p, q, 0);
}


// Small batches (fewer queries than SMs): latency, not throughput. One CTA per (query, part)
// stages the part's WHOLE level-2 codebook (k1 × m × k2 floats) and its fine parts' codebook
// slice with two TMA bulk copies issued at kernel start, in parallel with the query load, so the
// chain of dependent memory round trips is [query ‖ codebooks] → compute, instead of the
// per-parent block loads that follow the level-1 order. Same arithmetic and orders as
// traverse_part_kernel (pqtree.cpp:74-120).
struct TsLayout {
    size_t cb, ft, y, fine, l1d, l1o, keys, total;
};

__host__ __device__ inline TsLayout ts_layout(const DevParams& p) {
    TsLayout l{};
    size_t o = 0;
    l.cb = o;
    o += (size_t)p.k1 * p.m * p.k2 * 4;
    l.ft = o;
    o += (size_t)p.per_part * p.fd * p.k1 * 4;
    l.y = o;
    o += ((size_t)p.m * 4 + 15) & ~size_t(15);
    l.fine = o;
    o += (size_t)p.per_part * p.k1 * 4;
    l.l1d = o;
    o += (size_t)p.k1 * 4;
    l.l1o = o;
    o += (size_t)p.k1 * 4;
    l.keys = (o + 7) & ~size_t(7);
    uint32_t n2 = 1;
    while (n2 < p.W) n2 <<= 1;
    o = l.keys + (size_t)n2 * 8;
    l.total = (o + 15) & ~size_t(15);
    return l;
}

__global__ void __launch_bounds__(kTpThreads) traverse_small_kernel(DevParams p, const float* __restrict__ Q,
                                                                    float* __restrict__ fine_out,
                                                                    float* __restrict__ l2d_out,
                                                                    uint32_t* __restrict__ l2c_out, const TsLayout lay) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t k1 = p.k1, k2 = p.k2, P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W;
    float* cb = reinterpret_cast<float*>(smem + lay.cb);
    float* ft = reinterpret_cast<float*>(smem + lay.ft);
    float* y = reinterpret_cast<float*>(smem + lay.y);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    float* l1d = reinterpret_cast<float*>(smem + lay.l1d);
    uint32_t* l1o = reinterpret_cast<uint32_t*>(smem + lay.l1o);
    const uint64_t q = blockIdx.x / P;
    const uint32_t part = blockIdx.x - (uint32_t)q * P;
    qt_begin(p, q, 0);
    if (p.chain) griddep_launch();  // a chained chunk's bin selection may launch
    const uint32_t tid = threadIdx.x, f0 = part * pp;
    const uint32_t cb_bytes = k1 * m * k2 * 4, ft_bytes = pp * fd * k1 * 4;
    if (tid == 0) {
        mbar_init(&mbar, 1);
        mbar_expect_tx(&mbar, cb_bytes + ft_bytes);
        bulk_g2s(cb, p.l2_t + (size_t)part * k1 * m * k2, cb_bytes, &mbar);
        bulk_g2s(ft, p.fine_t + (size_t)f0 * fd * k1, ft_bytes, &mbar);
    }
    const float* yq = Q + q * p.D + (uint64_t)part * m;
    for (uint32_t t = tid; t < m; t += blockDim.x) y[t] = __ldg(yq + t);
    __syncthreads();
    mbar_wait(&mbar, 0);
    // fine_dists[f][i] = l2_sq(y_f, slice(f, i), fd), sequential (pqtree.cpp:90-93)
    for (uint32_t idx = tid; idx < pp * k1; idx += blockDim.x) {
        const uint32_t lf = idx / k1, i = idx - lf * k1;
        const float* c = ft + (size_t)lf * fd * k1 + i;
        const float* yf = y + lf * fd;
        float acc = 0.0f;
        for (uint32_t t = 0; t < fd; ++t) acc = sq_step(acc, yf[t], c[t * k1]);
        fine[idx] = acc;
        fine_out[(q * p.L + f0 + lf) * k1 + i] = acc;
    }
    __syncthreads();
    // level-1 totals in f order (pqtree.cpp:88-96), ranked by (dist, id) (:98-100)
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        float tot = 0.0f;
        for (uint32_t lf = 0; lf < pp; ++lf) tot = __fadd_rn(tot, fine[lf * k1 + i]);
        l1d[i] = tot;
    }
    __syncthreads();
    for (uint32_t i = tid; i < k1; i += blockDim.x) {
        const float d = l1d[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < k1; ++j) {
            const float dj = l1d[j];
            rank += (dj < d) || (dj == d && j < i);
        }
        l1o[rank] = i;
    }
    __syncthreads();
    // level-2 chains of the w best parents' children from the staged codebook (pqtree.cpp:102-111)
    const uint32_t j = tid, r = j / k2, c = j - r * k2;
    float acc = 0.0f;
    if (j < W) {
        const float* bp = cb + (size_t)l1o[r] * m * k2 + c;
        for (uint32_t t = 0; t < m; ++t) acc = sq_step(acc, y[t], bp[t * k2]);
    }
    uint64_t key = ~0ull;
    if (j < W) key = ((uint64_t)orderable(acc) << 32) | ((l1o[r] << 16) | c);
    uint64_t* kbuf = reinterpret_cast<uint64_t*>(smem + lay.keys);
    if (W <= 32) {
        if (tid < 32) key = bitonic_block<32>(key, tid, kbuf);
    } else if (W <= 64) {
        key = bitonic_block<64>(key, tid, kbuf);
    } else {
        key = bitonic_block<128>(key, tid, kbuf);
    }
    if (j < W) {
        const size_t out = (q * P + part) * W + j;
        l2d_out[out] = unorderable((uint32_t)(key >> 32));
        l2c_out[out] = (uint32_t)key;
    }
    qt_end(p, q, 0);
}

namespace {

template <int A, int B, int FB>
void tp_allow1(int optin) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, traverse_part_kernel<A, B, FB>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(traverse_part_kernel<A, B, FB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes));
}

template <int A, int B>
void tp_allow(int optin) {
    tp_allow1<A, B, 8>(optin);
    tp_allow1<A, B, 32>(optin);
}

}  // namespace

bool traverse_part_ok(const DevParams& p) {
    // one level-2 chain per thread; the staged chunks leave room for many CTAs per SM
    return p.W <= (uint32_t)kTpThreads && tp_layout(p).total <= 48 * 1024;
}

void configure_traverse_part() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    {
        cudaFuncAttributes a{};
        PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, traverse_small_kernel));
        PQTG_CUDA_CHECK(cudaFuncSetAttribute(traverse_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             optin - (int)a.sharedSizeBytes));
    }
    tp_allow<16, 8>(optin);
    tp_allow<32, 16>(optin);
    tp_allow<16, 16>(optin);
    tp_allow<0, 0>(optin);
}

size_t tw_smem(const DevParams& p) {
    return ((size_t)((p.D + 3) & ~3u) + (size_t)p.P * p.per_part * 32 + (size_t)p.P * 32 * 2) * 4;
}

bool traverse_warp_ok(const DevParams& p) {
    static const bool off = std::getenv("PQTG_NO_TRAVERSE_WARP") != nullptr;
    // short level-2 chains only: SIFT1M (m = 64) 59 -> 51 us, DEEP (m = 48) 54 -> 45 us; GIST1M
    // (m = 240) is faster with its blocks staged in shared memory (33 vs 37 us)
    return !off && p.W <= 32 && p.k1 <= 32 && p.P <= 4 && p.m <= 128 && tw_smem(p) <= 48 * 1024;
}

bool traverse_warp_wide_ok(const DevParams& p) {
    static const bool off = std::getenv("PQTG_NO_TRAVERSE_WARP") != nullptr;
    return !off && p.W == 128 && p.k1 == 32 && p.k2 == 16 && p.P <= 4 && p.m <= 128 && tw_smem(p) <= 48 * 1024 &&
           (reinterpret_cast<uintptr_t>(p.l2_t) & 15) == 0;
}

// the whole-codebook staging pays when the batch leaves SMs idle and the part's level-2 codebook
// fits shared memory (SIFT1M / DEEP: 32 / 24 KB); PQTG_NO_TRAVERSE_SMALL=1 disables
bool traverse_small_ok(const DevParams& p, uint64_t nq) {
    static const bool off = std::getenv("PQTG_NO_TRAVERSE_SMALL") != nullptr;
    const uint64_t cb = (uint64_t)p.k1 * p.m * p.k2 * 4, ft = (uint64_t)p.per_part * p.fd * p.k1 * 4;
    return !off && nq * p.P <= 2 * 148 && p.W <= (uint32_t)kTpThreads && cb % 16 == 0 && ft % 16 == 0 &&
           ((uint64_t)p.k1 * p.m * p.k2 * 4) % 16 == 0 && ts_layout(p).total <= 96 * 1024 &&
           (reinterpret_cast<uintptr_t>(p.l2_t) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.fine_t) & 15) == 0;
}

void launch_traverse_part(const DevParams& p, const float* queries, uint64_t nq, const WsSlice& ws,
                          cudaStream_t s) {
    if (traverse_small_ok(p, nq)) {
        const TsLayout lay = ts_layout(p);
        traverse_small_kernel<<<(unsigned)(nq * p.P), kTpThreads, lay.total, s>>>(p, queries, ws.fine, ws.l2_dist,
                                                                                ws.l2_code, lay);
        PQTG_CUDA_CHECK(cudaGetLastError());
        return;
    }
    if (traverse_warp_wide_ok(p)) {
        traverse_warp_wide_kernel<32, 16, 4><<<(unsigned)nq, 32 * p.P, tw_smem(p), s>>>(p, queries, ws.fine,
                                                                                      ws.l2_dist, ws.l2_code);
        PQTG_CUDA_CHECK(cudaGetLastError());
        return;
    }
    if (traverse_warp_ok(p)) {
        const size_t sm = tw_smem(p);
        const unsigned th = 32 * p.P;
#define PQTG_TW(A, B)                                                                                           \
    (p.fd <= 8 ? traverse_warp_kernel<A, B, 8><<<(unsigned)nq, th, sm, s>>>(p, queries, ws.fine, ws.l2_dist,     \
                                                                            ws.l2_code)                          \
               : traverse_warp_kernel<A, B, 32><<<(unsigned)nq, th, sm, s>>>(p, queries, ws.fine, ws.l2_dist,    \
                                                                             ws.l2_code))
        if (p.k1 == 16 && p.k2 == 8) PQTG_TW(16, 8);
        else if (p.k1 == 16 && p.k2 == 16) PQTG_TW(16, 16);
        else PQTG_TW(0, 0);
#undef PQTG_TW
        PQTG_CUDA_CHECK(cudaGetLastError());
        return;
    }
    const TpLayout lay = tp_layout(p);
    const uint64_t mk_bytes = (uint64_t)p.m * p.k2 * 4, row_bytes = (uint64_t)lay.rows * p.k2 * 4;
    const uint32_t bulk = (mk_bytes % 16 == 0 && row_bytes % 16 == 0 && (lay.blk_stride * 4) % 16 == 0 &&
                           (reinterpret_cast<uintptr_t>(p.l2_t) & 15) == 0)
                              ? 1u
                              : 0u;
    const unsigned grid = (unsigned)(nq * p.P);
#define PQTG_TP(A, B)                                                                                         \
    (p.fd <= 8 ? traverse_part_kernel<A, B, 8><<<grid, kTpThreads, lay.total, s>>>(p, queries, ws.fine, ws.l2_dist, \
                                                                                   ws.l2_code, bulk, lay)          \
               : traverse_part_kernel<A, B, 32><<<grid, kTpThreads, lay.total, s>>>(p, queries, ws.fine,          \
                                                                                    ws.l2_dist, ws.l2_code, bulk, lay))
    if (p.k1 == 16 && p.k2 == 8) PQTG_TP(16, 8);
    else if (p.k1 == 32 && p.k2 == 16) PQTG_TP(32, 16);
    else if (p.k1 == 16 && p.k2 == 16) PQTG_TP(16, 16);
    else PQTG_TP(0, 0);
#undef PQTG_TP
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
