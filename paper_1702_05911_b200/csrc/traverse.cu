// traverse.cu — K1 fast path: tree traversal (pqtree.cpp:74-120) with one CTA per
// (query, tree part) instead of one per query.
//
// A part's work is independent of the other parts' until bin selection: its fine-part LUT
// entries (pqtree.cpp:84-93), its level-1 totals and order (:88-100), and the level-2
// distances of its w best parents' children (:102-117). Splitting a query over P CTAs gives
// P times the parallelism of the latency-bound chains, and each CTA stages its w parents'
// level-2 codebook blocks ([m][k2] f32, contiguous) into shared memory with TMA bulk copies
// (cp.async.bulk → UBLKCP) on one mbarrier, so the whole working set is in flight at once
// instead of 16 registers' worth per thread. The level-2 chains then read shared memory.
// pick_slope_table (binorder.cpp:52-65) needs two parts' lists; bin selection computes it.
//
// Exactness: every sum is the reference's sequential fp32 chain (common.cuh sq_step,
// explicit __f*_rn), every sort reproduces its total order.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using namespace dev;

namespace {

constexpr int kTpThreads = 128;
constexpr int kFineBatch = 32;  // fine-part codebook values loaded per thread per batch

struct TpLayout {
    size_t blk, y, fine, l1d, l1o, l2d, l2c, total;
    uint32_t blk_stride;  // floats per staged parent block (padded; 16-byte multiple)
};

__host__ __device__ inline TpLayout tp_layout(const DevParams& p) {
    TpLayout l{};
    const uint32_t mk = p.m * p.k2;
    // pad so consecutive parents' blocks start k2 banks apart: the lanes (parent r, child c)
    // of a warp then read distinct banks at every t
    uint32_t pad = 0;
    while (((mk + pad) % 32 != p.k2 % 32 || pad % 4) && pad < 128) ++pad;
    if (pad >= 128) pad = (4 - mk % 4) % 4;
    l.blk_stride = mk + pad;
    size_t o = 0;
    l.blk = o;
    o += (size_t)p.w * l.blk_stride * 4;
    l.y = o;
    o += (size_t)p.m * 4;
    l.fine = o;
    o += (size_t)p.per_part * p.k1 * 4;
    l.l1d = o;
    o += (size_t)p.k1 * 4;
    l.l1o = o;
    o += (size_t)p.k1 * 4;
    l.l2d = o;
    o += (size_t)p.W * 4;
    l.l2c = o;
    o += (size_t)p.W * 4;
    l.total = (o + 15) & ~size_t(15);
    return l;
}

}  // namespace

template <int K1T, int K2T>
__global__ void __launch_bounds__(kTpThreads) traverse_part_kernel(DevParams p, const float* __restrict__ Q,
                                                                   float* __restrict__ fine_out,
                                                                   float* __restrict__ l2d_out,
                                                                   uint32_t* __restrict__ l2c_out, uint32_t bulk) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t k1 = K1T ? (uint32_t)K1T : p.k1, k2 = K2T ? (uint32_t)K2T : p.k2;
    const uint32_t P = p.P, m = p.m, fd = p.fd, pp = p.per_part, W = p.W, w = p.w;
    const TpLayout lay = tp_layout(p);
    float* blk = reinterpret_cast<float*>(smem + lay.blk);
    float* y = reinterpret_cast<float*>(smem + lay.y);
    float* fine = reinterpret_cast<float*>(smem + lay.fine);
    float* l1d = reinterpret_cast<float*>(smem + lay.l1d);
    uint32_t* l1o = reinterpret_cast<uint32_t*>(smem + lay.l1o);
    float* l2d = reinterpret_cast<float*>(smem + lay.l2d);
    uint32_t* l2c = reinterpret_cast<uint32_t*>(smem + lay.l2c);

    const uint64_t q = blockIdx.x / P;
    const uint32_t part = blockIdx.x - (uint32_t)q * P;
    const uint32_t tid = threadIdx.x;
    const uint32_t jobs = pp * k1;  // this part's fine LUT entries (f, i)
    const uint32_t f0 = part * pp;

    if (tid == 0) mbar_init(&mbar, 1);
    const float* yq = Q + q * p.D + (uint64_t)part * m;
    for (uint32_t t = tid; t < m; t += blockDim.x) y[t] = __ldg(yq + t);
    // first batch of this thread's first fine job, in flight across the barrier
    float cv[kFineBatch];
    auto load_batch = [&](uint32_t idx, uint32_t t0) {
        const uint32_t f = f0 + idx / k1, i = idx - (idx / k1) * k1;
        const float* c = p.fine_t + ((size_t)f * fd + t0) * k1 + i;
#pragma unroll
        for (int u = 0; u < kFineBatch; ++u) cv[u] = t0 + u < fd ? __ldg(c + (size_t)u * k1) : 0.0f;
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
            for (int u = 0; u < kFineBatch; ++u)
                if (t0 + u < fd) acc = sq_step(acc, yf[t0 + u], cv[u]);
            t0 += kFineBatch;
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

    // stage the w best parents' level-2 blocks L2[part][parent][m][k2]
    const uint32_t mk = m * k2, bs = lay.blk_stride;
    if (bulk) {
        if (tid == 0) {
            mbar_expect_tx(&mbar, w * mk * 4);
            for (uint32_t r = 0; r < w; ++r)
                bulk_g2s(blk + r * bs, p.l2_t + ((size_t)part * k1 + l1o[r]) * mk, mk * 4, &mbar);
        }
        mbar_wait(&mbar, 0);
    } else {
        for (uint32_t e = tid; e < w * mk; e += blockDim.x) {
            const uint32_t r = e / mk, o = e - r * mk;
            blk[r * bs + o] = __ldg(p.l2_t + ((size_t)part * k1 + l1o[r]) * mk + o);
        }
        __syncthreads();
    }

    // level-2: l2_sq(y_p, L2[part][parent][c], m) sequentially over m (pqtree.cpp:102-111)
    for (uint32_t j = tid; j < W; j += blockDim.x) {
        const uint32_t r = j / k2, c = j - r * k2;
        const float* b = blk + r * bs + c;
        float acc = 0.0f;
        uint32_t t = 0;
        for (; t + 16 <= m; t += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = sq_step(acc, y[t + u], b[(t + u) * k2]);
        }
        for (; t < m; ++t) acc = sq_step(acc, y[t], b[t * k2]);
        l2d[j] = acc;
        l2c[j] = (l1o[r] << 16) | c;
    }
    __syncthreads();

    // rank by (dist, parent, child) (pqtree.cpp:112-117)
    for (uint32_t j = tid; j < W; j += blockDim.x) {
        const float d = l2d[j];
        const uint32_t code = l2c[j];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < W; ++o) {
            const float dj = l2d[o];
            const uint32_t cj = l2c[o];
            rank += (dj < d) || (dj == d && cj < code);
        }
        const size_t out = (q * P + part) * W + rank;
        l2d_out[out] = d;
        l2c_out[out] = code;
    }
}

namespace {

template <int A, int B>
void tp_allow(int optin) {
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, traverse_part_kernel<A, B>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(traverse_part_kernel<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

}  // namespace

bool traverse_part_ok(const DevParams& p) {
    // the staged parent blocks should leave room for several CTAs per SM
    return tp_layout(p).total <= 64 * 1024 && p.W < 65536;
}

void configure_traverse_part() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    tp_allow<16, 8>(optin);
    tp_allow<32, 16>(optin);
    tp_allow<16, 16>(optin);
    tp_allow<0, 0>(optin);
}

void launch_traverse_part(const DevParams& p, const float* queries, uint64_t nq, const WsSlice& ws,
                          cudaStream_t s) {
    const TpLayout lay = tp_layout(p);
    const uint64_t mk_bytes = (uint64_t)p.m * p.k2 * 4;
    const uint32_t bulk = (mk_bytes % 16 == 0 && (lay.blk_stride * 4) % 16 == 0 &&
                           (reinterpret_cast<uintptr_t>(p.l2_t) & 15) == 0)
                              ? 1u
                              : 0u;
    const unsigned grid = (unsigned)(nq * p.P);
#define PQTG_TP(A, B)                                                                                   \
    traverse_part_kernel<A, B><<<grid, kTpThreads, lay.total, s>>>(p, queries, ws.fine, ws.l2_dist, \
                                                                   ws.l2_code, bulk)
    if (p.k1 == 16 && p.k2 == 8) PQTG_TP(16, 8);
    else if (p.k1 == 32 && p.k2 == 16) PQTG_TP(32, 16);
    else if (p.k1 == 16 && p.k2 == 16) PQTG_TP(16, 16);
    else PQTG_TP(0, 0);
#undef PQTG_TP
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
