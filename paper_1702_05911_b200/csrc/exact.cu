// exact.cu — K6: exact re-rank of the best line-quantized candidates (search.cpp:229-257).
//
// With raw vectors attached (PqtIndex::attach_database, search.cpp:44-49) and rerank_exact > 0,
// the reference takes rerank = min(max(rerank_exact, k), C) best candidates by line distance,
// replaces their distances by l2_sq(db.row(id), y, dim) (distance.hpp:11-18: sequential fp32,
// d = x − y) and re-sorts them by (dist, id); it returns the first min(k, C). K5 already
// produced the line-ranked prefix (its k' = max(k, rerank_exact) best); one CTA per query
// here streams those rows through shared memory with TMA bulk copies (below) and ranks them
// by the exact keys.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {
constexpr int kExThreads = 128;   // candidates per group (one thread each)
constexpr int kExDims = 64;       // dimensions per staged chunk
constexpr int kExStages = 3;      // chunks in flight
constexpr int kExRow = 272;       // bytes per staged row piece: 256 + 16 pad (conflict-free LDS.128)
}

// With the rows staged by TMA: per group of <= 128 candidates (thread r = candidate r), the
// 64-dimension pieces of all rows are bulk-copied (cp.async.bulk, one copy per row piece) into a
// 3-chunk shared ring on per-chunk mbarriers, so ~50 KB per CTA is in flight from HBM while each
// thread sums its own row's previous piece in order (distance.hpp:11-18). Device rows have a
// stride of D rounded up to 4 floats (16-byte bulk copies).
__global__ void __launch_bounds__(kExThreads) exact_rerank_kernel(DevParams p, const float* __restrict__ Q, uint32_t kp,
                                                                  const uint32_t* __restrict__ line_ids,
                                                                  const uint32_t* __restrict__ line_counts, uint32_t k,
                                                                  uint32_t* __restrict__ out_ids,
                                                                  float* __restrict__ out_dists,
                                                                  uint32_t* __restrict__ out_counts,
                                                                  pqtg_query_stats* __restrict__ stats) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t D = p.D, Dp = p.db_stride;
    unsigned char* ring = smem;                                     // kExStages × 128 × kExRow
    float* y = reinterpret_cast<float*>(smem + (size_t)kExStages * kExThreads * kExRow);
    uint64_t* keys = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(y) + ((size_t)D * 4 + 15) / 16 * 16);
    __shared__ __align__(8) uint64_t full[kExStages];
    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    const uint32_t n = line_counts[q];  // = rerank: min(max(k, rerank_exact), C) line-ranked candidates
    for (uint32_t t = tid; t < D; t += blockDim.x) y[t] = Q[q * D + t];
    if (tid == 0)
        for (int s = 0; s < kExStages; ++s) mbar_init(&full[s], 1);
    const uint32_t nch = (D + kExDims - 1) / kExDims;
    uint32_t uses = 0;  // chunks consumed so far (all groups): slot = uses % stages, parity = (uses / stages) & 1
    for (uint32_t g0 = 0; g0 < n; g0 += kExThreads) {
        const uint32_t cnt = n - g0 < (uint32_t)kExThreads ? n - g0 : (uint32_t)kExThreads;
        const uint32_t id = tid < cnt ? line_ids[q * kp + g0 + tid] : 0u;
        // chunk c's bytes are armed on its slot's barrier by thread 0 before a block barrier,
        // then every thread bulk-copies its own row's piece (the copies issue in parallel)
        auto chunk_bytes = [&](uint32_t c) {
            const uint32_t d0 = c * kExDims;
            return (Dp - d0 < (uint32_t)kExDims ? Dp - d0 : (uint32_t)kExDims) * 4;
        };
        auto issue_mine = [&](uint32_t c, uint32_t use) {
            if (tid < cnt)
                bulk_g2s(ring + (size_t)(use % kExStages) * kExThreads * kExRow + tid * kExRow,
                         p.db + (size_t)id * Dp + c * kExDims, chunk_bytes(c), &full[use % kExStages]);
        };
        if (tid == 0)
            for (uint32_t c = 0; c < nch && c < (uint32_t)kExStages; ++c)
                mbar_expect_tx(&full[(uses + c) % kExStages], chunk_bytes(c) * cnt);
        __syncthreads();
        for (uint32_t c = 0; c < nch && c < (uint32_t)kExStages; ++c) issue_mine(c, uses + c);
        float acc = 0.0f;
        for (uint32_t c = 0; c < nch; ++c, ++uses) {
            const uint32_t slot = uses % kExStages;
            mbar_wait(&full[slot], (uses / kExStages) & 1u);
            const uint32_t d0 = c * kExDims, dn = D - d0 < (uint32_t)kExDims ? D - d0 : (uint32_t)kExDims;
            if (tid < cnt) {
                const float4* x4 = reinterpret_cast<const float4*>(ring + (size_t)slot * kExThreads * kExRow + tid * kExRow);
                if (dn == (uint32_t)kExDims) {
#pragma unroll
                    for (int u = 0; u < kExDims / 4; ++u) {
                        const float4 v = x4[u];
                        acc = sq_step(acc, v.x, y[d0 + 4 * u + 0]);
                        acc = sq_step(acc, v.y, y[d0 + 4 * u + 1]);
                        acc = sq_step(acc, v.z, y[d0 + 4 * u + 2]);
                        acc = sq_step(acc, v.w, y[d0 + 4 * u + 3]);
                    }
                } else {
                    const float* x = reinterpret_cast<const float*>(x4);
                    for (uint32_t u = 0; u < dn; ++u) acc = sq_step(acc, x[u], y[d0 + u]);
                }
            }
            const bool more = c + kExStages < nch;
            if (tid == 0 && more) mbar_expect_tx(&full[slot], chunk_bytes(c + kExStages) * cnt);
            __syncthreads();  // the slot is free again and armed for chunk c + stages
            if (more) issue_mine(c + kExStages, uses + kExStages);
        }
        if (tid < cnt) keys[g0 + tid] = ((uint64_t)orderable(acc) << 32) | id;
    }
    __syncthreads();
    const uint32_t kk = n < k ? n : k;
    block_sort_write(keys, n, kk, k, q, out_ids, out_dists, out_counts);
    if (tid == 0 && stats) stats[q].exact_evals = n;
}

size_t exact_smem(const DevParams& p, uint32_t kp) {
    uint32_t n2 = 1;
    while (n2 < kp) n2 <<= 1;  // block_sort_write's bitonic fallback pads to a power of two
    return (size_t)kExStages * kExThreads * kExRow + ((size_t)p.D * 4 + 15) / 16 * 16 + (size_t)n2 * 8;
}

void configure_exact() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, exact_rerank_kernel));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(exact_rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

void launch_exact(const DevParams& p, const float* queries, uint64_t nq, uint32_t kp, const uint32_t* line_ids,
                  const uint32_t* line_counts, uint32_t k, uint32_t* ids, float* dists, uint32_t* counts,
                  pqtg_query_stats* stats, cudaStream_t s) {
    if (nq == 0) return;
    exact_rerank_kernel<<<(unsigned)nq, kExThreads, exact_smem(p, kp), s>>>(p, queries, kp, line_ids, line_counts, k,
                                                                              ids, dists, counts, stats);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
