// exact.cu — K6: exact re-rank of the best line-quantized candidates (search.cpp:229-257).
//
// With raw vectors attached (PqtIndex::attach_database, search.cpp:44-49) and rerank_exact > 0,
// the reference takes rerank = min(max(rerank_exact, k), C) best candidates by line distance,
// replaces their distances by l2_sq(db.row(id), y, dim) (distance.hpp:11-18: sequential fp32,
// d = x − y) and re-sorts them by (dist, id); it returns the first min(k, C). K5 already
// produced the line-ranked prefix (its k' = max(k, rerank_exact) best); one CTA per query
// here streams each of those rows (16-byte loads, the query in shared memory), one thread per
// candidate, and ranks them by the exact keys.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {
constexpr int kExThreads = 128;
}

__global__ void __launch_bounds__(kExThreads) exact_rerank_kernel(DevParams p, const float* __restrict__ Q, uint32_t kp,
                                                                  const uint32_t* __restrict__ line_ids,
                                                                  const uint32_t* __restrict__ line_counts, uint32_t k,
                                                                  uint32_t* __restrict__ out_ids,
                                                                  float* __restrict__ out_dists,
                                                                  uint32_t* __restrict__ out_counts,
                                                                  pqtg_query_stats* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t D = p.D;
    float* y = reinterpret_cast<float*>(smem);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + ((size_t)D * 4 + 15) / 16 * 16);
    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    const uint32_t n = line_counts[q];  // = rerank: min(max(k, rerank_exact), C) line-ranked candidates
    for (uint32_t t = tid; t < D; t += blockDim.x) y[t] = Q[q * D + t];
    __syncthreads();
    const bool vec = (D & 3) == 0;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
        const uint32_t id = line_ids[q * kp + i];
        const float* x = p.db + (size_t)id * D;
        float acc = 0.0f;
        if (vec) {
            const float4* x4 = reinterpret_cast<const float4*>(x);
            uint32_t t = 0;
            for (; t + 16 <= D; t += 16) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(x4 + t / 4 + u);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc = sq_step(acc, v[u].x, y[t + 4 * u + 0]);
                    acc = sq_step(acc, v[u].y, y[t + 4 * u + 1]);
                    acc = sq_step(acc, v[u].z, y[t + 4 * u + 2]);
                    acc = sq_step(acc, v[u].w, y[t + 4 * u + 3]);
                }
            }
            for (; t < D; t += 4) {
                const float4 v = __ldg(x4 + t / 4);
                acc = sq_step(acc, v.x, y[t + 0]);
                acc = sq_step(acc, v.y, y[t + 1]);
                acc = sq_step(acc, v.z, y[t + 2]);
                acc = sq_step(acc, v.w, y[t + 3]);
            }
        } else {
            for (uint32_t t = 0; t < D; ++t) acc = sq_step(acc, __ldg(x + t), y[t]);
        }
        keys[i] = ((uint64_t)orderable(acc) << 32) | id;
    }
    __syncthreads();
    const uint32_t kk = n < k ? n : k;
    block_sort_write(keys, n, kk, k, q, out_ids, out_dists, out_counts);
    if (tid == 0 && stats) stats[q].exact_evals = n;
}

size_t exact_smem(const DevParams& p, uint32_t kp) {
    uint32_t n2 = 1;
    while (n2 < kp) n2 <<= 1;  // block_sort_write's bitonic fallback pads to a power of two
    return ((size_t)p.D * 4 + 15) / 16 * 16 + (size_t)n2 * 8;
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
