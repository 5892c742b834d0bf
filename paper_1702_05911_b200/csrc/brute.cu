// brute.cu — exact brute-force k-NN (the reference's brute_force_knn, search.cpp:276-299), the
// ground truth the recall of the PQT search is measured against (bench.cpp:23-44).
//
// For every query: l2_sq(db.row(i), y, dim) for all n rows (distance.hpp:11-18: sequential fp32,
// d = x − y, no FMA), then partial_sort by candidate_less = (dist, id) and the first min(k, n).
// One CTA per query streams the rows in blocks of 8 per thread (thread t: rows t, t + 256, …),
// keeps a running top-k in shared memory: each block's (dist, id) keys are appended to the
// current top-k and block_topk (topk.cuh: radix select + bitonic sort) keeps the k smallest —
// keys are distinct, so the result is the reference's ordering exactly.
#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"
#include "topk.cuh"

namespace pqtg {

using namespace dev;

namespace {
constexpr int kBfThreads = 256;
constexpr int kBfRows = 8;                               // rows per thread per block
constexpr uint32_t kBfBlock = kBfThreads * kBfRows;      // rows per block

uint32_t bf_sel_cap(uint32_t k) {
    uint32_t c = 256;
    while (c < k) c <<= 1;
    return c;
}

size_t bf_smem(uint32_t dim, uint32_t k) {
    return ((size_t)dim * 4 + 15) / 16 * 16 + ((size_t)k + kBfBlock) * 8 + (size_t)bf_sel_cap(k) * 8 + 256 * 4;
}
}  // namespace

__global__ void __launch_bounds__(kBfThreads) brute_force_kernel(const float* __restrict__ db, uint64_t n, uint32_t dim,
                                                                  const float* __restrict__ queries, uint32_t k,
                                                                  uint32_t sel_cap, uint32_t* __restrict__ out_ids,
                                                                  float* __restrict__ out_dists,
                                                                  uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    float* y = reinterpret_cast<float*>(smem);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + ((size_t)dim * 4 + 15) / 16 * 16);  // [k + block]
    uint64_t* sel = keys + k + kBfBlock;
    uint32_t* hist = reinterpret_cast<uint32_t*>(sel + sel_cap);
    __shared__ TopkShared sh;
    const uint64_t q = blockIdx.x;
    const uint32_t tid = threadIdx.x;
    for (uint32_t t = tid; t < dim; t += blockDim.x) y[t] = queries[q * dim + t];
    __syncthreads();
    const bool vec = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(db) & 15) == 0);
    uint32_t held = 0;  // keys[0..held): the running top-k, ascending
    for (uint64_t b0 = 0; b0 < n; b0 += kBfBlock) {
        const uint32_t nb = n - b0 < kBfBlock ? (uint32_t)(n - b0) : kBfBlock;
#pragma unroll
        for (int i = 0; i < kBfRows; ++i) {
            const uint32_t r = tid + i * kBfThreads;
            if (r >= nb) continue;
            const uint64_t row = b0 + r;
            const float* x = db + row * dim;
            float acc = 0.0f;
            if (vec) {
                const float4* x4 = reinterpret_cast<const float4*>(x);
                const float4* y4 = reinterpret_cast<const float4*>(y);
                for (uint32_t u = 0; u < dim / 4; ++u) {
                    const float4 a = __ldg(x4 + u), c = y4[u];
                    acc = sq_step(acc, a.x, c.x);
                    acc = sq_step(acc, a.y, c.y);
                    acc = sq_step(acc, a.z, c.z);
                    acc = sq_step(acc, a.w, c.w);
                }
            } else {
                for (uint32_t t = 0; t < dim; ++t) acc = sq_step(acc, __ldg(x + t), y[t]);
            }
            keys[held + r] = ((uint64_t)orderable(acc) << 32) | (uint32_t)row;
        }
        __syncthreads();
        const uint32_t total = held + nb;
        const uint32_t kk = total < k ? total : k;
        block_topk(keys, total, kk, sel, sel_cap, hist, sh);
        __syncthreads();
        for (uint32_t j = tid; j < kk; j += blockDim.x) keys[j] = sel[j];
        held = kk;
        __syncthreads();
    }
    write_topk(keys, held, k, q, out_ids, out_dists, out_counts);
}

bool brute_force_ok(uint32_t dim, uint32_t k) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return k <= 4096 && bf_smem(dim, k) + 1024 <= (size_t)optin;
}

void launch_brute_force(const float* d_db, uint64_t n, uint32_t dim, const float* d_queries, uint64_t nq, uint32_t k,
                        uint32_t* d_ids, float* d_dists, uint32_t* d_counts, cudaStream_t s) {
    if (nq == 0) return;
    {  // per device: the opt-in shared memory
        int dev = 0, optin = 0;
        PQTG_CUDA_CHECK(cudaGetDevice(&dev));
        PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        cudaFuncAttributes a{};
        PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, brute_force_kernel));
        PQTG_CUDA_CHECK(cudaFuncSetAttribute(brute_force_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             optin - (int)a.sharedSizeBytes));
    }
    brute_force_kernel<<<(unsigned)nq, kBfThreads, bf_smem(dim, k), s>>>(d_db, n, dim, d_queries, k, bf_sel_cap(k),
                                                                       d_ids, d_dists, d_counts);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
