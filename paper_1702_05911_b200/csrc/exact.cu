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
#include <mutex>

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
template <bool PREFIX>  // PREFIX: write every prefix entry's exact distance in line order, no cut
__global__ void __launch_bounds__(kExThreads) exact_rerank_kernel(DevParams p, const float* __restrict__ Q, uint32_t kp,
                                                                  const uint32_t* __restrict__ line_ids,
                                                                  const uint32_t* __restrict__ line_counts, uint32_t k,
                                                                  uint32_t* __restrict__ out_ids,
                                                                  float* __restrict__ out_dists,
                                                                  uint32_t* __restrict__ out_counts,
                                                                  pqtg_query_stats* __restrict__ stats,
                                                                  float* __restrict__ exact_out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t D = p.D, Dp = p.db_stride;
    unsigned char* ring = smem;                                     // kExStages × 128 × kExRow
    float* y = reinterpret_cast<float*>(smem + (size_t)kExStages * kExThreads * kExRow);
    uint64_t* keys = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(y) + ((size_t)D * 4 + 15) / 16 * 16);
    __shared__ __align__(8) uint64_t full[kExStages];
    const uint64_t q = blockIdx.x;
    if (p.chain) griddep_wait();  // the re-rank's line-ranked prefix (a PDL dependent in a chained chunk)
    qt_begin(p, q, 2);
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
        // the row of this id: by id, or through a position shard's id -> row table
        const uint64_t row = p.id2row ? (tid < cnt ? p.id2row[id] : 0u) : id;
        // chunk c's bytes are armed on its slot's barrier by thread 0 before a block barrier,
        // then every thread bulk-copies its own row's piece (the copies issue in parallel)
        auto chunk_bytes = [&](uint32_t c) {
            const uint32_t d0 = c * kExDims;
            return (Dp - d0 < (uint32_t)kExDims ? Dp - d0 : (uint32_t)kExDims) * 4;
        };
        auto issue_mine = [&](uint32_t c, uint32_t use) {
            if (tid < cnt)
                bulk_g2s(ring + (size_t)(use % kExStages) * kExThreads * kExRow + tid * kExRow,
                         p.db + (size_t)row * Dp + c * kExDims, chunk_bytes(c), &full[use % kExStages]);
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
        if (tid < cnt) {
            if (PREFIX) exact_out[q * kp + g0 + tid] = acc;
            else keys[g0 + tid] = ((uint64_t)orderable(acc) << 32) | id;
        }
    }
    if (PREFIX) return;
    __syncthreads();
    const uint32_t kk = n < k ? n : k;
    block_sort_write(keys, n, kk, k, q, out_ids, out_dists, out_counts);
    if (tid == 0 && stats) stats[q].exact_evals = n;
    qt_end(p, q, 2);
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
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, exact_rerank_kernel<false>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(exact_rerank_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, exact_rerank_kernel<true>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(exact_rerank_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

void launch_exact(const DevParams& p, const float* queries, uint64_t nq, uint32_t kp, const uint32_t* line_ids,
                  const uint32_t* line_counts, uint32_t k, uint32_t* ids, float* dists, uint32_t* counts,
                  pqtg_query_stats* stats, cudaStream_t s) {
    if (nq == 0) return;
    launch_kernel(p.chain, exact_rerank_kernel<false>, dim3((unsigned)nq), dim3(kExThreads), exact_smem(p, kp), s, 
        p, queries, kp, line_ids, line_counts, k, ids, dists, counts, stats, nullptr);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_exact_prefix(const DevParams& p, const float* queries, uint64_t nq, uint32_t kp, const uint32_t* line_ids,
                         const uint32_t* line_counts, float* exact, cudaStream_t s) {
    if (nq == 0) return;
    launch_kernel(p.chain, exact_rerank_kernel<true>, dim3((unsigned)nq), dim3(kExThreads), exact_smem(p, kp), s, 
        p, queries, kp, line_ids, line_counts, 0, nullptr, nullptr, nullptr, nullptr, exact);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

namespace {

__global__ void fill_id2row_kernel(const uint32_t* __restrict__ ids, uint64_t count, uint32_t* __restrict__ id2row) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        id2row[ids[i]] = (uint32_t)i;
}

// One CTA per query: the G (line, id)-sorted lists in shared memory; each element's global
// (line, id) rank by binary searches in the other lists; the first R' = min(R, C) form the
// reference's exact prefix (search.cpp:229-240), ranked again by (exact, id) (:242-249).
constexpr int kMxThreads = 256;

__global__ void __launch_bounds__(kMxThreads) merge_exact_kernel(uint32_t G, uint64_t nq, uint32_t kp, uint32_t R,
                                                                 uint32_t k, const uint32_t* __restrict__ ids,
                                                                 const float* __restrict__ line,
                                                                 const float* __restrict__ exact,
                                                                 const uint32_t* __restrict__ counts,
                                                                 pqtg_query_stats* __restrict__ stats,
                                                                 uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                                                                 uint32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* lk = reinterpret_cast<uint64_t*>(smem);   // [G][kp] (line, id) keys
    uint64_t* pre = lk + (size_t)G * kp;                 // [R'] (exact, id) keys at their line rank
    __shared__ uint32_t cnt[16];
    const uint64_t q = blockIdx.x;
    if (threadIdx.x < G) cnt[threadIdx.x] = min(counts[(uint64_t)threadIdx.x * nq + q], kp);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < G * kp; e += blockDim.x) {
        const uint32_t g = e / kp, i = e - g * kp;
        if (i < cnt[g]) {
            const uint64_t off = ((uint64_t)g * nq + q) * kp + i;
            lk[e] = ((uint64_t)orderable(line[off]) << 32) | ids[off];
        }
    }
    __syncthreads();
    const uint64_t C = stats[q].candidates;
    const uint32_t Rp = (uint32_t)(C < R ? C : R);
    for (uint32_t e = threadIdx.x; e < G * kp; e += blockDim.x) {
        const uint32_t g = e / kp, i = e - g * kp;
        if (i >= cnt[g] || i >= Rp) continue;
        const uint64_t key = lk[e];
        uint32_t rank = i;
        for (uint32_t h = 0; h < G && rank < Rp; ++h) {
            if (h == g) continue;
            const uint64_t* l = lk + (uint64_t)h * kp;
            uint32_t lo = 0, hi = cnt[h];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (l[mid] < key) lo = mid + 1; else hi = mid;
            }
            rank += lo;
        }
        if (rank < Rp) {
            const uint64_t off = ((uint64_t)g * nq + q) * kp + i;
            pre[rank] = ((uint64_t)orderable(exact[off]) << 32) | (uint32_t)(key & 0xFFFFFFFFu);
        }
    }
    __syncthreads();
    const uint32_t kk = Rp < k ? Rp : k;
    for (uint32_t e = threadIdx.x; e < Rp; e += blockDim.x) {  // rank by (exact, id): O(R'^2) counts
        const uint64_t me = pre[e];
        uint32_t r = 0;
        for (uint32_t j = 0; j < Rp; ++j) r += pre[j] < me;
        if (r < kk) {
            out_ids[q * k + r] = (uint32_t)(me & 0xFFFFFFFFu);
            out_dists[q * k + r] = unorderable((uint32_t)(me >> 32));
        }
    }
    for (uint32_t i = kk + threadIdx.x; i < k; i += blockDim.x) {
        out_ids[q * k + i] = 0xFFFFFFFFu;
        out_dists[q * k + i] = __uint_as_float(0x7F800000u);
    }
    if (threadIdx.x == 0) {
        out_counts[q] = kk;
        stats[q].exact_evals = Rp;
    }
}

}  // namespace

void launch_fill_id2row(const uint32_t* ids, uint64_t count, uint32_t* id2row, cudaStream_t s) {
    if (count == 0) return;
    const uint64_t blocks = (count + 255) / 256;
    fill_id2row_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(ids, count, id2row);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_merge_exact(uint32_t G, uint64_t nq, uint32_t kp, uint32_t R, uint32_t k, const uint32_t* ids,
                        const float* line, const float* exact, const uint32_t* counts, pqtg_query_stats* stats,
                        uint32_t* out_ids, float* out_dists, uint32_t* out_counts, cudaStream_t s) {
    if (nq == 0) return;
    const size_t sm = ((size_t)G * kp + R) * 8;
    if (sm + 1024 > (size_t)optin_bytes()) throw Error{PQTG_ERR_UNSUPPORTED, "sharded exact re-rank: prefix too long"};
    static std::once_flag once[64];
    int dev = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    std::call_once(once[dev & 63], [] {
        cudaFuncAttributes a{};
        cudaFuncGetAttributes(&a, merge_exact_kernel);
        cudaFuncSetAttribute(merge_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_bytes() - (int)a.sharedSizeBytes);
    });
    merge_exact_kernel<<<(unsigned)nq, kMxThreads, sm, s>>>(G, nq, kp, R, k, ids, line, exact, counts, stats, out_ids,
                                                          out_dists, out_counts);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
