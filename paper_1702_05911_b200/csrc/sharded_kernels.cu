// sharded_kernels.cu — the per-query range lists of a query-partitioned sharded search
// (sharded.cpp): each rank runs traversal + bin selection for its block of the batch, packs
// every query's (start position, candidate offset) ranges densely, the packed blocks are
// all-gathered, and every rank unpacks the whole batch's ranges into its workspace before
// re-ranking its position shard.
#include <cub/block/block_scan.cuh>

#include <cstdint>

#include "pqtg_internal.h"

namespace pqtg {

namespace {

constexpr int kScanThreads = 256;

// off[i] = sum of cnt[0..i) for i <= n (off[n] = the total), one block
__global__ void __launch_bounds__(kScanThreads) scan_counts_kernel(const uint32_t* __restrict__ cnt, uint64_t n,
                                                                   uint64_t* __restrict__ off) {
    using Scan = cub::BlockScan<uint64_t, kScanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < n; base += kScanThreads) {
        const uint64_t i = base + threadIdx.x;
        const uint64_t v = i < n ? cnt[i] : 0;
        uint64_t excl, tot;
        Scan(tmp).ExclusiveSum(v, excl, tot);
        const uint64_t carry = s_carry;
        if (i < n) off[i] = carry + excl;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[n] = s_carry;
}

// dense <- per-query rows (pack) or per-query rows <- dense (unpack); one block per query
template <bool PACK>
__global__ void __launch_bounds__(256) move_ranges_kernel(uint2* __restrict__ rows, uint32_t stride,
                                                          const uint32_t* __restrict__ cnt,
                                                          const uint64_t* __restrict__ off, uint2* __restrict__ dense) {
    const uint64_t q = blockIdx.x;
    const uint32_t c = cnt[q];
    uint2* row = rows + q * (uint64_t)stride;
    uint2* d = dense + off[q];
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        if (PACK) d[i] = row[i];
        else row[i] = d[i];
    }
}

}  // namespace

void launch_scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* off, cudaStream_t s) {
    scan_counts_kernel<<<1, kScanThreads, 0, s>>>(cnt, n, off);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_pack_ranges(const uint2* ranges, uint32_t stride, const uint32_t* cnt, const uint64_t* off, uint64_t n,
                        uint2* dense, cudaStream_t s) {
    if (n == 0) return;
    move_ranges_kernel<true><<<(unsigned)n, 256, 0, s>>>(const_cast<uint2*>(ranges), stride, cnt, off, dense);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_unpack_ranges(const uint2* dense, const uint32_t* cnt, const uint64_t* off, uint64_t n, uint32_t stride,
                          uint2* ranges, cudaStream_t s) {
    if (n == 0) return;
    move_ranges_kernel<false><<<(unsigned)n, 256, 0, s>>>(ranges, stride, cnt, off, const_cast<uint2*>(dense));
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
