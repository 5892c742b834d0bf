// sharded_kernels.cu — the per-query range lists of a query-partitioned sharded search
// (sharded.cpp): each rank runs traversal + bin selection for its block of the batch, packs
// every query's (start position, candidate offset) ranges densely, the packed blocks are
// all-gathered, and every rank unpacks the whole batch's ranges into its workspace before
// re-ranking its position shard.
#include <cub/block/block_scan.cuh>

#include <cstdint>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using dev::sq_step;

namespace {

constexpr int kScanThreads = 512;

// off[i] = sum of cnt[0..i) for i <= n (off[n] = the total), one block: each thread sums a
// contiguous chunk, one block scan of the chunk sums, each thread writes its chunk's offsets
__global__ void __launch_bounds__(kScanThreads) scan_counts_kernel(const uint32_t* __restrict__ cnt, uint64_t n,
                                                                   uint64_t* __restrict__ off) {
    using Scan = cub::BlockScan<uint64_t, kScanThreads>;
    __shared__ typename Scan::TempStorage tmp;
    const uint64_t per = (n + kScanThreads - 1) / kScanThreads;
    const uint64_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
    uint64_t sum = 0;
    for (uint64_t i = b; i < e; ++i) sum += cnt[i];
    uint64_t excl, tot;
    Scan(tmp).ExclusiveSum(sum, excl, tot);
    for (uint64_t i = b; i < e; ++i) {
        off[i] = excl;
        excl += cnt[i];
    }
    if (threadIdx.x == 0) off[n] = tot;
}

// dense <- per-query rows (pack) or per-query rows <- dense (unpack); one warp per query
template <bool PACK>
__global__ void __launch_bounds__(256) move_ranges_kernel(uint2* __restrict__ rows, uint32_t stride,
                                                          const uint32_t* __restrict__ cnt,
                                                          const uint64_t* __restrict__ off, uint2* __restrict__ dense,
                                                          uint64_t n) {
    const uint64_t q = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= n) return;
    const uint32_t c = cnt[q];
    uint2* row = rows + q * (uint64_t)stride;
    uint2* d = dense + off[q];
    for (uint32_t i = threadIdx.x & 31; i < c; i += 32) {
        if (PACK) d[i] = row[i];
        else row[i] = d[i];
    }
}

// fine_dists[q][f][i] = l2_sq(y_f, slice(f, i), fd) in the traversal's (and the reference's,
// pqtree.cpp:90-93) sequential fp32 order: the sharded search recomputes the batch's fine LUTs on
// every rank (L·k1·fd multiply-adds per query) instead of all-gathering them (4·L·k1 bytes per
// query, 4 KB on the SIFT1B tree)
__global__ void __launch_bounds__(256) fine_lut_kernel(DevParams p, const float* __restrict__ Q, uint64_t nq,
                                                       float* __restrict__ fine) {
    extern __shared__ float y[];  // the current query
    const uint32_t L = p.L, k1 = p.k1, fd = p.fd, D = p.D;
    for (uint64_t q = blockIdx.x; q < nq; q += gridDim.x) {  // a few resident CTAs loop over the batch
        for (uint32_t t = threadIdx.x; t < D; t += blockDim.x) y[t] = Q[q * D + t];
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < L * k1; idx += blockDim.x) {
            const uint32_t f = idx / k1, i = idx - f * k1;
            const float* c = p.fine_t + (size_t)f * fd * k1 + i;
            const float* yf = y + f * fd;
            float acc = 0.0f;
            for (uint32_t t = 0; t < fd; ++t, c += k1) acc = sq_step(acc, yf[t], __ldg(c));
            fine[q * L * k1 + idx] = acc;
        }
        __syncthreads();
    }
}

// many small device-to-device copies in one launch (the local / simulated transports' stand-in
// for one NCCL group): blockIdx.y = segment, 4-byte words, grid-stride over the segment
__global__ void __launch_bounds__(256) copy_segments_kernel(CopySegments segs) {
    const CopySegment sg = segs.s[blockIdx.y];
    const uint32_t* src = static_cast<const uint32_t*>(sg.src);
    uint32_t* dst = static_cast<uint32_t*>(sg.dst);
    const uint64_t words = sg.bytes / 4;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = __ldg(src + i);
}

}  // namespace

void launch_copy_segments(const std::vector<CopySegment>& segs, cudaStream_t s) {
    for (size_t b = 0; b < segs.size(); b += kCopySegmentsMax) {
        CopySegments batch{};
        uint64_t most = 0;
        for (size_t i = b; i < segs.size() && i < b + kCopySegmentsMax; ++i) {
            const CopySegment& c = segs[i];
            if ((c.bytes & 3) || (reinterpret_cast<uintptr_t>(c.src) & 3) || (reinterpret_cast<uintptr_t>(c.dst) & 3))
                throw Error{PQTG_ERR_ARG, "copy segment not 4-byte aligned"};
            batch.s[batch.n++] = c;
            most = c.bytes > most ? c.bytes : most;
        }
        if (!batch.n || !most) continue;
        const uint64_t blocks = (most / 4 + 1023) / 1024;
        copy_segments_kernel<<<dim3((unsigned)(blocks < 64 ? (blocks ? blocks : 1) : 64), batch.n), 256, 0, s>>>(batch);
        PQTG_CUDA_CHECK(cudaGetLastError());
    }
}

void launch_fine_lut(const DevParams& p, const float* queries, uint64_t nq, float* fine, cudaStream_t s) {
    if (nq == 0) return;
    const uint64_t grid = nq < 148 * 8 ? nq : 148 * 8;
    fine_lut_kernel<<<(unsigned)grid, 256, p.D * sizeof(float), s>>>(p, queries, nq, fine);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* off, cudaStream_t s) {
    scan_counts_kernel<<<1, kScanThreads, 0, s>>>(cnt, n, off);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_pack_ranges(const uint2* ranges, uint32_t stride, const uint32_t* cnt, const uint64_t* off, uint64_t n,
                        uint2* dense, cudaStream_t s) {
    if (n == 0) return;
    move_ranges_kernel<true><<<(unsigned)((n + 7) / 8), 256, 0, s>>>(const_cast<uint2*>(ranges), stride, cnt, off, dense, n);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_unpack_ranges(const uint2* dense, const uint32_t* cnt, const uint64_t* off, uint64_t n, uint32_t stride,
                          uint2* ranges, cudaStream_t s) {
    if (n == 0) return;
    move_ranges_kernel<false><<<(unsigned)((n + 7) / 8), 256, 0, s>>>(ranges, stride, cnt, off, const_cast<uint2*>(dense), n);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
