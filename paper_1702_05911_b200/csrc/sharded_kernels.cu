// sharded_kernels.cu — the per-query range lists of a query-partitioned sharded search
// (sharded.cpp): each rank runs traversal + bin selection for its block of the batch, packs
// every query's (start position, candidate offset) ranges densely, the packed blocks are
// all-gathered, and every rank unpacks the whole batch's ranges into its workspace before
// re-ranking its position shard.
#include <cub/block/block_load.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_store.cuh>

#include <cstdint>
#include <mutex>

#include "common.cuh"
#include "pqtg_internal.h"

namespace pqtg {

using dev::sq_step;

namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;

// off[i] = sum of cnt[0..i) for i <= n (off[n] = the total), one block over tiles of
// kScanThreads·kScanItems counts: each tile is loaded coalesced (all loads in flight), scanned
// and stored, the running total carried to the next tile
__global__ void __launch_bounds__(kScanThreads) scan_counts_kernel(const uint32_t* __restrict__ cnt, uint64_t n,
                                                                   uint64_t* __restrict__ off) {
    using Load = cub::BlockLoad<uint32_t, kScanThreads, kScanItems, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
    using Store = cub::BlockStore<uint64_t, kScanThreads, kScanItems, cub::BLOCK_STORE_WARP_TRANSPOSE>;
    using Scan = cub::BlockScan<uint64_t, kScanThreads>;
    __shared__ union {
        typename Load::TempStorage load;
        typename Store::TempStorage store;
        typename Scan::TempStorage scan;
    } tmp;
    constexpr uint64_t kTile = (uint64_t)kScanThreads * kScanItems;
    uint64_t carry = 0;
    for (uint64_t base = 0; base < n; base += kTile) {
        const int valid = (int)(n - base < kTile ? n - base : kTile);
        uint32_t v[kScanItems];
        Load(tmp.load).Load(cnt + base, v, valid, 0u);
        __syncthreads();
        uint64_t w[kScanItems];
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) w[i] = v[i];
        uint64_t tot;
        Scan(tmp.scan).ExclusiveSum(w, w, tot);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) w[i] += carry;
        Store(tmp.store).Store(off + base, w, valid);
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[n] = carry;
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
// one warp per query: its block by a search of m.lo, its offset and count from the gathered
// block-relative offsets, then the row copy
__global__ void __launch_bounds__(256) unpack_blocks_kernel(const uint2* __restrict__ dense,
                                                            const uint64_t* __restrict__ v, const BlockMap m,
                                                            uint64_t n, uint32_t stride, uint2* __restrict__ rows,
                                                            uint32_t* __restrict__ cnt) {
    const uint64_t q = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= n) return;
    uint32_t g = 0;
    while (g + 1 < m.G && m.lo[g + 1] <= q) ++g;
    const uint64_t a = v[q], b = q + 1 < m.lo[g + 1] ? v[q + 1] : m.vend[g];
    const uint32_t c = (uint32_t)(b - a);
    const uint2* d = dense + m.base[g] + a;
    uint2* row = rows + q * (uint64_t)stride;
    for (uint32_t i = threadIdx.x & 31; i < c; i += 32) row[i] = d[i];
    if ((threadIdx.x & 31) == 0) cnt[q] = c;
}

// One warp per query (eight per CTA, no block barriers): the warp stages its query in shared
// memory, then walks the parts, lane l computing centroids l, l + 32, ... of each (k1 = 32: the
// centroid loads and the LUT stores are 128-byte coalesced rows; no index division).
constexpr uint32_t kLutWarps = 8;
// FD, K1: compile-time part width and centroid count (0: read from p), so the inner loop's loads
// sit at immediate offsets from one base
template <int FD, int K1>
__global__ void __launch_bounds__(kLutWarps * 32) fine_lut_kernel(DevParams p, const float* __restrict__ Q, uint64_t nq,
                                                                   float* __restrict__ fine) {
    extern __shared__ float ys[];  // [kLutWarps][D]
    const uint32_t L = p.L, k1 = K1 ? (uint32_t)K1 : p.k1, fd = FD ? (uint32_t)FD : p.fd, D = p.D;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t q = (uint64_t)blockIdx.x * kLutWarps + warp;
    if (q >= nq) return;
    float* y = ys + (size_t)warp * D;
    for (uint32_t t = lane; t < D; t += 32) y[t] = __ldg(Q + q * D + t);
    __syncwarp();
    float* out = fine + q * L * k1;
    const float* cf = p.fine_t;
    for (uint32_t f = 0; f < L; ++f, cf += fd * k1, out += k1) {
        const float* yf = y + f * fd;
        for (uint32_t i = lane; i < k1; i += 32) {
            const float* c = cf + i;
            float acc = 0.0f;
#pragma unroll
            for (uint32_t t = 0; t < (FD ? (uint32_t)FD : fd); ++t) acc = sq_step(acc, yf[t], __ldg(c + t * k1));
            out[i] = acc;
        }
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
    const uint64_t grid = (nq + kLutWarps - 1) / kLutWarps;
    const size_t sm = (size_t)kLutWarps * p.D * sizeof(float);
    auto run = [&](auto kernel) {
        if (sm > 48 * 1024) {
            int d = 0, optin = 0;
            PQTG_CUDA_CHECK(cudaGetDevice(&d));
            PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d));
            if (sm > (size_t)optin) throw Error{PQTG_ERR_UNSUPPORTED, "fine LUT: query does not fit shared memory"};
            PQTG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        }
        kernel<<<(unsigned)grid, kLutWarps * 32, sm, s>>>(p, queries, nq, fine);
    };
    if (p.fd == 4 && p.k1 == 32) run(fine_lut_kernel<4, 32>);
    else if (p.fd == 4 && p.k1 == 16) run(fine_lut_kernel<4, 16>);
    else run(fine_lut_kernel<0, 0>);
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

void launch_unpack_blocks(const uint2* dense, const uint64_t* v, const BlockMap& m, uint64_t n, uint32_t stride,
                          uint2* rows, uint32_t* cnt, cudaStream_t s) {
    if (n == 0) return;
    unpack_blocks_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(dense, v, m, n, stride, rows, cnt);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

void launch_unpack_ranges(const uint2* dense, const uint32_t* cnt, const uint64_t* off, uint64_t n, uint32_t stride,
                          uint2* ranges, cudaStream_t s) {
    if (n == 0) return;
    move_ranges_kernel<false><<<(unsigned)((n + 7) / 8), 256, 0, s>>>(ranges, stride, cnt, off, const_cast<uint2*>(dense), n);
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
