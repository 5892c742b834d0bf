// binsel_fast.cu — K3 fast path: bin selection + gather (binorder.cpp:178-283,
// search.cpp:139-217) without resort_bins, for indexes whose slot arithmetic fits 32 bits.
//
// Per query (one CTA), the heuristic rank-tuple stream is walked in passes of growing size
// (256, 512, ... tuples). Every thread turns its tuples into slots (per-part slot terms
// pre-reduced mod H in shared memory; for P = 4 the two pair streams are folded into
// per-pair-rank terms A[u], B[v] so a tuple costs one merge-entry load) and tests the
// non-empty-slot bitmap. The few non-empty tuples are compacted IN STREAM ORDER into a
// shared queue (ballot + a 1-warp scan of per-warp counts). Warp 0 then walks the queue in
// order, 32 at a time: first occurrences by __match_any_sync within the batch plus a shared
// hash set of visited slots across batches (only when two tuples can share a slot, i.e.
// (k1·k2)^P > H), the offsets of first occurrences, a warp prefix sum of their sizes, and
// the budget cut. Output: one (start position, candidate offset) range per visited bin —
// exactly the reference's gather order.
#include <cstdint>

#include "binsel_fast.cuh"

namespace pqtg {

using namespace dev;

using namespace bsf;

template <int P, bool HASH>
__global__ void __launch_bounds__(kBsThreads, 4)
    binsel_fast_kernel(DevParams p, const uint32_t* __restrict__ l2c_in, const float* __restrict__ l2d_in,
                       uint8_t* __restrict__ slope_out,
                       uint2* __restrict__ ranges, uint32_t* __restrict__ nranges, uint32_t* __restrict__ ncand,
                       uint32_t* __restrict__ ntuples, pqtg_query_stats* __restrict__ stats, uint32_t ts_log2,
                       uint32_t* __restrict__ ghash, uint32_t W2ab) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (p.chain) {  // the traversal's lists (a PDL dependent in a chained chunk)
        griddep_wait();
        griddep_launch();
    }
    qt_begin(p, blockIdx.x, 1);
    binsel_fast_body<P, HASH, SyncBlock>(p, blockIdx.x, l2c_in, l2d_in, slope_out, ranges, nranges, ncand, ntuples,
                                         stats, ts_log2, ghash, W2ab, smem, threadIdx.x);
    qt_end(p, blockIdx.x, 1);
}

namespace {

template <int P, bool HASH>
void configure_one() {
    int dev = 0, optin = 0;
    PQTG_CUDA_CHECK(cudaGetDevice(&dev));
    PQTG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a{};
    PQTG_CUDA_CHECK(cudaFuncGetAttributes(&a, binsel_fast_kernel<P, HASH>));
    PQTG_CUDA_CHECK(cudaFuncSetAttribute(binsel_fast_kernel<P, HASH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         optin - (int)a.sharedSizeBytes));
}

}  // namespace

bool binsel_fast_ok(const DevParams& p) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const BsConfig c = bs_config(p);
    return !p.resort && !p.exact_order && p.mod_fast && p.H < 0xFFFFFFFFull && (!c.use_hash || p.H <= (1ull << 26)) &&
           c.smem + 2048 <= (size_t)optin;
}

bool binsel_prefers_walker(const DevParams& p) {
    return p.P == 4 && p.W2 <= 4096;  // the whole pair-stream grid folded (GIST1M-shaped)
}

uint64_t binsel_hash_words(const DevParams& p, uint64_t max_batch) {
    const BsConfig c = bs_config(p);
    return c.use_hash ? (max_batch << c.ts_log2) : 0;
}

uint64_t binsel_hash_stride(const DevParams& p) {
    const BsConfig c = bs_config(p);
    return c.use_hash ? (1ull << c.ts_log2) : 0;
}

void configure_binsel_fast() {
    configure_one<1, false>();
    configure_one<2, false>();
    configure_one<2, true>();
    configure_one<4, false>();
    configure_one<4, true>();
}

void launch_binsel_fast(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats, cudaStream_t s) {
    const BsConfig c = bs_config(p);
#define PQTG_BS(PP, HH)                                                                                       \
    launch_kernel(p.chain, binsel_fast_kernel<PP, HH>, dim3((unsigned)nq), dim3(kBsThreads), c.smem, s, p, ws.l2_code, ws.l2_dist, ws.slope, ws.ranges,     \
                                                                       ws.nranges, ws.ncand, ws.ntuples, stats, \
                                                                       c.ts_log2, ws.hash, c.W2ab)
    if (p.P == 1) {
        PQTG_BS(1, false);
    } else if (p.P == 2) {
        if (c.use_hash) PQTG_BS(2, true); else PQTG_BS(2, false);
    } else {
        if (c.use_hash) PQTG_BS(4, true); else PQTG_BS(4, false);
    }
#undef PQTG_BS
    PQTG_CUDA_CHECK(cudaGetLastError());
}

}  // namespace pqtg
