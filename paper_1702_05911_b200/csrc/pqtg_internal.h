// pqtg_internal.h — device index layout, workspace and kernel launch interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pqtg.h"

namespace pqtg {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
const char* last_error();

struct Error {
    int status;
    std::string msg;
};

#define PQTG_CUDA_CHECK(expr)                                                              \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) {                                                           \
            throw ::pqtg::Error{PQTG_ERR_CUDA, std::string(#expr) + ": " +                 \
                                                   cudaGetErrorString(_e)};                \
        }                                                                                  \
    } while (0)

// Kernel launch; with `chain`, as a programmatic dependent of the stream's previous kernel (PDL:
// its CTAs may start while that kernel drains, and call griddep_wait() before reading its
// results); with a cluster shape other than 1x1x1, as thread-block clusters of that shape
template <typename... KArgs, typename... Args>
void launch_kernel_cluster(bool chain, dim3 cluster, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    if (chain) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster.x * cluster.y * cluster.z > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster.x;
        at[n].val.clusterDim.y = cluster.y;
        at[n].val.clusterDim.z = cluster.z;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    PQTG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}


template <typename... KArgs, typename... Args>
void launch_kernel(bool chain, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args&&... args) {
    launch_kernel_cluster(chain, dim3(1, 1, 1), kernel, grid, block, smem, s, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- constants
constexpr uint32_t kSlopeTables = 10;      // binorder.hpp:25
constexpr uint32_t kSlopeOne = 5;          // slope 1.08^0 (binorder.cpp:59-64, :237)
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kPartialFold = 256;    // pair ranks folded when W² > 4096 (binsel_fast.cuh bs_config)

// Everything a kernel needs, passed by value (fits the parameter space).
struct DevParams {
    // config
    uint32_t D, P, k1, k2, w, L, m, fd, per_part, W, npairs, pw, row_bytes;
    uint32_t budget;            // min(candidate_budget, n) (search.cpp:148)
    uint32_t resort;            // resort_bins
    uint64_t H;                 // slots
    uint64_t n;
    uint64_t shard_lo, shard_hi;  // positions re-ranked here
    uint64_t mult[8];           // (k1*k2)^p mod 2^64 (pqtree.cpp:12-21), p < P <= 8
    uint32_t exact_order;       // no slope tables for this P: exact (Dijkstra) order (binorder.cpp:114-167)
    uint32_t tuple_bits;        // exact order: bits per rank in a packed tuple (P · bits <= 64)
    uint64_t total_tuples;      // W^P: stream length (BinStream::total)
    double inv_log108;          // 1 / log(1.08), host glibc value
    double log108;
    uint32_t h_pow2;            // H is a power of two
    uint32_t mod_fast;          // (k1k2)^P < 2^64 and H < 2^32: slot by sum of reduced terms
    // static bin-order streams
    const uint32_t* pair_streams;  // [10][W*W] (a | b << 16), PairCursor order per table
    const uint2* merge;            // [merge_count] (u, v) for P == 4
    const uint32_t* merge16;       // [merge_count] u | v << 16 (W2 <= 65536), or null
    uint64_t merge_fold_end;       // merge entries [0, this) have u, v < kPartialFold
    uint64_t merge_count;
    uint64_t merge_row0;           // first closed-form sweep row
    uint64_t W2;
    // arrays
    const float* fine_t;        // [L][fd][k1]
    const float* l2_t;          // [P][k1][m][k2]
    const uint32_t* pairs;      // [npairs] (i | j << 16)
    const float* c2;            // [L][npairs]  d2[f][i][j] per pair
    const uint32_t* bitmap;     // [ceil(H / 32)] non-empty slots
    const uint32_t* bitmap_coarse;  // 1 bit per 2^coarse_shift slots (sparse slots only), or null
    uint32_t coarse_shift;
    const uint32_t* offsets;    // [H + 1] u32
    const uint32_t* ids;        // [shard positions]
    const uint8_t* codes;       // [shard positions][row_bytes]
    uint32_t code_ij;           // 1-byte codes hold i << 4 | ((i + j) & 15) instead of the pair id (k1 <= 16)
    uint32_t code_pi;           // 2-byte codes hold pid | i << 9 (16 < k1 <= 32)
    // code_pi on a position shard holding <= 1/4 of the lists (the re-rank's DIRECT mode): the
    // 2-byte codes hold v = i | j << 5 instead, so the re-rank reads fine[f][j] and c2 by v
    // without a pair-table lookup
    uint32_t code_j;
    const float* c2v;           // [L][1024] d2[f][i][j] at i | j << 5 (code_j only)
    const float* c2ij;          // [L][256] d2[f][i][j] at the pair's slot t (code_ij only)
    // code_ij with a per-part bank map (index_prep.cpp bank_map): slot t = i << 4 | n_f(pair) and
    // [L][npairs] (c2 bits, t) for the re-rank's table build, [L][256] j of slot t for the generic
    // kernel; null: the fixed slot i << 4 | ((i + j) & 15)
    const uint2* c2slot;
    const uint8_t* jt_ij;
    const float* c2p;           // [L][512] d2[f][pair] (code_pi only)
    // exact re-rank (search.cpp:229-249): raw vectors n × D f32 in id order, or null
    const float* db;            // [n][db_stride] by id; on a position shard [shard rows][db_stride] by position
    const uint32_t* id2row;     // shard only: id -> row of db (0xFFFFFFFF: not in this shard), else null
    uint32_t db_stride;         // D rounded up to 4 floats
    uint32_t rerank_exact;
    // tensor-core level-2 screen (screen.cu)
    const float* scr_c;         // [P][scr_nj][scr_kpad] children minus their parent: c'' = c - mu_i
    const float* scr_mu;        // [P][scr_kpad] the part's mean child mu_p (query centring)
    const float* scr_cn;        // [P][scr_nj] |c''|^2
    const float* scr_kc;        // [P][scr_nj] (mu_i - mu_p) . c''
    uint32_t scr_nj, scr_kpad;  // k1·k2 padded to the N tile; m padded to 16
    // per-query stage clock of the current chunk ([q][3][~start, end] ns), null when not collected
    unsigned long long* qtime;
    // the chunk's stages run as one programmatic-dependent chain (PDL): bin selection and the
    // re-rank (and the exact stage) are launched as dependents of the previous stage's kernel
    uint32_t chain;
    // the split re-rank's slices of a query form one thread-block cluster: the lists meet in
    // distributed shared memory instead of global memory (set per launch, rerank_ij.cu)
    uint32_t split_cluster;
};

struct DevIndex {
    pqtg_config cfg{};
    uint64_t n = 0;
    int device = 0;
    DevParams prm{};
    uint64_t bytes = 0;
    std::vector<void*> allocations;
    float* db = nullptr;  // attached raw vectors (pqtg_index_attach_database)
    uint32_t* id2row = nullptr;  // a shard's id -> db row table (n entries)
    ~DevIndex();
};

// Per-query intermediate buffers of one contiguous group of queries (a workspace slice).
struct WsSlice {
    float* fine = nullptr;        // [q][L][k1]
    float* l2_dist = nullptr;     // [q][P][W]
    uint32_t* l2_code = nullptr;  // [q][P][W]
    uint8_t* slope = nullptr;     // [q][2]
    uint2* ranges = nullptr;      // [q][budget]
    uint32_t* nranges = nullptr;
    uint32_t* ncand = nullptr;
    uint32_t* ntuples = nullptr;
    uint32_t* hash = nullptr;     // [q][hash_stride] visited-slot table (binsel_fast.cu)
    float* scr = nullptr;         // [q][P][scr_nj] tensor-core dot products (screen.cu)
    uint32_t* err = nullptr;      // the workspace's device error word (PQTG_WS_ERR_*), shared by all slices
    uint64_t* keys = nullptr;     // [q][budget] candidate keys when they do not fit shared memory, or null
    uint64_t* bscr = nullptr;     // [q][binsel_scratch_stride] generic bin selection scratch, or null
    // small batches: the split re-rank's per-(query, slice) top-k keys [q][kSplitMax][split_k], their
    // counts [q][kSplitMax] and per-query arrival counters [q] (zero between calls)
    uint64_t* split_keys = nullptr;
    uint32_t* split_ctr = nullptr;
    uint64_t split_q = 0, split_k = 0;
};

constexpr uint64_t kChainBelow = 256;  // chunks below this many queries run as one PDL chain
constexpr uint32_t kSplitMax = 16;     // CTAs per query of the split re-rank (< 32: one warp scans the counts)
constexpr uint64_t kSplitBelow = 148;  // batches below one query per SM spread each query over CTAs

// device error word bits (Workspace::err): set by kernels, cleared at the start of every search
// call, reported by pqtg_search / pqtg_workspace_status / pqtg_workspace_stage_ms
constexpr uint32_t PQTG_WS_ERR_HEAP = 1u;  // exact bin order: a query's tuple heap outgrew shared memory

struct Workspace {
    const DevIndex* index = nullptr;
    uint64_t max_batch = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t last_stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t last_nq = 0;
    // per-query intermediates
    float* fine = nullptr;        // [B][L][k1]
    float* l2_dist = nullptr;     // [B][P][W]
    uint32_t* l2_code = nullptr;  // [B][P][W]
    uint8_t* slope = nullptr;     // [B][2]
    uint2* ranges = nullptr;      // [B][budget] (start position, candidate offset)
    uint32_t* nranges = nullptr;  // [B]
    uint32_t* ncand = nullptr;    // [B]
    uint32_t* ntuples = nullptr;  // [B] stream tuples consumed by the gather
    uint32_t* err = nullptr;      // [1] device error word (PQTG_WS_ERR_*)
    uint64_t* keys = nullptr;     // [B][budget] re-rank keys for budgets too large for shared memory
    unsigned long long* qtime = nullptr;  // [B][3][2] per-query stage clock (pqtg_workspace_query_times)
    unsigned long long* h_qtime = nullptr;  // pinned [qtime_cap][6]: the last pqtg_search call's clocks
    uint64_t qtime_cap = 0;
    bool qtime_on = false;
    bool qtime_host = false;              // the last call was pqtg_search (clocks in h_qtime)
    uint64_t* split_keys = nullptr;   // small-batch split re-rank lists (see WsSlice)
    uint32_t* split_ctr = nullptr;
    uint64_t split_q = 0, split_k = 0;
    float* scr = nullptr;         // [B][P][scr_nj] (y - mu_p) . c'' on the tensor cores (screen.cu)
    uint32_t* hash = nullptr;     // [B << ts_log2] visited slots, cleared on use (binsel_fast.cu)
    uint64_t hash_words = 0;
    uint64_t hash_stride = 0;     // words per query
    uint64_t* bscr = nullptr;     // [B][bscr_stride] (binsel_scratch_stride), or null
    uint64_t bscr_stride = 0;
    cudaStream_t aux_stream = nullptr;  // second stream of the pipelined searches
    uint32_t chunks = 0;                // sub-batch chunks per search (0 = automatic)
    cudaEvent_t join = nullptr;
    cudaEvent_t fork = nullptr;         // graph capture: brings aux_stream into the capture
    cudaEvent_t done = nullptr;         // the end of the last call's work on its stream: the next call
                                        // (any stream, either entry point) starts after it
    // pqtg_search replays: CUDA graphs of whole host-buffer searches, keyed by their arguments
    struct GraphEntry {
        uint64_t key[12];
        cudaGraphExec_t exec;
        uint64_t used;
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    uint64_t dev_last_key[12] = {};     // pqtg_search_device: a small batch is captured the second
                                        // time the same arguments arrive in a row
    uint64_t gen = 0;                   // bumped when buffers / settings a graph bakes in change
    bool stages_timed = true;           // the last timed chunk recorded events between its stages
    WsSlice slice(uint64_t q0) const;
    // host-call staging (grown on demand)
    float* d_queries = nullptr;
    uint32_t* d_ids = nullptr;
    float* d_dists = nullptr;
    uint32_t* d_counts = nullptr;
    pqtg_query_stats* d_stats = nullptr;
    uint64_t stage_k = 0;
    // line-ranked prefix feeding the exact re-rank (grown on demand): [max_batch][ex_k]
    uint32_t* ex_ids = nullptr;
    float* ex_dists = nullptr;
    uint32_t* ex_counts = nullptr;
    uint64_t ex_k = 0;    // row stride (k') of the current search
    uint64_t ex_cap = 0;  // rows' capacity in entries per query
    std::mutex mu;
    std::vector<void*> allocations;
    ~Workspace();
};

// ---------------------------------------------------------------- host helpers
template <class T>
T* dev_alloc(std::vector<void*>& owner, uint64_t count, uint64_t* bytes = nullptr) {
    void* p = nullptr;
    size_t sz = count * sizeof(T);
    if (sz == 0) sz = 16;
    cudaError_t e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
        throw Error{PQTG_ERR_OOM, "cudaMalloc(" + std::to_string(sz) + "): " + cudaGetErrorString(e)};
    }
    owner.push_back(p);
    if (bytes) *bytes += sz;
    return static_cast<T*>(p);
}

// Source arrays for building a device index (a view, or a parsed PQTINDEX file).
struct Source {
    pqtg_config cfg{};
    uint64_t n = 0;
    const float* level1 = nullptr;
    const float* level2 = nullptr;
    const float* d2 = nullptr;
    uint32_t table_count = 0, table_len = 0;
    const double* slopes = nullptr;
    const uint32_t* entries = nullptr;
    const uint64_t* offsets = nullptr;
    const uint32_t* ids = nullptr;
    // line codes: SoA (view) or interleaved records (file: (lambda, pair) per record)
    const uint8_t* lambda_q = nullptr;
    const uint16_t* pair_id = nullptr;
    const uint8_t* records = nullptr;
    // or the shard's codes in position order (pqtg_index_create_shard)
    const uint8_t* pos_lambda_q = nullptr;
    const uint16_t* pos_pair_id = nullptr;
    uint32_t record_pw = 0;
};

// Static bin-order streams of one index (host copy; uploaded into DevParams).
struct HostStreams {
    uint32_t W = 0, P = 0;
    uint64_t W2 = 0, total = 0, merge_row0 = 0;
    std::vector<uint32_t> pair;  // [10][W2] (a | b << 16)
    std::vector<uint2> merge;    // P == 4: materialized merge prefix
    void tuple_at(uint64_t s, uint32_t ta, uint32_t tb, uint32_t* ranks) const;
};
HostStreams build_streams(const uint32_t* entries, uint32_t table_len, uint32_t W, uint32_t P);
[[noreturn]] void unsupported(const std::string& m);
[[noreturn]] void format(const std::string& m);

// A PQTINDEX v1 file parsed into a Source (index_file.cpp).
struct MappedFile {
    const uint8_t* base = nullptr;
    size_t size = 0;
    int fd = -1;
    ~MappedFile();
};
struct LoadedFile {
    MappedFile map;
    Source src;
    std::vector<float> level1, level2, d2;
    std::vector<double> slopes;
    std::vector<uint32_t> entries, ids;
    std::vector<uint64_t> offsets;
};
void parse_index(const char* path, LoadedFile& lf);

DevIndex* build_device_index(const Source& src, int device, uint64_t shard_lo, uint64_t shard_hi);
void validate_config(const pqtg_config& c);

// ---------------------------------------------------------------- kernels (kernels.cu)
size_t traverse_smem(const DevParams& p);
size_t binsel_smem(const DevParams& p, bool global_visited = false);
uint64_t binsel_scratch_stride(const DevParams& p);  // u64 words per query of ws.bscr (0: none)
size_t rerank_smem(const DevParams& p, uint32_t k, bool gkeys = false);
void launch_traverse(const DevParams& p, const float* queries, uint64_t nq, const WsSlice& ws,
                     cudaStream_t s);
void launch_binsel(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats,
                   cudaStream_t s);
void launch_rerank(const DevParams& p, uint64_t nq, uint32_t k, const WsSlice& ws, uint32_t* ids,
                   float* dists, uint32_t* counts, cudaStream_t s);
void launch_merge(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* ids,
                  const float* dists, const uint32_t* counts, uint32_t* out_ids,
                  float* out_dists, uint32_t* out_counts, cudaStream_t s);
void configure_kernels(const DevParams& p, uint32_t k);
// rerank_ij.cu (1-byte (i, j) pair codes, k1 <= 16, p_line in {16, 32, 64})
bool rerank_ij_ok(const DevParams& p, uint32_t k);
// the opt-in re-rank loops that derive j from the fixed slot i << 4 | ((i + j) & 15) (PQTG_RERANK=
// packed / c3): indexes uploaded under them keep the fixed slots (no per-part bank map)
bool rerank_needs_fixed_slots();
bool rerank_ij_gkeys(const DevParams& p, uint32_t k);  // its keys go to the workspace (large budgets)
uint32_t rerank_split(const DevParams& p, uint64_t nq, uint32_t k);  // CTAs per query (1 = no split)
bool rerank_needs_gkeys(const DevParams& p, uint32_t k);  // launch_rerank will use ws.keys
int optin_bytes();  // the device's opt-in shared memory per block
void configure_rerank_ij();
unsigned long long* phase_buffer();  // PQTG_PHASES=1: the re-rank's phase clocks (managed memory), else null
void launch_rerank_ij(const DevParams& p, uint64_t nq, uint32_t k, const WsSlice& ws, uint32_t* ids,
                      float* dists, uint32_t* counts, cudaStream_t s);
// binsel_fast.cu (no resort, 32-bit slot arithmetic)
bool binsel_fast_ok(const DevParams& p);
uint64_t binsel_hash_words(const DevParams& p, uint64_t max_batch);
uint64_t binsel_hash_stride(const DevParams& p);
void configure_binsel_fast();
// brute.cu (exact brute-force k-NN, search.cpp:276-299)
bool brute_force_ok(uint32_t dim, uint32_t k);
void launch_brute_force(const float* d_db, uint64_t n, uint32_t dim, const float* d_queries, uint64_t nq, uint32_t k,
                        uint32_t* d_ids, float* d_dists, uint32_t* d_counts, cudaStream_t s);
// binsel_par.cu (same contract; all warps finish each pass together, no walker warp)
void launch_binsel_par(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats, cudaStream_t s);
uint64_t binsel_par_hash_stride(const DevParams& p);
bool binsel_prefers_walker(const DevParams& p);  // the auto choice between the two
void configure_binsel_par();
void launch_binsel_fast(const DevParams& p, uint64_t nq, const WsSlice& ws, pqtg_query_stats* stats, cudaStream_t s);
// traverse.cu (one CTA per (query, part), TMA-staged level-2 blocks)
bool traverse_part_ok(const DevParams& p);
void configure_traverse_part();
void launch_traverse_part(const DevParams& p, const float* queries, uint64_t nq, const WsSlice& ws,
                          cudaStream_t s);
// exact.cu (exact re-rank of the line-ranked prefix with attached raw vectors)
void configure_exact();
void launch_exact(const DevParams& p, const float* queries, uint64_t nq, uint32_t kp, const uint32_t* line_ids,
                  const uint32_t* line_counts, uint32_t k, uint32_t* ids, float* dists, uint32_t* counts,
                  pqtg_query_stats* stats, cudaStream_t s);
// the exact distances of the whole line-ranked prefix, in its (line, id) order, into exact[q][kp]
// (a position shard's part of the sharded exact stage; no cut, no sort)
void launch_exact_prefix(const DevParams& p, const float* queries, uint64_t nq, uint32_t kp, const uint32_t* line_ids,
                         const uint32_t* line_counts, float* exact, cudaStream_t s);
// the sharded exact stage's merge: G lists of (id, line, exact) sorted by (line, id), counts;
// per query the first min(R, C) by (line, id) over all lists (C = stats.candidates), then the
// first min(k, that) of those by (exact, id) (search.cpp:229-257); exact_evals = min(R, C)
void launch_merge_exact(uint32_t G, uint64_t nq, uint32_t kp, uint32_t R, uint32_t k, const uint32_t* ids,
                        const float* line, const float* exact, const uint32_t* counts, pqtg_query_stats* stats,
                        uint32_t* out_ids, float* out_dists, uint32_t* out_counts, cudaStream_t s);
// id2row[ids[p]] = p for the shard's positions (the table pre-filled with 0xFFFFFFFF)
void launch_fill_id2row(const uint32_t* ids, uint64_t count, uint32_t* id2row, cudaStream_t s);
// screen.cu (tcgen05 level-2 screen + certified exact residual check)
bool screen_ok(const DevParams& p);
void configure_screen();
void launch_screen_gemm(const DevParams& p, const float* queries, uint64_t nq, float* out, cudaStream_t s);
void launch_traverse_screen(const DevParams& p, const float* queries, uint64_t nq, const float* scr,
                            const WsSlice& ws, cudaStream_t s);
// 0 = pick the fastest kernel per stage, 1 = generic kernels only (parity tests run both)
int kernel_variant();
// grow a workspace's k-dependent buffers (exact prefix, HBM candidate keys) before a search
void prepare_workspace(Workspace& ws, uint32_t k);
// sharded_kernels.cu: dense per-query range lists of the query-partitioned sharded search, and
// the batch's fine LUTs recomputed on every rank
void launch_fine_lut(const DevParams& p, const float* queries, uint64_t nq, float* fine, cudaStream_t s);
struct CopySegment {
    void* dst;
    const void* src;
    uint64_t bytes;  // multiple of 4, 4-byte aligned pointers
};
constexpr uint32_t kCopySegmentsMax = 64;
struct CopySegments {
    uint32_t n;
    CopySegment s[kCopySegmentsMax];
};
// device-to-device copies of one device's buffers in one launch per 64 segments
void launch_copy_segments(const std::vector<CopySegment>& segs, cudaStream_t s);
void launch_scan_counts(const uint32_t* cnt, uint64_t n, uint64_t* off, cudaStream_t s);
void launch_pack_ranges(const uint2* ranges, uint32_t stride, const uint32_t* cnt, const uint64_t* off, uint64_t n,
                        uint2* dense, cudaStream_t s);
// The sharded exchange's query blocks (sharded.cpp): queries [lo[g], lo[g+1]) belong to block g;
// v[q] is the gathered offset of q's ranges in its block's packed array, so q's ranges start at
// base[g] + v[q] in the batch's packed array and end at base[g] + v[q + 1] (vend[g] for a block's
// last query)
constexpr uint32_t kMaxBlocks = 64;
struct BlockMap {
    uint32_t G;
    uint64_t lo[kMaxBlocks + 1];
    uint64_t base[kMaxBlocks];
    uint64_t vend[kMaxBlocks];
};
// per-query rows + counts <- the batch's packed ranges, offsets from the blocks' own scans (no
// scan over the batch)
void launch_unpack_blocks(const uint2* dense, const uint64_t* v, const BlockMap& m, uint64_t n, uint32_t stride,
                          uint2* rows, uint32_t* cnt, cudaStream_t s);
void launch_unpack_ranges(const uint2* dense, const uint32_t* cnt, const uint64_t* off, uint64_t n, uint32_t stride,
                          uint2* ranges, cudaStream_t s);

}  // namespace pqtg

struct pqtg_index {
    std::unique_ptr<pqtg::DevIndex> dev;
};

struct pqtg_workspace {
    std::unique_ptr<pqtg::Workspace> ws;
};
