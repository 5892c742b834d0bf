/*
 * pqtg.h — C ABI of the B200 (sm_100a) query path for the Product Quantization Tree.
 *
 * This is the drop-in boundary. Plain pointers and sizes only; no C++ or torch types.
 * Each entry point names the reference interface it replaces (paths relative to
 * the reference checkout, proj/…):
 *
 *   pqtg_index_load          ← pqt::load_index            include/pqt/index_io.hpp:16, src/index_io.cpp:148-229
 *   pqtg_index_create        ← constructing pqt::PqtIndex  include/pqt/search.hpp:34-47 (build_index /
 *                              IndexBuilder::finalize output, src/search.cpp:93-124)
 *   pqtg_search              ← pqt::knn_query_batch        include/pqt/search.hpp:83, src/search.cpp:262-274
 *                              (each row = pqt::knn_query, src/search.cpp:126-260)
 *   pqtg_search_device       ← same, device-resident inputs/outputs on a caller stream
 *   pqtg_index_attach_database ← pqt::PqtIndex::attach_database  include/pqt/search.hpp:53,
 *                              src/search.cpp:44-49 (enables the exact re-rank, :229-249)
 *   pqtg_merge_topk_host     ← no reference counterpart: merges per-shard top-k lists by the
 *                              reference's (dist, id) order (candidate_less, src/search.cpp:39-41)
 *   pqtg_sharded_*           ← pqt::knn_query_batch (src/search.cpp:262-274) over G position shards,
 *                              one process per GPU, query-partitioned, NCCL (no reference counterpart)
 *   pqtg_brute_force_knn     ← pqt::brute_force_knn        include/pqt/search.hpp:86, src/search.cpp:276-299
 *
 * Errors: every int-returning call returns PQTG_OK (0) or a negative pqtg_status; the message
 * is available from pqtg_last_error() (thread-local). The C++ drop-in (include/pqt/) maps
 * PQTG_ERR_BAD_DIM / PQTG_ERR_CONFIG to std::invalid_argument and PQTG_ERR_FORMAT to
 * pqt::FormatError, like the reference (src/search.cpp:264-266, src/codebook.cpp:15-35,
 * src/index_io.cpp:28-42,155-165,211-213).
 *
 * There is no CPU fallback: configurations the GPU path does not implement (p_tree > 8; an
 * exact-order tuple wider than 64 bits; an exact Dijkstra-order frontier larger than the
 * shared-memory heap -- src/binorder.cpp:114-167, used for p_tree not in {1,2,4} or without
 * slope tables; a candidate budget above 65535) return PQTG_ERR_UNSUPPORTED. resort_bins runs at
 * every budget up to that (batches longer than 4096 tuples are sorted through the workspace).
 */
#ifndef PQTG_H
#define PQTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQTG_ABI_VERSION 1

typedef enum pqtg_status {
    PQTG_OK = 0,
    PQTG_ERR_BAD_DIM = -1,      /* query dim != index dim (search.cpp:264-266) */
    PQTG_ERR_CONFIG = -2,       /* PqtConfig::validate failure (codebook.cpp:15-35) */
    PQTG_ERR_FORMAT = -3,       /* malformed PQTINDEX container (index_io.cpp) */
    PQTG_ERR_UNSUPPORTED = -4,  /* valid for the reference, not implemented on the GPU path */
    PQTG_ERR_OOM = -5,
    PQTG_ERR_CUDA = -6,
    PQTG_ERR_ARG = -7,          /* null pointer / bad size from the caller */
    PQTG_ERR_NCCL = -8
} pqtg_status;

/* Mirrors pqt::PqtConfig (include/pqt/codebook.hpp:12-36) field for field.
 * hash_size is the RESOLVED slot count H (search.cpp:106 stores it resolved). */
typedef struct pqtg_config {
    uint32_t dim;
    uint32_t p_tree;
    uint32_t k1;
    uint32_t k2;
    uint32_t w;
    uint32_t p_line;
    uint64_t hash_size;
    uint32_t candidate_budget;
    uint32_t rerank_exact;
    uint32_t resort_bins;       /* bool in the reference; 0/1 here */
    uint32_t train_iters;
    uint64_t seed;
} pqtg_config;

/* Borrowed host view of everything pqt::PqtIndex holds that the query path reads
 * (include/pqt/search.hpp:34-47). Array layouts are the reference's in-memory layouts:
 *   level1      p_tree × k1 × m            (TreeCodebooks::level1[p].centroids, concatenated)
 *   level2      p_tree × k1 × k2 × m       (TreeCodebooks::level2[p][i].centroids, concatenated)
 *   d2          p_line × k1 × k1           (PairDistanceTable::d2 — as stored in the index file)
 *   tables      table_count × table_len × (a, b)  plus one slope per table (OrderTable)
 *   offsets     hash_size + 1              (InvertedLists::offsets)
 *   ids         n                          (InvertedLists::ids)
 *   lambda_q    n × p_line                 (LineCodes::lambda_q, vector-id order)
 *   pair_id     n × p_line                 (LineCodes::pair_id, vector-id order)
 * m = dim / p_tree.
 *
 * shard_lo/shard_hi select the range of inverted-list POSITIONS (indices into ids[]) whose
 * line codes this device holds and re-ranks; 0/0 means all of [0, n). Traversal and bin
 * selection always run over the full replicated offsets, so bins_visited / candidates stay
 * global and per-shard top-k lists merge bit-exactly (pqtg_merge_topk_host). */
typedef struct pqtg_index_view {
    pqtg_config config;
    uint64_t n;
    const float* level1;
    const float* level2;
    const float* d2;
    uint32_t table_count;
    uint32_t table_len;
    const double* table_slopes;
    const uint32_t* table_entries;
    const uint64_t* offsets;
    const uint32_t* ids;
    const uint8_t* lambda_q;
    const uint16_t* pair_id;
    uint64_t shard_lo;
    uint64_t shard_hi;
} pqtg_index_view;

/* Per-query counters of pqt::QueryStats (include/pqt/search.hpp:15-23). The reference's
 * *_us wall-clock timers have no per-query meaning on a batched GPU; per-stage batch times
 * come from pqtg_workspace_stage_ms. exact_evals = min(max(rerank_exact, k), C) when raw vectors
 * are attached (pqtg_index_attach_database) and rerank_exact > 0, else 0 (as for an index from
 * load_index, search.cpp:229-238). */
typedef struct pqtg_query_stats {
    uint64_t bins_visited;
    uint64_t candidates;
    uint64_t exact_evals;
} pqtg_query_stats;

typedef struct pqtg_index_info {
    pqtg_config config;
    uint64_t n;
    uint64_t shard_lo, shard_hi;
    uint32_t list_len;          /* W = w * k2, entries per part in the level-2 list */
    uint32_t pair_count;        /* k1(k1-1)/2, or 1 when k1 == 1 */
    uint32_t pair_width;        /* 1 or 2 bytes per stored pair id (index_io.cpp:132) */
    uint32_t code_row_bytes;    /* device bytes per line-code row (slot order) */
    uint64_t device_bytes;      /* device memory owned by the index */
    int device;
} pqtg_index_info;

typedef struct pqtg_index pqtg_index;
typedef struct pqtg_workspace pqtg_workspace;

/* ---- library ---------------------------------------------------------------------- */
int pqtg_abi_version(void);
const char* pqtg_last_error(void);
/* Kernel selection, process-wide: 0 = fastest kernel for each stage (default), 1 = the generic
 * kernels only, 2 = the fast kernels with the level-2 distances screened on the tensor cores
 * (tcgen05) and an exact fp32 residual check (screen.cu), 3 / 4 = the fast kernels with the
 * walker-warp bin selection (binsel_fast.cu) / the all-warp one (binsel_par.cu) forced (0 picks
 * per index). The parity tests run all five; search results are identical by construction. */
int pqtg_set_kernel_variant(int variant);
/* 1 when a CUDA device with compute capability 10.x is usable, else 0. */
int pqtg_device_ok(int device);

/* ---- index ------------------------------------------------------------------------ */
/* Copy a host index view to `device` (re-laid out for the kernels; the caller keeps
 * ownership of the view arrays). Validates like PqtConfig::validate. */
int pqtg_index_create(const pqtg_index_view* view, int device, pqtg_index** out);
/* Parse a PQTINDEX v1 file (index_io.cpp:148-229 format) and upload it; shard_lo/hi as in
 * the view (0/0 = whole index). */
int pqtg_index_load(const char* path, int device, uint64_t shard_lo, uint64_t shard_hi,
                    pqtg_index** out);
int pqtg_index_info_get(const pqtg_index* index, pqtg_index_info* out);
/* One position shard [view->shard_lo, view->shard_hi) of an index whose ids and line codes were
 * never gathered on one host (a sharded billion-scale build): view->ids points to the SHARD's ids
 * (positions shard_lo..shard_hi-1, in order), view->lambda_q / pair_id are not read, and the
 * shard's codes come in position order (shard_lambda_q, shard_pair_id: (shard_hi - shard_lo) ×
 * p_line each). offsets and the codebooks are the whole index's.
 * The device index is identical to pqtg_index_create on the full view with the same range. */
int pqtg_index_create_shard(const pqtg_index_view* view, const uint8_t* shard_lambda_q,
                            const uint16_t* shard_pair_id, int device, pqtg_index** out);
/* pqt::PqtIndex::attach_database (src/search.cpp:44-49): copy n × dim float32 raw vectors
 * (vector-id order, row-major) to the index's device. Searches then run the exact re-rank
 * stage when config.rerank_exact > 0 (src/search.cpp:229-249): the min(max(rerank_exact, k), C)
 * best candidates by line distance get l2_sq(row, y) distances in the reference's fp32 order
 * and are re-sorted by (dist, id). rows == NULL detaches. A mismatched n or dim returns
 * PQTG_ERR_BAD_DIM (std::invalid_argument in the reference). A position shard takes its own
 * rows, n = shard_hi - shard_lo in position order (db[ids[shard_lo..shard_hi)]); its exact stage
 * then runs in the sharded search (pqtg_sharded_*), and pqtg_search on it returns
 * PQTG_ERR_UNSUPPORTED. Not safe to call concurrently with a search on the same index. */
int pqtg_index_attach_database(pqtg_index* index, const float* rows, uint64_t n, uint32_t dim);
void pqtg_index_destroy(pqtg_index* index);

/* ---- workspace (per stream; not shared by concurrent searches) -------------------- */
int pqtg_workspace_create(const pqtg_index* index, uint64_t max_batch, pqtg_workspace** out);
void pqtg_workspace_destroy(pqtg_workspace* ws);
/* Split each (sub-)batch into `chunks` pieces that alternate between two streams so one
 * piece's re-rank overlaps the next piece's traversal / bin selection (and, in pqtg_search, the
 * copies). 0 = automatic (2 from 256 queries; 4 for host batches from 4096), 1 = no overlap.
 * Results are identical. Calls on one workspace serialise on its lock (host) and on the device:
 * each call's work starts after the previous call's (any stream, either entry point). Use one
 * workspace per concurrent caller. */
int pqtg_workspace_set_chunks(pqtg_workspace* ws, uint32_t chunks);
/* Device milliseconds of the last pqtg_search* call per stage: [0] traversal, [1] bin
 * selection + gather, [2] re-rank + top-k, [3] whole search — of the call's first chunk (see
 * pqtg_workspace_set_chunks). A chunk below 256 queries runs its stages as one programmatic-
 * dependent (PDL) chain with no events between them: [0..2] are then -1 and [3] is the whole
 * search (pqtg_workspace_query_times has per-stage clocks). Synchronises the last stream. */
int pqtg_workspace_stage_ms(pqtg_workspace* ws, float* ms4);
/* Synchronise the workspace's streams and report what the kernels of its last search call
 * flagged: PQTG_ERR_UNSUPPORTED when a query's exact-order tuple heap outgrew shared memory
 * (that query's candidate list is truncated). pqtg_search checks this itself; a caller of the
 * asynchronous pqtg_search_device checks it here (pqtg_workspace_stage_ms reports it too). */
int pqtg_workspace_status(pqtg_workspace* ws);
/* Per-query stage clocks -- the GPU counterpart of the reference's per-query timers
 * (QueryStats::traversal_us / bin_selection_us / vector_proposal_us / rerank_us,
 * src/search.cpp:134-137,167-216,220,258): with them enabled, each query's traversal, bin
 * selection + gather and re-rank (+ exact) kernels record the first start and the last end of
 * their CTAs for that query (globaltimer). pqtg_workspace_read_query_times gives, for the last
 * call's queries (pqtg_search: all sub-batches; pqtg_search_device: its batch), nq × 3 stage
 * durations in microseconds. A query's stage duration is its CTAs' wall time on the device, with
 * the batch's other queries running beside it. */
int pqtg_workspace_query_times(pqtg_workspace* ws, int enable);
/* Diagnostic: phase clocks (ns) of the re-rank's first CTA in its last launch -- start, prologue,
 * range map, candidates scored, selected, written, merged (split) -- when the process started with
 * PQTG_PHASES=1 (tools/phase_probe.py); PQTG_ERR_ARG otherwise. */
int pqtg_debug_rerank_phases(uint64_t* out16);
/* Diagnostic: the raw per-query stage clocks of the last pqtg_search_device call (globaltimer
 * ns, nq x 3 stages x [start, end]) when per-query times are on. */
int pqtg_debug_query_clocks(pqtg_workspace* ws, uint64_t nq, uint64_t* out);
int pqtg_workspace_read_query_times(pqtg_workspace* ws, uint64_t nq, float* us3);
/* Copy per-query intermediates of the LAST sub-batch searched with `ws` to host buffers
 * (any pointer may be NULL). Used by the per-stage parity tests.
 *   fine         nq × p_line × k1              traversal fine_dists (pqtree.cpp:84-97)
 *   l2_code      nq × p_tree × W  (parent << 16 | child)   sorted level-2 lists (pqtree.cpp:102-117)
 *   l2_dist      nq × p_tree × W
 *   slope        nq × 2           picked slope-table indices (binorder.cpp:52-65)
 *   positions    nq × budget      gathered candidate positions (search.cpp:166-217), in order
 *   ncand        nq               candidates gathered (global count)
 *   ntuples      nq               bin-order tuples the gather consumed (T_q) */
int pqtg_workspace_read(pqtg_workspace* ws, uint64_t nq, float* fine, uint32_t* l2_code,
                        float* l2_dist, uint8_t* slope, uint32_t* positions, uint32_t* ncand,
                        uint32_t* ntuples);

/* ---- search ----------------------------------------------------------------------- */
/* Host buffers (copied in and out inside the call); synchronous. Outputs are nq × k
 * row-major; counts[q] = min(k, candidates) valid entries (the reference's short results,
 * search.cpp:251). stats may be NULL. dim must equal the index dim (else BAD_DIM). With
 * page-locked host buffers the whole chunked copy/kernel sequence is recorded once per argument
 * set as a CUDA graph and replayed (PQTG_NO_GRAPH=1 disables). */
int pqtg_search(pqtg_index* index, pqtg_workspace* ws, const float* queries, uint64_t nq,
                uint32_t dim, uint32_t k, uint32_t* ids, float* dists, uint32_t* counts,
                pqtg_query_stats* stats);
/* Device pointers, asynchronous on `stream` (a cudaStream_t; NULL = legacy default).
 * nq must be <= the workspace max_batch. */
int pqtg_search_device(pqtg_index* index, pqtg_workspace* ws, const float* d_queries,
                       uint64_t nq, uint32_t k, uint32_t* d_ids, float* d_dists,
                       uint32_t* d_counts, pqtg_query_stats* d_stats, void* stream);

/* Host twin of the kernels' bin-order addressing (test hook; needs no GPU). Materializes the
 * static slope-table streams of `view` exactly as the device index does and writes the first
 * max_tuples rank tuples (p_tree entries each) of the heuristic order for the sorted per-part
 * lists `lists` (p_tree × w·k2) — BinStream (binorder.cpp:178-283). The slope pick here uses
 * the host libm (the GPU uses CUDA's fp64 log). Returns the tuple count or a negative status. */
int64_t pqtg_bin_stream_host(const pqtg_index_view* view, const float* lists, uint64_t max_tuples,
                             uint32_t* out);

/* ---- offline build on the GPU -------------------------------- */
/* For n database vectors d_x (n × dim, device) compute, in the reference's exact fp32 order:
 *   d_part_codes  n × p_tree   flat per-part bin code i1*k2+i2   (assign_bin, pqtree.cpp:27-38)
 *   d_slots       n            global_code % hash_size (global_code when hash_size == 0)
 *                                                                (pqtree.cpp:12-25)
 *   d_lambda/d_pair n × p_line line codes                         (encode_line, linequant.cpp:84-152)
 * Codebooks are device arrays in the view layouts (level1, level2); d_fine is the p_line × k1 ×
 * fine_dim slice table, d_fine_sq its |slice|^2 (linequant.cpp:13-46), d_d2 the pair table
 * (linequant.cpp:60-75). Asynchronous on `stream`. */
/* (d_part_codes, d_slots) NULL: skip the bins; (d_lambda, d_pair) NULL: skip the line codes. */
int pqtg_build_codes(const pqtg_config* cfg, const float* d_level1, const float* d_level2,
                     const float* d_fine, const float* d_fine_sq, const float* d_d2, const float* d_x,
                     uint64_t n, uint32_t* d_part_codes, uint64_t* d_slots, uint8_t* d_lambda,
                     uint16_t* d_pair, void* stream);

/* ---- multi-GPU helpers ------------------------------------------------------------ */
/* Merge G per-shard top-k lists (each nq × k, counts per query) into the global top-k by
 * ascending (dist, id). Host-side; inputs laid out shard-major: ids[g][q][k]. */
int pqtg_merge_topk_host(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* ids,
                         const float* dists, const uint32_t* counts, uint32_t* out_ids,
                         float* out_dists, uint32_t* out_counts);
/* Same on device, asynchronous on `stream`. */
int pqtg_merge_topk_device(uint32_t shards, uint64_t nq, uint32_t k, const uint32_t* d_ids,
                           const float* d_dists, const uint32_t* d_counts, uint32_t* d_out_ids,
                           float* d_out_dists, uint32_t* d_out_counts, void* stream);
/* Even split of [0, n) into `shards` position ranges (the shard_lo/shard_hi to pass). */
int pqtg_shard_range(uint64_t n, uint32_t shards, uint32_t rank, uint64_t* lo, uint64_t* hi);

/* ---- sharded search over G GPUs ------------------------------------
 * The billion-scale deployment of pqt::knn_query_batch (src/search.cpp:262-274): the inverted
 * lists' positions are split into G contiguous ranges (pqtg_shard_range), shard g holds the
 * whole index's small state plus its range's ids and codes (pqtg_index_load with the range,
 * or pqtg_index_create_shard). A search is query-partitioned end to end:
 *   1. rank g runs traversal + bin selection for its block of the batch
 *      (queries pqtg_shard_range(nq, G, g));
 *   2. the blocks' fine LUTs, candidate range lists (packed densely) and counters are
 *      all-gathered, so every rank holds the whole batch's candidate ranges;
 *   3. every rank re-ranks the batch's candidates inside its position range -> local top-k;
 *   4. all-to-all: rank j receives every rank's lists for its query block and merges them by
 *      (dist, id) (candidate_less, search.cpp:39-41);
 *   5. the merged blocks are all-gathered: every rank ends with the whole batch's results,
 *      bit-identical to the unsharded search.
 * Collectives: NCCL over NVLink (one process per GPU, pqtg_sharded_create_nccl; libnccl.so.2 is
 * loaded at run time) or, with every shard in this process (pqtg_sharded_create_local, any
 * devices), device-to-device copies -- the same protocol, used by the single-GPU tests.
 * Calls are collective: every rank calls with the same nq and k. With raw rows attached to every
 * shard (pqtg_index_attach_database of its positions) the exact stage runs across the shards: each
 * ships its line prefix with exact distances, the merge reproduces the reference's prefix cut. */
typedef struct pqtg_sharded pqtg_sharded;
#define PQTG_NCCL_ID_BYTES 128
/* A fresh NCCL unique id (ncclGetUniqueId) for rank 0 to hand to every rank. PQTG_ERR_NCCL if
 * libnccl.so.2 cannot be loaded. */
int pqtg_nccl_unique_id(uint8_t* id /* PQTG_NCCL_ID_BYTES */);
/* One rank of a `world`-process (world <= 64) deployment; `shard` holds positions
 * pqtg_shard_range(n, world, rank) and lives on this process's device. Borrowed, must outlive
 * the handle. Collective (ncclCommInitRank). */
int pqtg_sharded_create_nccl(pqtg_index* shard, const uint8_t* nccl_id, uint32_t rank, uint32_t world,
                             uint64_t max_batch, pqtg_sharded** out);
/* All `world` (<= 16) shards driven by this process: shards[g] holds pqtg_shard_range(n, world, g),
 * on any devices. Borrowed. */
int pqtg_sharded_create_local(pqtg_index* const* shards, uint32_t world, uint64_t max_batch,
                              pqtg_sharded** out);
/* Measurement harness: ONE real rank -- global rank `rank` of a `world`-GPU deployment, holding
 * its shard -- whose peers are simulated: the first search of a batch computes every block's
 * traversal + bin selection on this GPU (the peers' contributions), later searches of the same
 * batch run this rank's real device work (its block, the re-rank of the whole batch over its
 * shard, the merge of its block) with each transfer replaced by a device copy of the same bytes.
 * Results are this rank's; the other blocks' outputs are stand-ins. Used by bench.py
 * --sim-ranks to time a rank of the 8-GPU SIFT1B step on one GPU. */
int pqtg_sharded_create_sim(pqtg_index* shard, uint32_t rank, uint32_t world, uint64_t max_batch,
                            pqtg_sharded** out);
/* Ranks this handle drives: 1 (NCCL) or world (local). */
int pqtg_sharded_local_ranks(const pqtg_sharded* sh);
/* The workspace a local rank searched its last batch in (borrowed; pqtg_workspace_read gives
 * the whole batch's gathered candidate positions and counts; ntuples only for this rank's query
 * block). NULL on a bad argument. */
pqtg_workspace* pqtg_sharded_workspace(pqtg_sharded* sh, uint32_t local_rank);
/* Device buffers, one entry per local rank (on that rank's device): d_queries nq × dim (when
 * broadcast != 0 only global rank 0's batch is read and it is broadcast first), results nq × k
 * plus counts and (optional, may be NULL) stats -- on every rank, for the whole batch.
 * streams[i] (NULL entries / array = the legacy default stream) order the call: the search
 * starts after the work already queued there and later work there sees its results. nq <=
 * max_batch. */
int pqtg_sharded_search_device(pqtg_sharded* sh, const float* const* d_queries, uint64_t nq, uint32_t k,
                               int broadcast, uint32_t* const* d_ids, float* const* d_dists,
                               uint32_t* const* d_counts, pqtg_query_stats* const* d_stats,
                               void* const* streams);
/* Host buffers (pqt::knn_query_batch's contract): queries nq × dim are read on global rank 0
 * (NULL elsewhere), ids/dists nq × k, counts, stats (optional) are written on every rank that
 * passes them (local handle: rank 0's view). Synchronous. */
int pqtg_sharded_search(pqtg_sharded* sh, const float* queries, uint64_t nq, uint32_t dim, uint32_t k,
                        uint32_t* ids, float* dists, uint32_t* counts, pqtg_query_stats* stats);
/* Per-stage device time of the last search on local rank 0, in ms: [0] traversal + bin
 * selection of its block, [1] exchange of the range lists (with the batch's fine LUTs, computed while the host reads the sizes), [2] re-rank, [3] all-to-all + merge +
 * gather of the results. Synchronises. */
int pqtg_sharded_stage_ms(pqtg_sharded* sh, float* ms4);
void pqtg_sharded_destroy(pqtg_sharded* sh);

/* ---- exact ground truth ---------------------------------------------------------- */
/* pqt::brute_force_knn (src/search.cpp:276-299) for a batch: for every query the min(k, n)
 * rows of db (n × dim float32, row-major, vector id = row) nearest by l2_sq (distance.hpp:11-18,
 * sequential fp32), ordered by (dist, id); ids/dists are nq × k (padded with UINT32_MAX / +inf),
 * counts[q] = min(k, n); stats (optional) = {0, n, n} as the reference reports. n < 2^32,
 * k <= 4096. Host buffers, copied to and from `device` inside the call. */
int pqtg_brute_force_knn(const float* db, uint64_t n, uint32_t dim, const float* queries, uint64_t nq,
                         uint32_t k, int device, uint32_t* ids, float* dists, uint32_t* counts,
                         pqtg_query_stats* stats);
/* Same with device buffers, asynchronous on `stream` (no stats). */
int pqtg_brute_force_knn_device(const float* d_db, uint64_t n, uint32_t dim, const float* d_queries,
                                uint64_t nq, uint32_t k, uint32_t* d_ids, float* d_dists,
                                uint32_t* d_counts, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PQTG_H */
