/*
 * pqt_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the reference's online
 * query path (traverse → BinStream → slot gather → line_distance → top-k), used as the
 * parity checker for the CUDA path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. Every function cites the reference file:line it restates
 * (paths relative to the reference checkout's proj/).
 *
 * Pinning: the restatement is checked against (a) the reference itself compiled from its
 * own sources (oracle/_ref, see Makefile) on random indexes, and (b) golden fixtures under
 * tests/golden/ generated from that compiled reference (tests/golden/make_golden.py).
 */
#ifndef PQT_ORACLE_H
#define PQT_ORACLE_H

#include <stdint.h>

#include "../include/pqtg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pqto_index pqto_index;

const char* pqto_last_error(void);

/* Deep copy of a view (src/index_io.cpp:186-190: fine slices derived from level1). */
pqto_index* pqto_from_view(const pqtg_index_view* view);
/* A position shard [v->shard_lo, v->shard_hi) of an n-vector index: whole-index offsets, the
 * shard's ids, its line codes in position order (borrowed, not copied). */
pqto_index* pqto_from_shard_view(const pqtg_index_view* v, const uint8_t* lambda_q, const uint16_t* pair_id);
/* PQTINDEX v1 reader (src/index_io.cpp:148-229). NULL + pqto_last_error() on failure. */
pqto_index* pqto_load(const char* path);
/* PQTINDEX v1 writer (src/index_io.cpp:94-146). 0 on success. */
int pqto_save(const pqto_index* index, const char* path);
void pqto_free(pqto_index* index);
/* Borrowed view of the oracle's arrays (valid while the index lives). */
void pqto_view(const pqto_index* index, pqtg_index_view* out);

/* traverse (src/pqtree.cpp:74-120). fine: L×k1; l1_*: P×k1; l2_*: P×(w·k2). */
int pqto_traverse(const pqto_index* index, const float* y, float* fine, uint32_t* l1_id,
                  float* l1_dist, uint32_t* l2_parent, uint32_t* l2_child, float* l2_dist);

/* pick_slope_table (src/binorder.cpp:52-65). */
uint32_t pqto_pick_slope_table(const float* a, uint64_t na, const float* b, uint64_t nb);

/* heuristic_order / BinStream over the index's tables (src/binorder.cpp:178-316).
 * lists: parts × len sorted distances. Writes up to max_bins tuples; returns the count or
 * a negative status (PQTG_ERR_UNSUPPORTED for the exact-order fallback). */
int64_t pqto_heuristic_order(const pqto_index* index, const float* lists, uint32_t parts,
                             uint32_t len, uint64_t max_bins, uint32_t* out);

/* encode_slot (src/pqtree.cpp:12-25). parts_i1i2: parts × (i1, i2). */
uint64_t pqto_encode_slot(const uint32_t* parts_i1i2, uint32_t parts, uint32_t k1, uint32_t k2,
                          uint64_t hash_size);

/* line_distance (src/linequant.cpp:169-182) with the index's pair table. */
float pqto_line_distance(const pqto_index* index, const uint8_t* lambda_q,
                         const uint16_t* pair_id, const float* fine_dists);

/* Candidate gathering of knn_query (src/search.cpp:139-217) for one query. Writes the
 * gathered inverted-list POSITIONS (ids[] indices) in gather order; returns the count C
 * (<= cap) or a negative status. bins_visited may be NULL. */
int64_t pqto_candidates(const pqto_index* index, const float* y, uint32_t* positions,
                        uint64_t cap, uint64_t* bins_visited);

/* PqtIndex::attach_database (src/search.cpp:44-49): borrow n × dim raw vectors (id order) for
 * the exact re-rank stage; NULL detaches. */
void pqto_attach_database(pqto_index* index, const float* rows);

/* knn_query_batch (src/search.cpp:262-274); the exact re-rank runs only with raw vectors
 * attached (else as for a loaded index). Outputs nq × k; counts[q] valid entries; stats nq × 3
 * (bins_visited, candidates, exact_evals) may be NULL. shard_lo/hi restrict re-ranking to
 * positions in [lo, hi) (0/0 = all) and return that shard's local top-k. threads <= 0 means
 * all hardware threads. Returns 0 or a negative status. */
int pqto_knn_batch(const pqto_index* index, const float* queries, uint64_t nq, uint32_t dim,
                   uint32_t k, int threads, uint64_t shard_lo, uint64_t shard_hi, uint32_t* ids,
                   float* dists, uint32_t* counts, uint64_t* stats);

#ifdef __cplusplus
}
#endif

#endif
