// pqt/search.hpp — drop-in replacement for the reference's query API
// (proj/include/pqt/search.hpp:15-47, :80-83), served by the B200 kernels in libpqtg.so.
//
// Same types, same signatures, same exceptions. Differences a caller can observe:
//  * queries run on a CUDA device (device 0 unless PQTG_DEVICE is set); the first query on
//    an index uploads it and caches the device copy in PqtIndex::gpu, keyed by the config and
//    the arrays' addresses/sizes (a changed config or re-assigned arrays re-upload; in-place
//    element edits need index.gpu.reset());
//  * exact re-ranking against attached raw vectors runs on the GPU (the database is copied to
//    the device on the first query after attach_database); without one the calls warn once and
//    disable it, exactly as the reference does (search.cpp:25-32);
//  * QueryStats *_us are each query's per-stage device wall times (its stage kernels' CTAs, with
//    the batch's other queries running beside them); bin selection and candidate gathering are one
//    kernel, reported as bin_selection_us (vector_proposal_us = 0).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "pqt/binorder.hpp"
#include "pqt/codebook.hpp"
#include "pqt/linequant.hpp"
#include "pqt/pqtree.hpp"
#include "pqt/vecio.hpp"

namespace pqt {

struct QueryStats {
    std::uint64_t bins_visited = 0;
    std::uint64_t candidates = 0;
    std::uint64_t exact_evals = 0;
    double traversal_us = 0.0;
    double bin_selection_us = 0.0;
    double vector_proposal_us = 0.0;
    double rerank_us = 0.0;
};

struct QueryResult {
    std::vector<std::uint32_t> ids;
    std::vector<float> dists;  // squared, non-decreasing
    QueryStats stats;
};

struct PqtIndex {
    PqtConfig config;  // hash_size resolved
    TreeCodebooks tree;
    FineCentroids fine;
    PairDistanceTable pair_table;
    std::vector<OrderTable> tables;
    InvertedLists lists;
    LineCodes codes;
    std::shared_ptr<const VectorSet> database;  // optional
    mutable std::shared_ptr<void> gpu;          // device copy (pqtg_index + workspace), lazily built

    std::size_t size() const { return lists.ids.size(); }
    void attach_database(std::shared_ptr<const VectorSet> db);
};

QueryResult knn_query(const PqtIndex& index, const float* y, std::uint32_t k);

std::vector<QueryResult> knn_query_batch(const PqtIndex& index, const VectorSet& queries, std::uint32_t k,
                                         int threads = 0);

// Exact k-NN by brute force over db (search.cpp:276-299), computed on the GPU.
QueryResult brute_force_knn(const VectorSet& db, const float* y, std::uint32_t k);

}  // namespace pqt
