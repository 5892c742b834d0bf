// pqt/sharded.hpp — knn_query_batch (proj/src/search.cpp:262-274) over an index sharded by
// inverted-list position across the GPUs of one box, one process per GPU (pqtg_sharded_* in
// pqtg.h: query-partitioned traversal / bin selection, NCCL exchange of the candidate range
// lists, per-shard re-rank, all-to-all + merge by (dist, id)). No reference counterpart: the
// reference is single-process; results are bit-identical to its knn_query_batch on the whole index.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "pqt/search.hpp"

struct pqtg_index;
struct pqtg_sharded;

namespace pqt {

class ShardedIndex {
public:
    using UniqueId = std::array<std::uint8_t, 128>;  // an NCCL unique id

    // A fresh id; rank 0 creates it and hands it to every rank (MPI, a file, a socket, ...).
    static UniqueId nccl_unique_id();

    // This rank's shard (positions pqtg_shard_range(n, world, rank)) of the PQTINDEX file at
    // `path`, on `device`. Collective: every rank constructs with the same id and world.
    ShardedIndex(const std::string& path, std::uint32_t rank, std::uint32_t world, const UniqueId& id, int device,
                 std::size_t max_batch = 4096);
    ~ShardedIndex();
    ShardedIndex(const ShardedIndex&) = delete;
    ShardedIndex& operator=(const ShardedIndex&) = delete;

    // Collective: every rank calls with the same batch (size and k; the contents are read on
    // rank 0 only and broadcast); every rank gets all results.
    std::vector<QueryResult> knn_query_batch(const VectorSet& queries, std::uint32_t k);

    // PqtIndex::attach_database (search.cpp:44-49) for this rank: its positions' raw rows in
    // position order (db rows ids[lo..hi)); with rows on every rank and rerank_exact > 0 the
    // exact stage runs across the shards. nullptr detaches. Not concurrent with a search.
    void attach_database(const VectorSet* shard_rows);
    std::pair<std::uint64_t, std::uint64_t> positions() const { return {lo_, hi_}; }

    std::size_t size() const { return n_; }
    std::uint32_t rank() const { return rank_; }

private:
    pqtg_index* shard_ = nullptr;
    pqtg_sharded* sh_ = nullptr;
    std::size_t n_ = 0;
    std::uint64_t lo_ = 0, hi_ = 0;
    std::uint32_t dim_ = 0, rank_ = 0;
    std::size_t max_batch_ = 0;
};

}  // namespace pqt
