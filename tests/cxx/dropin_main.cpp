// A reference-style C++ caller of the drop-in API (include/pqt/), exactly as code written
// against the reference's proj/include/pqt would call it. Used by tests/test_dropin_cxx.py.
//
//   dropin_main io    <index.pqt> <copy.pqt>                         load + save (no GPU)
//   dropin_main query <index.pqt> <queries.f32> <dim> <k> <out.bin> [db.f32]
//                                                      load (+ attach_database) + knn_query_batch
//   dropin_main sharded <index.pqt> <queries.f32> <dim> <k> <out.bin>
//                                  pqt::ShardedIndex over a one-rank NCCL communicator
//   dropin_main stages <index.pqt> <queries.f32> <dim> <max_bins> <out.bin>
//                                  per query: traverse, pick_slope_table, heuristic_order,
//                                  dijkstra_order, line_distance of stored codes 0..7; then
//                                  decode_pair of every pair id and build_slope_tables (no GPU)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqt/binorder.hpp"
#include "pqt/index_io.hpp"
#include "pqt/linequant.hpp"
#include "pqt/pqtree.hpp"
#include "pqt/search.hpp"
#include "pqt/sharded.hpp"

template <class T>
static void put(std::ofstream& o, const T* p, std::size_t n) {
    o.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}

static int stages(const pqt::PqtIndex& index, const pqt::VectorSet& q, std::size_t max_bins, const char* path) {
    std::ofstream out(path, std::ios::binary);
    const auto& c = index.config;
    for (std::size_t i = 0; i < q.count(); ++i) {
        const pqt::TraversalLists tl = pqt::traverse(index.tree, index.fine, q.row(i), c);
        put(out, tl.fine_dists.data(), tl.fine_dists.size());
        for (const auto& l : tl.level1)
            for (const auto& e : l) {
                put(out, &e.id, 1);
                put(out, &e.dist, 1);
            }
        std::vector<std::vector<float>> lists;
        for (const auto& l : tl.level2) {
            lists.emplace_back();
            for (const auto& e : l) {
                put(out, &e.parent, 1);
                put(out, &e.child, 1);
                put(out, &e.dist, 1);
                lists.back().push_back(e.dist);
            }
        }
        const std::uint32_t slope = lists.size() >= 2 ? pqt::pick_slope_table(lists[0], lists[1]) : 5u;
        put(out, &slope, 1);
        for (const auto& seq : {pqt::heuristic_order(lists, index.tables, max_bins), pqt::dijkstra_order(lists, max_bins)}) {
            const std::uint32_t cnt = static_cast<std::uint32_t>(seq.size());
            put(out, &cnt, 1);
            put(out, seq.ranks.data(), seq.ranks.size());
        }
        for (std::size_t v = 0; v < 8 && v < index.size(); ++v) {
            const float d = pqt::line_distance(index.codes.lambda_row(v), index.codes.pair_row(v), tl.fine_dists.data(),
                                               index.pair_table);
            put(out, &d, 1);
        }
    }
    for (std::uint32_t p = 0; p < index.pair_table.pair_count(); ++p) {
        const auto ij = pqt::decode_pair(p, c.k1);
        put(out, ij.data(), 2);
    }
    const auto tables = pqt::build_slope_tables(pqt::kDefaultOrderTableLen);
    for (const auto& t : tables) {
        put(out, &t.slope, 1);
        for (const auto& [a, b] : t.entries) {
            put(out, &a, 1);
            put(out, &b, 1);
        }
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const std::string mode = argv[1];
    pqt::PqtIndex index = pqt::load_index(argv[2]);
    if (mode == "io") {
        pqt::save_index(index, argv[3]);
        std::printf("n=%zu H=%llu\n", index.size(), (unsigned long long)index.lists.slots());
        return 0;
    }
    const unsigned dim = std::atoi(argv[4]), k = std::atoi(argv[5]);
    pqt::VectorSet q;
    q.dim = dim;
    {
        std::ifstream in(argv[3], std::ios::binary | std::ios::ate);
        const auto bytes = static_cast<std::size_t>(in.tellg());
        q.data.resize(bytes / sizeof(float));
        in.seekg(0);
        in.read(reinterpret_cast<char*>(q.data.data()), bytes);
    }
    if (mode == "stages") return stages(index, q, k, argv[6]);
    // the reference's error behaviour: wrong dimension -> std::invalid_argument
    bool threw = false;
    try {
        pqt::VectorSet bad;
        bad.dim = dim + 1;
        bad.data.assign(dim + 1, 0.0f);
        pqt::knn_query_batch(index, bad, k);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    if (!threw) return 3;
    if (argc > 7) {  // raw vectors for the exact re-rank stage (PqtIndex::attach_database)
        auto db = std::make_shared<pqt::VectorSet>();
        db->dim = dim;
        std::ifstream in(argv[7], std::ios::binary | std::ios::ate);
        const auto bytes = static_cast<std::size_t>(in.tellg());
        db->data.resize(bytes / sizeof(float));
        in.seekg(0);
        in.read(reinterpret_cast<char*>(db->data.data()), bytes);
        index.attach_database(db);
    }
    if (mode == "sharded") {
        pqt::ShardedIndex sh(argv[2], 0, 1, pqt::ShardedIndex::nccl_unique_id(), 0, 64);
        const std::vector<pqt::QueryResult> res = sh.knn_query_batch(q, k);
        std::ofstream out(argv[6], std::ios::binary);
        for (const auto& r : res) {
            const std::uint32_t c = static_cast<std::uint32_t>(r.ids.size());
            const std::uint64_t st[3] = {r.stats.bins_visited, r.stats.candidates, r.stats.exact_evals};
            out.write(reinterpret_cast<const char*>(&c), 4);
            out.write(reinterpret_cast<const char*>(st), sizeof st);
            out.write(reinterpret_cast<const char*>(r.ids.data()), 4 * c);
            out.write(reinterpret_cast<const char*>(r.dists.data()), 4 * c);
        }
        return 0;
    }
    std::vector<pqt::QueryResult> res = pqt::knn_query_batch(index, q, k);
    pqt::QueryResult one = pqt::knn_query(index, q.row(0), k);
    if (one.ids != res[0].ids) return 4;
    std::ofstream out(argv[6], std::ios::binary);
    for (const auto& r : res) {
        const std::uint32_t c = static_cast<std::uint32_t>(r.ids.size());
        const std::uint64_t st[3] = {r.stats.bins_visited, r.stats.candidates, r.stats.exact_evals};
        out.write(reinterpret_cast<const char*>(&c), 4);
        out.write(reinterpret_cast<const char*>(st), sizeof st);
        out.write(reinterpret_cast<const char*>(r.ids.data()), 4 * c);
        out.write(reinterpret_cast<const char*>(r.dists.data()), 4 * c);
    }
    return 0;
}
