// A reference-style C++ caller of the drop-in API (include/pqt/), exactly as code written
// against the reference's proj/include/pqt would call it. Used by tests/test_dropin_cxx.py.
//
//   dropin_main io    <index.pqt> <copy.pqt>                         load + save (no GPU)
//   dropin_main query <index.pqt> <queries.f32> <dim> <k> <out.bin> [db.f32]
//                                                      load (+ attach_database) + knn_query_batch
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqt/index_io.hpp"
#include "pqt/search.hpp"

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
