// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product path).
//
// extern "C" shim over the UNMODIFIED reference sources compiled in place from
// /root/reference/proj/src by oracle/Makefile with -Dpqt=pqtref (every reference symbol
// becomes pqtref::…). Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
// --impl reference legs load the resulting oracle/_ref/libpqtref.so.
//
// Each function forwards to the reference's public API named beside it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#ifndef PQTREF_NO_BENCH
#include "pqt/bench.hpp"
#endif
#include "pqt/binorder.hpp"
#include "pqt/codebook.hpp"
#include "pqt/index_io.hpp"
#include "pqt/linequant.hpp"
#include "pqt/pqtree.hpp"
#include "pqt/search.hpp"
#include "pqt/vecio.hpp"

#include "../include/pqtg.h"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

pqt::PqtConfig to_cfg(const pqtg_config* c) {
    pqt::PqtConfig cfg;
    cfg.dim = c->dim;
    cfg.p_tree = c->p_tree;
    cfg.k1 = c->k1;
    cfg.k2 = c->k2;
    cfg.w = c->w;
    cfg.p_line = c->p_line;
    cfg.hash_size = c->hash_size;
    cfg.candidate_budget = c->candidate_budget;
    cfg.rerank_exact = c->rerank_exact;
    cfg.resort_bins = c->resort_bins != 0;
    cfg.train_iters = c->train_iters;
    cfg.seed = c->seed;
    return cfg;
}

void from_cfg(const pqt::PqtConfig& cfg, pqtg_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->dim = cfg.dim;
    c->p_tree = cfg.p_tree;
    c->k1 = cfg.k1;
    c->k2 = cfg.k2;
    c->w = cfg.w;
    c->p_line = cfg.p_line;
    c->hash_size = cfg.hash_size;
    c->candidate_budget = cfg.candidate_budget;
    c->rerank_exact = cfg.rerank_exact;
    c->resort_bins = cfg.resort_bins ? 1u : 0u;
    c->train_iters = cfg.train_iters;
    c->seed = cfg.seed;
}

pqt::VectorSet make_set(const float* data, size_t n, uint32_t dim) {
    pqt::VectorSet s;
    s.dim = dim;
    s.data.assign(data, data + n * dim);
    return s;
}

// Index plus the flattened arrays handed out by ref_index_view (kept alive with it).
struct Handle {
    pqt::PqtIndex index;
    std::vector<float> level1, level2;
    std::vector<double> slopes;
    std::vector<uint32_t> entries;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// pqt::synth_clustered (bench.cpp:66-95)
int ref_synth_clustered(uint64_t n, uint32_t dim, uint32_t blobs, float sigma, uint64_t seed,
                        float* out) {
#ifdef PQTREF_NO_BENCH
    (void)n; (void)dim; (void)blobs; (void)sigma; (void)seed; (void)out;
    g_err = "bench.cpp not compiled (json.hpp missing)";
    return -1;
#else
    try {
        pqt::VectorSet s = pqt::synth_clustered(n, dim, blobs, sigma, seed);
        std::memcpy(out, s.data.data(), s.data.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
#endif
}

// pqt::IndexBuilder(train, cfg, threads, keep_raw) + add(db) + finalize() (search.cpp:52-117)
void* ref_build_index(const float* train, uint64_t ntrain, const float* db, uint64_t n,
                      const pqtg_config* cfg, int threads, int keep_raw) {
    try {
        pqt::PqtConfig c = to_cfg(cfg);
        pqt::VectorSet tr = make_set(train, ntrain, c.dim);
        pqt::IndexBuilder b(tr, c, threads, keep_raw != 0);
        if (n > 0) {
            b.add(make_set(db, n, c.dim));
        }
        auto* h = new Handle;
        h->index = b.finalize();
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// pqt::IndexBuilder streamed in waves (search.cpp:52-117): new(train) → add(chunk)* →
// finalize. This is how the reference builds an index larger than one in-memory set
// (DEEP100M / SIFT1B-shaped), keep_raw = false.
void* ref_builder_new(const float* train, uint64_t ntrain, const pqtg_config* cfg, int threads) {
    try {
        pqt::PqtConfig c = to_cfg(cfg);
        pqt::VectorSet tr = make_set(train, ntrain, c.dim);
        return new pqt::IndexBuilder(tr, c, threads, false);
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int ref_builder_add(void* builder, const float* rows, uint64_t n, uint32_t dim) {
    try {
        static_cast<pqt::IndexBuilder*>(builder)->add(make_set(rows, n, dim));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// finalize() consumes the builder (freed here) and returns an index handle
void* ref_builder_finalize(void* builder) {
    auto* b = static_cast<pqt::IndexBuilder*>(builder);
    try {
        auto* h = new Handle;
        h->index = b->finalize();
        delete b;
        return h;
    } catch (const std::exception& e) {
        delete b;
        fail(e);
        return nullptr;
    }
}

// pqt::load_index (index_io.cpp:148)
void* ref_load_index(const char* path) {
    try {
        auto* h = new Handle;
        h->index = pqt::load_index(path);
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// pqt::save_index (index_io.cpp:94)
int ref_save_index(void* handle, const char* path) {
    try {
        pqt::save_index(static_cast<Handle*>(handle)->index, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_free(void* handle) { delete static_cast<Handle*>(handle); }

// Builds a pqtref::PqtIndex from a view the same way load_index does: fine centroids and the
// pair table are rebuilt from the codebooks, then d2 is overwritten by the stored one
// (index_io.cpp:186-190).
void* ref_from_view(const pqtg_index_view* v) {
    try {
        auto* h = new Handle;
        pqt::PqtIndex& ix = h->index;
        ix.config = to_cfg(&v->config);
        ix.config.validate();
        const uint32_t P = ix.config.p_tree, k1 = ix.config.k1, k2 = ix.config.k2;
        const uint32_t m = ix.config.dim / P;
        ix.tree.level1.resize(P);
        ix.tree.level2.resize(P);
        for (uint32_t p = 0; p < P; ++p) {
            auto& b = ix.tree.level1[p];
            b.part_dim = m;
            b.k = k1;
            b.centroids.assign(v->level1 + (size_t)p * k1 * m, v->level1 + (size_t)(p + 1) * k1 * m);
            ix.tree.level2[p].resize(k1);
            for (uint32_t i = 0; i < k1; ++i) {
                auto& c = ix.tree.level2[p][i];
                c.part_dim = m;
                c.k = k2;
                const float* src = v->level2 + ((size_t)p * k1 + i) * k2 * m;
                c.centroids.assign(src, src + (size_t)k2 * m);
            }
        }
        ix.fine = pqt::build_fine_centroids(ix.tree, ix.config.p_line);
        ix.pair_table = pqt::build_pair_table(ix.fine);
        ix.pair_table.d2.assign(v->d2, v->d2 + (size_t)ix.config.p_line * k1 * k1);
        ix.tables.resize(v->table_count);
        for (uint32_t t = 0; t < v->table_count; ++t) {
            ix.tables[t].slope = v->table_slopes[t];
            ix.tables[t].entries.resize(v->table_len);
            for (uint32_t e = 0; e < v->table_len; ++e) {
                const uint32_t* pe = v->table_entries + ((size_t)t * v->table_len + e) * 2;
                ix.tables[t].entries[e] = {pe[0], pe[1]};
            }
        }
        ix.lists.offsets.assign(v->offsets, v->offsets + ix.config.hash_size + 1);
        ix.lists.ids.assign(v->ids, v->ids + v->n);
        ix.codes.p_line = ix.config.p_line;
        ix.codes.lambda_q.assign(v->lambda_q, v->lambda_q + v->n * ix.config.p_line);
        ix.codes.pair_id.assign(v->pair_id, v->pair_id + v->n * ix.config.p_line);
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Flattens the index into a pqtg_index_view (arrays owned by the handle).
int ref_index_view(void* handle, pqtg_index_view* v) {
    try {
        auto* h = static_cast<Handle*>(handle);
        const pqt::PqtIndex& ix = h->index;
        std::memset(v, 0, sizeof(*v));
        from_cfg(ix.config, &v->config);
        v->n = ix.size();
        h->level1.clear();
        h->level2.clear();
        for (const auto& b : ix.tree.level1) {
            h->level1.insert(h->level1.end(), b.centroids.begin(), b.centroids.end());
        }
        for (const auto& kids : ix.tree.level2) {
            for (const auto& b : kids) {
                h->level2.insert(h->level2.end(), b.centroids.begin(), b.centroids.end());
            }
        }
        h->slopes.clear();
        h->entries.clear();
        for (const auto& t : ix.tables) {
            h->slopes.push_back(t.slope);
            for (const auto& [a, b] : t.entries) {
                h->entries.push_back(a);
                h->entries.push_back(b);
            }
        }
        v->level1 = h->level1.data();
        v->level2 = h->level2.data();
        v->d2 = ix.pair_table.d2.data();
        v->table_count = static_cast<uint32_t>(ix.tables.size());
        v->table_len = ix.tables.empty() ? 0u : static_cast<uint32_t>(ix.tables[0].entries.size());
        v->table_slopes = h->slopes.data();
        v->table_entries = h->entries.data();
        v->offsets = ix.lists.offsets.data();
        v->ids = ix.lists.ids.data();
        v->lambda_q = ix.codes.lambda_q.data();
        v->pair_id = ix.codes.pair_id.data();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Raw database attached to the index (only present for keep_raw builds): n × dim floats.
const float* ref_index_database(void* handle) {
    auto* h = static_cast<Handle*>(handle);
    return h->index.database ? h->index.database->data.data() : nullptr;
}

// Detach the raw database so queries run the loaded-index path (rerank disabled).
void ref_detach_database(void* handle) { static_cast<Handle*>(handle)->index.database.reset(); }

// pqt::PqtIndex::attach_database (search.cpp:44-49) with a copy of n × dim raw vectors.
int ref_attach_database(void* handle, const float* rows, uint64_t n) {
    try {
        auto* h = static_cast<Handle*>(handle);
        auto db = std::make_shared<pqt::VectorSet>(make_set(rows, n, h->index.config.dim));
        h->index.attach_database(db);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pqt::knn_query_batch (search.cpp:262-274). stats: nq × 3 (bins_visited, candidates, exact_evals);
// stage_us: nq × 4 (traversal, bin_selection, vector_proposal, rerank) or NULL.
int ref_knn_batch(void* handle, const float* queries, uint64_t nq, uint32_t k, int threads,
                  uint32_t* ids, float* dists, uint32_t* counts, uint64_t* stats,
                  double* stage_us) {
    try {
        auto* h = static_cast<Handle*>(handle);
        pqt::VectorSet q = make_set(queries, nq, h->index.config.dim);
        std::vector<pqt::QueryResult> res = pqt::knn_query_batch(h->index, q, k, threads);
        for (uint64_t i = 0; i < nq; ++i) {
            const auto& r = res[i];
            counts[i] = static_cast<uint32_t>(r.ids.size());
            for (size_t j = 0; j < r.ids.size(); ++j) {
                ids[i * k + j] = r.ids[j];
                dists[i * k + j] = r.dists[j];
            }
            if (stats) {
                stats[i * 3 + 0] = r.stats.bins_visited;
                stats[i * 3 + 1] = r.stats.candidates;
                stats[i * 3 + 2] = r.stats.exact_evals;
            }
            if (stage_us) {
                stage_us[i * 4 + 0] = r.stats.traversal_us;
                stage_us[i * 4 + 1] = r.stats.bin_selection_us;
                stage_us[i * 4 + 2] = r.stats.vector_proposal_us;
                stage_us[i * 4 + 3] = r.stats.rerank_us;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pqt::traverse (pqtree.cpp:74-120). fine: p_line × k1; l1_*: p_tree × k1; l2_*: p_tree × (w·k2).
int ref_traverse(void* handle, const float* y, float* fine, uint32_t* l1_id, float* l1_dist,
                 uint32_t* l2_parent, uint32_t* l2_child, float* l2_dist) {
    try {
        auto* h = static_cast<Handle*>(handle);
        const auto& ix = h->index;
        pqt::TraversalLists tl = pqt::traverse(ix.tree, ix.fine, y, ix.config);
        std::memcpy(fine, tl.fine_dists.data(), tl.fine_dists.size() * sizeof(float));
        const uint32_t P = ix.config.p_tree, k1 = ix.config.k1, W = ix.config.w * ix.config.k2;
        for (uint32_t p = 0; p < P; ++p) {
            for (uint32_t i = 0; i < k1; ++i) {
                l1_id[p * k1 + i] = tl.level1[p][i].id;
                l1_dist[p * k1 + i] = tl.level1[p][i].dist;
            }
            for (uint32_t r = 0; r < W; ++r) {
                l2_parent[p * W + r] = tl.level2[p][r].parent;
                l2_child[p * W + r] = tl.level2[p][r].child;
                l2_dist[p * W + r] = tl.level2[p][r].dist;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pqt::dijkstra_order (binorder.cpp:114-167). lists: parts × len. Returns the tuple count.
int64_t ref_dijkstra_order(const float* lists, uint32_t parts, uint32_t len, uint64_t max_bins, uint32_t* out) {
    try {
        std::vector<std::vector<float>> dl(parts);
        for (uint32_t p = 0; p < parts; ++p) dl[p].assign(lists + (size_t)p * len, lists + (size_t)(p + 1) * len);
        pqt::BinSequence s = pqt::dijkstra_order(dl, max_bins);
        std::memcpy(out, s.ranks.data(), s.ranks.size() * sizeof(uint32_t));
        return static_cast<int64_t>(s.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// pqt::decode_pair (linequant.cpp) for every pair id < count
int ref_decode_pairs(uint32_t k1, uint32_t count, uint16_t* out) {
    for (uint32_t q = 0; q < count; ++q) {
        const auto ij = pqt::decode_pair(q, k1);
        out[2 * q] = ij[0];
        out[2 * q + 1] = ij[1];
    }
    return 0;
}

// pqt::heuristic_order over the index's tables (binorder.cpp:301-316). lists: parts × len.
// Returns the number of tuples written to out (parts × count), or -1.
int64_t ref_heuristic_order(void* handle, const float* lists, uint32_t parts, uint32_t len,
                            uint64_t max_bins, uint32_t* out) {
    try {
        auto* h = static_cast<Handle*>(handle);
        std::vector<std::vector<float>> dl(parts);
        for (uint32_t p = 0; p < parts; ++p) {
            dl[p].assign(lists + (size_t)p * len, lists + (size_t)(p + 1) * len);
        }
        pqt::BinSequence s = pqt::heuristic_order(dl, h->index.tables, max_bins);
        std::memcpy(out, s.ranks.data(), s.ranks.size() * sizeof(uint32_t));
        return static_cast<int64_t>(s.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// pqt::pick_slope_table (binorder.cpp:52-65)
uint32_t ref_pick_slope_table(const float* a, uint64_t na, const float* b, uint64_t nb) {
    return pqt::pick_slope_table(std::span<const float>(a, na), std::span<const float>(b, nb));
}

// pqt::build_slope_tables (binorder.cpp:13-50): slopes[10], entries[10 × len × 2]
int ref_build_slope_tables(uint32_t len, double* slopes, uint32_t* entries) {
    try {
        auto t = pqt::build_slope_tables(len);
        for (size_t i = 0; i < t.size(); ++i) {
            slopes[i] = t[i].slope;
            for (size_t e = 0; e < t[i].entries.size(); ++e) {
                entries[(i * len + e) * 2] = t[i].entries[e].first;
                entries[(i * len + e) * 2 + 1] = t[i].entries[e].second;
            }
        }
        return static_cast<int>(t.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pqt::encode_slot (pqtree.cpp:23-25) for parts × (i1, i2)
uint64_t ref_encode_slot(const uint32_t* parts_i1i2, uint32_t parts, uint32_t k1, uint32_t k2,
                         uint64_t hash_size) {
    pqt::BinCode code;
    code.parts.resize(parts);
    for (uint32_t p = 0; p < parts; ++p) {
        code.parts[p] = {parts_i1i2[2 * p], parts_i1i2[2 * p + 1]};
    }
    pqt::PqtConfig cfg;
    cfg.p_tree = parts;
    cfg.k1 = k1;
    cfg.k2 = k2;
    return pqt::encode_slot(code, cfg, hash_size);
}

// pqt::line_distance (linequant.cpp:169-182) against the index's pair table
float ref_line_distance(void* handle, const uint8_t* lambda_q, const uint16_t* pair_id,
                        const float* fine_dists) {
    auto* h = static_cast<Handle*>(handle);
    return pqt::line_distance(lambda_q, pair_id, fine_dists, h->index.pair_table);
}

// pqt::assign_bin + global_code (pqtree.cpp:12-38) and pqt::encode_line (linequant.cpp:84-152)
// for n vectors against the index's codebooks: codes[n] (unhashed global code), lambda/pair n × L.
int ref_assign_encode(void* handle, const float* x, uint64_t n, uint64_t* codes,
                      uint8_t* lambda_q, uint16_t* pair_id) {
    try {
        auto* h = static_cast<Handle*>(handle);
        const auto& ix = h->index;
        const uint32_t D = ix.config.dim, L = ix.config.p_line;
        for (uint64_t i = 0; i < n; ++i) {
            codes[i] = pqt::global_code(pqt::assign_bin(ix.tree, x + i * D), ix.config);
            pqt::encode_line(ix.fine, ix.pair_table, x + i * D, lambda_q + i * L, pair_id + i * L);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pqt::brute_force_knn (search.cpp:276-299) over a raw set
int ref_brute_force(const float* db, uint64_t n, uint32_t dim, const float* queries, uint64_t nq,
                    uint32_t k, uint32_t* ids, float* dists) {
    try {
        pqt::VectorSet s = make_set(db, n, dim);
        for (uint64_t q = 0; q < nq; ++q) {
            pqt::QueryResult r = pqt::brute_force_knn(s, queries + q * dim, k);
            for (size_t j = 0; j < r.ids.size(); ++j) {
                ids[q * k + j] = r.ids[j];
                dists[q * k + j] = r.dists[j];
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
