// pqt_dropin.cpp — the reference's C++ query API (include/pqt/*.hpp in this repo, mirroring
// proj/include/pqt/{search,index_io,codebook,linequant}.hpp) implemented over the C-ABI.
//
//   pqt::load_index        ← index_io.cpp:148-229   (shared PQTINDEX parser, index_file.cpp)
//   pqt::save_index        ← index_io.cpp:94-146    (byte-identical container)
//   pqt::knn_query_batch   ← search.cpp:262-274     → pqtg_search on the cached device index
//   pqt::knn_query         ← search.cpp:126-260     → a batch of one
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/pqt/index_io.hpp"
#include "../../include/pqt/search.hpp"
#include "../../include/pqt/sharded.hpp"
#include "pqtg_internal.h"

namespace pqt {

// ------------------------------------------------------------------ config + tables
void PqtConfig::validate() const {
    pqtg_config c{};
    c.dim = dim;
    c.p_tree = p_tree;
    c.k1 = k1;
    c.k2 = k2;
    c.w = w;
    c.p_line = p_line;
    try {
        pqtg::validate_config(c);
    } catch (const pqtg::Error& e) {
        throw std::invalid_argument(e.msg);
    }
}

std::uint64_t PqtConfig::resolved_hash_size(std::size_t n) const {
    if (hash_size > 0) return hash_size;
    const std::uint64_t h = std::min<std::uint64_t>(1ULL << 26, 4 * static_cast<std::uint64_t>(n));
    return std::max<std::uint64_t>(1, h);
}

// Slices of the level-1 centroids per fine part, |slice|^2 by sequential fp32 dot
// (linequant.cpp:13-46).
FineCentroids build_fine_centroids(const TreeCodebooks& tree, std::uint32_t p_line) {
    if (tree.level1.empty()) throw std::invalid_argument("build_fine_centroids: empty tree");
    const std::uint32_t P = tree.parts(), m = tree.level1[0].part_dim, k1 = tree.level1[0].k;
    if (p_line % P != 0 || m % (p_line / P) != 0) throw std::invalid_argument("build_fine_centroids: p_line incompatible with tree");
    const std::uint32_t per = p_line / P, fd = m / per;
    FineCentroids f;
    f.p_line = p_line;
    f.k1 = k1;
    f.fine_dim = fd;
    f.slices.resize(static_cast<std::size_t>(p_line) * k1 * fd);
    f.sqnorm.resize(static_cast<std::size_t>(p_line) * k1);
    for (std::uint32_t fp = 0; fp < p_line; ++fp) {
        for (std::uint32_t i = 0; i < k1; ++i) {
            const float* src = tree.level1[fp / per].row(i) + static_cast<std::size_t>(fp % per) * fd;
            float* dst = f.slices.data() + (static_cast<std::size_t>(fp) * k1 + i) * fd;
            float acc = 0.0f;
            for (std::uint32_t t = 0; t < fd; ++t) {
                dst[t] = src[t];
                acc += dst[t] * dst[t];
            }
            f.sqnorm[static_cast<std::size_t>(fp) * k1 + i] = acc;
        }
    }
    return f;
}

// d2 by sequential fp32 l2_sq and the lexicographic (i < j) pairs (linequant.cpp:60-82).
PairDistanceTable build_pair_table(const FineCentroids& fine) {
    PairDistanceTable t;
    t.p_line = fine.p_line;
    t.k1 = fine.k1;
    t.d2.assign(static_cast<std::size_t>(fine.p_line) * fine.k1 * fine.k1, 0.0f);
    for (std::uint32_t f = 0; f < fine.p_line; ++f)
        for (std::uint32_t i = 0; i < fine.k1; ++i)
            for (std::uint32_t j = i + 1; j < fine.k1; ++j) {
                const float* a = fine.slice(f, i);
                const float* b = fine.slice(f, j);
                float acc = 0.0f;
                for (std::uint32_t d = 0; d < fine.fine_dim; ++d) {
                    const float x = a[d] - b[d];
                    acc += x * x;
                }
                t.d2[(static_cast<std::size_t>(f) * fine.k1 + i) * fine.k1 + j] = acc;
                t.d2[(static_cast<std::size_t>(f) * fine.k1 + j) * fine.k1 + i] = acc;
            }
    if (fine.k1 == 1) {
        t.pairs.push_back({0, 0});
    } else {
        for (std::uint16_t i = 0; i < fine.k1; ++i)
            for (std::uint16_t j = i + 1; j < fine.k1; ++j) t.pairs.push_back({i, j});
    }
    return t;
}

void PqtIndex::attach_database(std::shared_ptr<const VectorSet> db) {
    if (db && (db->count() != size() || db->dim != config.dim))
        throw std::invalid_argument("attach_database: vector set does not match index");
    database = std::move(db);
}

// ------------------------------------------------------------------ container
namespace {

[[noreturn]] void rethrow(int status) {
    const std::string msg = pqtg_last_error();
    if (status == PQTG_ERR_BAD_DIM || status == PQTG_ERR_CONFIG) throw std::invalid_argument(msg);
    if (status == PQTG_ERR_FORMAT) throw FormatError(msg);
    throw std::runtime_error("pqtg: " + msg);
}

void check(int status) {
    if (status != PQTG_OK) rethrow(status);
}

template <class T>
void put(std::ofstream& out, const T& v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

}  // namespace

PqtIndex load_index(const std::string& path) {
    pqtg::LoadedFile lf;
    try {
        pqtg::parse_index(path.c_str(), lf);
    } catch (const pqtg::Error& e) {
        if (e.status == PQTG_ERR_CONFIG) throw std::invalid_argument(e.msg);
        throw FormatError(e.msg);
    }
    const pqtg::Source& s = lf.src;
    PqtIndex ix;
    PqtConfig& c = ix.config;
    c.dim = s.cfg.dim;
    c.p_tree = s.cfg.p_tree;
    c.k1 = s.cfg.k1;
    c.k2 = s.cfg.k2;
    c.w = s.cfg.w;
    c.p_line = s.cfg.p_line;
    c.hash_size = s.cfg.hash_size;
    c.candidate_budget = s.cfg.candidate_budget;
    c.rerank_exact = s.cfg.rerank_exact;
    c.resort_bins = s.cfg.resort_bins != 0;
    c.train_iters = s.cfg.train_iters;
    c.seed = s.cfg.seed;
    const std::uint32_t P = c.p_tree, k1 = c.k1, k2 = c.k2, m = c.dim / P;
    ix.tree.level1.resize(P);
    ix.tree.level2.resize(P);
    for (std::uint32_t p = 0; p < P; ++p) {
        ix.tree.level1[p] = {m, k1, std::vector<float>(s.level1 + (std::size_t)p * k1 * m,
                                                      s.level1 + (std::size_t)(p + 1) * k1 * m)};
        ix.tree.level2[p].resize(k1);
        for (std::uint32_t i = 0; i < k1; ++i) {
            const float* b = s.level2 + ((std::size_t)p * k1 + i) * k2 * m;
            ix.tree.level2[p][i] = {m, k2, std::vector<float>(b, b + (std::size_t)k2 * m)};
        }
    }
    ix.fine = build_fine_centroids(ix.tree, c.p_line);
    ix.pair_table = build_pair_table(ix.fine);
    ix.pair_table.d2.assign(s.d2, s.d2 + (std::size_t)c.p_line * k1 * k1);  // stored table wins
    ix.tables.resize(s.table_count);
    for (std::uint32_t t = 0; t < s.table_count; ++t) {
        ix.tables[t].slope = s.slopes[t];
        ix.tables[t].entries.resize(s.table_len);
        for (std::uint32_t e = 0; e < s.table_len; ++e)
            ix.tables[t].entries[e] = {s.entries[((std::size_t)t * s.table_len + e) * 2],
                                       s.entries[((std::size_t)t * s.table_len + e) * 2 + 1]};
    }
    ix.lists.offsets = std::move(lf.offsets);
    ix.lists.ids = std::move(lf.ids);
    const std::size_t records = (std::size_t)s.n * c.p_line;
    ix.codes.p_line = c.p_line;
    ix.codes.lambda_q.resize(records);
    ix.codes.pair_id.resize(records);
    const std::uint32_t w = 1 + s.record_pw;
    for (std::size_t i = 0; i < records; ++i) {
        const std::uint8_t* r = s.records + i * w;
        ix.codes.lambda_q[i] = r[0];
        ix.codes.pair_id[i] = s.record_pw == 1 ? r[1] : (std::uint16_t)(r[1] | (r[2] << 8));
    }
    return ix;
}

void save_index(const PqtIndex& ix, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw FormatError("cannot open " + path + " for writing");
    const PqtConfig& c = ix.config;
    out.write("PQTINDEX", 8);
    put(out, std::uint32_t{1});
    put(out, c.dim);
    put(out, c.p_tree);
    put(out, c.k1);
    put(out, c.k2);
    put(out, c.w);
    put(out, c.p_line);
    put(out, c.hash_size);
    put(out, c.candidate_budget);
    put(out, c.rerank_exact);
    put(out, static_cast<std::uint8_t>(c.resort_bins ? 1 : 0));
    put(out, c.train_iters);
    put(out, c.seed);
    put(out, static_cast<std::uint64_t>(ix.size()));
    auto book = [&](const Codebook& b) {
        put(out, b.part_dim);
        put(out, b.k);
        out.write(reinterpret_cast<const char*>(b.centroids.data()), b.centroids.size() * sizeof(float));
    };
    for (const auto& b : ix.tree.level1) book(b);
    for (const auto& kids : ix.tree.level2)
        for (const auto& b : kids) book(b);
    out.write(reinterpret_cast<const char*>(ix.pair_table.d2.data()), ix.pair_table.d2.size() * sizeof(float));
    put(out, static_cast<std::uint32_t>(ix.tables.size()));
    put(out, static_cast<std::uint32_t>(ix.tables.empty() ? 0 : ix.tables[0].entries.size()));
    for (const auto& t : ix.tables) {
        put(out, t.slope);
        for (const auto& [a, b] : t.entries) {
            put(out, a);
            put(out, b);
        }
    }
    out.write(reinterpret_cast<const char*>(ix.lists.offsets.data()), ix.lists.offsets.size() * 8);
    out.write(reinterpret_cast<const char*>(ix.lists.ids.data()), ix.lists.ids.size() * 4);
    const bool narrow = ix.pair_table.pair_count() <= 256;
    put(out, static_cast<std::uint8_t>(narrow ? 1 : 2));
    for (std::size_t i = 0; i < ix.codes.lambda_q.size(); ++i) {
        put(out, ix.codes.lambda_q[i]);
        if (narrow) put(out, static_cast<std::uint8_t>(ix.codes.pair_id[i]));
        else put(out, ix.codes.pair_id[i]);
    }
    if (!out) throw FormatError("write failed for " + path);
}

// ------------------------------------------------------------------ queries
namespace {

// page-locked staging for small batches (<= kStageMax queries): the search then replays a CUDA
// graph that writes the results straight into these buffers (pqtg_search's zero-copy path), and
// a serving loop of knn_query calls keeps hitting the same graph
constexpr std::size_t kStageMax = 128;

struct DeviceCopy {
    pqtg_index* ix = nullptr;
    pqtg_workspace* ws = nullptr;
    const VectorSet* db = nullptr;  // raw vectors currently on the device (exact re-rank)
    std::uint64_t fingerprint = 0;  // of the host index the copy was made from
    std::mutex stage_mu;
    std::uint32_t stage_k = 0, stage_dim = 0;
    float* h_q = nullptr;
    std::uint32_t* h_ids = nullptr;
    float* h_dists = nullptr;
    std::uint32_t* h_counts = nullptr;
    pqtg_query_stats* h_stats = nullptr;
    void free_stage() {
        for (void* p : {static_cast<void*>(h_q), static_cast<void*>(h_ids), static_cast<void*>(h_dists),
                        static_cast<void*>(h_counts), static_cast<void*>(h_stats)})
            if (p) cudaFreeHost(p);
        h_q = nullptr;
        h_ids = nullptr;
        h_dists = nullptr;
        h_counts = nullptr;
        h_stats = nullptr;
        stage_k = stage_dim = 0;
    }
    // staging for kStageMax queries of `dim` floats and k results; false when it cannot be had
    bool stage(std::uint32_t dim, std::uint32_t k) {
        if (h_q && stage_dim == dim && stage_k >= k) return true;
        free_stage();
        const bool ok = cudaMallocHost(reinterpret_cast<void**>(&h_q), kStageMax * dim * sizeof(float)) == cudaSuccess &&
                        cudaMallocHost(reinterpret_cast<void**>(&h_ids), kStageMax * k * sizeof(std::uint32_t)) == cudaSuccess &&
                        cudaMallocHost(reinterpret_cast<void**>(&h_dists), kStageMax * k * sizeof(float)) == cudaSuccess &&
                        cudaMallocHost(reinterpret_cast<void**>(&h_counts), kStageMax * sizeof(std::uint32_t)) == cudaSuccess &&
                        cudaMallocHost(reinterpret_cast<void**>(&h_stats), kStageMax * sizeof(pqtg_query_stats)) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            free_stage();
            return false;
        }
        stage_dim = dim;
        stage_k = k;
        return true;
    }
    ~DeviceCopy() {
        free_stage();
        pqtg_workspace_destroy(ws);
        pqtg_index_destroy(ix);
    }
};

std::mutex g_upload_mu;

// FNV-1a over the config and every array's (address, size) -- O(P·k1) per call:
// the reference reads index.config and the arrays on every call (search.cpp:126-260), so a
// changed config (budget, w, rerank_exact, ...), a copy with other arrays, or re-assigned lists
// or codes rebuild the device copy instead of silently serving the old one. (In-place edits of
// array elements behind unchanged vectors need index.gpu.reset().)
struct Fnv {
    std::uint64_t h = 1469598103934665603ull;
    void bytes(const void* p, std::size_t n) {
        const auto* b = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    }
    template <class T>
    void pod(const T& v) { bytes(&v, sizeof(T)); }
    template <class T>
    void where(const std::vector<T>& v) { pod(reinterpret_cast<std::uintptr_t>(v.data())); pod(v.size()); }
};

std::uint64_t fingerprint(const PqtIndex& index) {
    Fnv f;
    const PqtConfig& c = index.config;
    f.pod(c.dim); f.pod(c.p_tree); f.pod(c.k1); f.pod(c.k2); f.pod(c.w); f.pod(c.p_line);
    f.pod(c.hash_size); f.pod(c.candidate_budget); f.pod(c.rerank_exact); f.pod(c.resort_bins);
    f.pod(c.train_iters); f.pod(c.seed);
    for (const auto& b : index.tree.level1) f.where(b.centroids);
    for (const auto& kids : index.tree.level2)
        for (const auto& b : kids) f.where(b.centroids);
    f.where(index.pair_table.d2);
    for (const auto& t : index.tables) {
        f.pod(t.slope);
        f.where(t.entries);
    }
    f.where(index.lists.offsets);
    f.where(index.lists.ids);
    f.where(index.codes.lambda_q);
    f.where(index.codes.pair_id);
    return f.h;
}

DeviceCopy& device_copy(const PqtIndex& index) {
    std::lock_guard<std::mutex> lock(g_upload_mu);
    const std::uint64_t fp = fingerprint(index);
    if (index.gpu) {
        auto* d = static_cast<DeviceCopy*>(index.gpu.get());
        if (d->fingerprint == fp) return *d;
        index.gpu.reset();  // stale: the index changed since its upload
    }
    const PqtConfig& c = index.config;
    std::vector<float> l1, l2;
    for (const auto& b : index.tree.level1) l1.insert(l1.end(), b.centroids.begin(), b.centroids.end());
    for (const auto& kids : index.tree.level2)
        for (const auto& b : kids) l2.insert(l2.end(), b.centroids.begin(), b.centroids.end());
    std::vector<double> slopes;
    std::vector<std::uint32_t> entries;
    for (const auto& t : index.tables) {
        slopes.push_back(t.slope);
        for (const auto& [a, b] : t.entries) {
            entries.push_back(a);
            entries.push_back(b);
        }
    }
    pqtg_index_view v{};
    v.config = {c.dim, c.p_tree, c.k1, c.k2, c.w, c.p_line, index.lists.slots(), c.candidate_budget, c.rerank_exact,
                c.resort_bins ? 1u : 0u, c.train_iters, c.seed};
    v.n = index.size();
    v.level1 = l1.data();
    v.level2 = l2.data();
    v.d2 = index.pair_table.d2.data();
    v.table_count = static_cast<std::uint32_t>(index.tables.size());
    v.table_len = index.tables.empty() ? 0 : static_cast<std::uint32_t>(index.tables[0].entries.size());
    v.table_slopes = slopes.data();
    v.table_entries = entries.data();
    v.offsets = index.lists.offsets.data();
    v.ids = index.lists.ids.data();
    v.lambda_q = index.codes.lambda_q.data();
    v.pair_id = index.codes.pair_id.data();
    const char* dev_env = std::getenv("PQTG_DEVICE");
    const int device = dev_env ? std::atoi(dev_env) : 0;
    auto copy = std::make_shared<DeviceCopy>();
    check(pqtg_index_create(&v, device, &copy->ix));
    check(pqtg_workspace_create(copy->ix, 4096, &copy->ws));
    check(pqtg_workspace_query_times(copy->ws, 1));  // QueryStats *_us per query (device clocks)
    copy->fingerprint = fp;
    index.gpu = copy;
    return *copy;
}

void warn_missing_database() {
    static std::atomic<bool> warned{false};
    if (!warned.exchange(true))
        std::fprintf(stderr, "pqt: rerank_exact > 0 but no raw vectors attached; exact re-ranking disabled\n");
}

}  // namespace

std::vector<QueryResult> knn_query_batch(const PqtIndex& index, const VectorSet& queries, std::uint32_t k,
                                         int /*threads*/) {
    if (queries.count() > 0 && queries.dim != index.config.dim)
        throw std::invalid_argument("knn_query_batch: query dimension mismatch");
    const std::size_t nq = queries.count();
    std::vector<QueryResult> results(nq);
    if (nq == 0 || k == 0 || index.size() == 0) return results;  // search.cpp:130-132
    if (index.config.rerank_exact > 0 && !index.database) warn_missing_database();  // search.cpp:229-238
    DeviceCopy& d = device_copy(index);
    {
        // mirror PqtIndex::database on the device: the exact re-rank stage (search.cpp:229-249)
        std::lock_guard<std::mutex> lock(g_upload_mu);
        const VectorSet* want = index.config.rerank_exact > 0 ? index.database.get() : nullptr;
        if (d.db != want) {
            check(pqtg_index_attach_database(d.ix, want ? want->data.data() : nullptr, want ? want->count() : 0,
                                             want ? want->dim : 0));
            d.db = want;
        }
    }
    std::vector<std::uint32_t> ids(nq * k), counts(nq);
    std::vector<float> dists(nq * k);
    std::vector<pqtg_query_stats> stats(nq);
    {
        std::unique_lock<std::mutex> stage_lock(d.stage_mu, std::defer_lock);
        if (nq <= kStageMax) stage_lock.lock();
        if (nq <= kStageMax && d.stage(queries.dim, k)) {
            // the latency path: page-locked staging, a replayed graph, zero-copy results
            std::memcpy(d.h_q, queries.data.data(), nq * queries.dim * sizeof(float));
            check(pqtg_search(d.ix, d.ws, d.h_q, nq, queries.dim, k, d.h_ids, d.h_dists, d.h_counts, d.h_stats));
            std::memcpy(ids.data(), d.h_ids, nq * k * sizeof(std::uint32_t));
            std::memcpy(dists.data(), d.h_dists, nq * k * sizeof(float));
            std::memcpy(counts.data(), d.h_counts, nq * sizeof(std::uint32_t));
            std::memcpy(stats.data(), d.h_stats, nq * sizeof(pqtg_query_stats));
        } else {
            check(pqtg_search(d.ix, d.ws, queries.data.data(), nq, queries.dim, k, ids.data(), dists.data(),
                              counts.data(), stats.data()));
        }
    }
    // the reference times each query's stages (search.cpp:134-137,167-216,220,258); here each
    // query's stage kernels record their CTAs' device wall time (pqtg_workspace_query_times).
    // Bin selection and candidate gathering are one kernel: its time is bin_selection_us.
    std::vector<float> us(nq * 3);
    check(pqtg_workspace_read_query_times(d.ws, nq, us.data()));
    for (std::size_t q = 0; q < nq; ++q) {
        QueryResult& r = results[q];
        r.ids.assign(ids.begin() + q * k, ids.begin() + q * k + counts[q]);
        r.dists.assign(dists.begin() + q * k, dists.begin() + q * k + counts[q]);
        r.stats.bins_visited = stats[q].bins_visited;
        r.stats.candidates = stats[q].candidates;
        r.stats.exact_evals = stats[q].exact_evals;
        r.stats.traversal_us = us[q * 3];
        r.stats.bin_selection_us = us[q * 3 + 1];
        r.stats.vector_proposal_us = 0.0;
        r.stats.rerank_us = us[q * 3 + 2];
    }
    return results;
}

QueryResult knn_query(const PqtIndex& index, const float* y, std::uint32_t k) {
    VectorSet one;
    one.dim = index.config.dim;
    one.data.assign(y, y + index.config.dim);
    return knn_query_batch(index, one, k).front();
}

// brute_force_knn (search.cpp:276-299): exact l2_sq to every row of db on the GPU
// (pqtg_brute_force_knn, brute.cu), (dist, id) order, min(k, n) results.
QueryResult brute_force_knn(const VectorSet& db, const float* y, std::uint32_t k) {
    QueryResult result;
    const std::size_t n = db.count();
    const std::size_t out = std::min<std::size_t>(k, n);
    if (out == 0) return result;
    const char* dev_env = std::getenv("PQTG_DEVICE");
    const int device = dev_env ? std::atoi(dev_env) : 0;
    std::vector<std::uint32_t> ids(k);
    std::vector<float> dists(k);
    std::uint32_t count = 0;
    pqtg_query_stats st{};
    const auto t0 = std::chrono::steady_clock::now();
    check(pqtg_brute_force_knn(db.data.data(), n, db.dim, y, 1, k, device, ids.data(), dists.data(), &count, &st));
    result.ids.assign(ids.begin(), ids.begin() + count);
    result.dists.assign(dists.begin(), dists.begin() + count);
    result.stats.candidates = n;
    result.stats.exact_evals = n;
    result.stats.rerank_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    return result;
}

// ------------------------------------------------------------------ sharded (pqtg_sharded_*)
ShardedIndex::UniqueId ShardedIndex::nccl_unique_id() {
    UniqueId id{};
    check(pqtg_nccl_unique_id(id.data()));
    return id;
}

ShardedIndex::ShardedIndex(const std::string& path, std::uint32_t rank, std::uint32_t world, const UniqueId& id,
                           int device, std::size_t max_batch)
    : rank_(rank), max_batch_(max_batch) {
    if (world == 0 || rank >= world) throw std::invalid_argument("ShardedIndex: rank must be < world");
    {
        std::ifstream in(path, std::ios::binary);  // n from the fixed header (index_io.cpp:94-106)
        char hdr[73];
        if (!in.read(hdr, sizeof hdr)) throw FormatError(path + ": truncated index file");
        std::uint64_t n = 0;
        std::uint32_t dim = 0;
        std::memcpy(&dim, hdr + 12, 4);
        std::memcpy(&n, hdr + 65, 8);
        n_ = n;
        dim_ = dim;
    }
    std::uint64_t lo = 0, hi = 0;
    check(pqtg_shard_range(n_, world, rank, &lo, &hi));
    lo_ = lo;
    hi_ = hi;
    if (world == 1) lo = hi = 0;
    check(pqtg_index_load(path.c_str(), device, lo, hi, &shard_));
    const int rc = pqtg_sharded_create_nccl(shard_, id.data(), rank, world, max_batch, &sh_);
    if (rc != PQTG_OK) {
        pqtg_index_destroy(shard_);
        shard_ = nullptr;
        rethrow(rc);
    }
}

void ShardedIndex::attach_database(const VectorSet* shard_rows) {
    if (!shard_rows) {
        check(pqtg_index_attach_database(shard_, nullptr, 0, 0));
        return;
    }
    check(pqtg_index_attach_database(shard_, shard_rows->data.data(), shard_rows->count(), shard_rows->dim));
}

ShardedIndex::~ShardedIndex() {
    pqtg_sharded_destroy(sh_);
    pqtg_index_destroy(shard_);
}

std::vector<QueryResult> ShardedIndex::knn_query_batch(const VectorSet& queries, std::uint32_t k) {
    if (queries.count() > 0 && queries.dim != dim_) throw std::invalid_argument("knn_query_batch: query dimension mismatch");
    const std::size_t nq = queries.count();
    std::vector<QueryResult> results(nq);
    std::vector<std::uint32_t> ids(nq * std::max<std::uint32_t>(k, 1)), counts(nq);
    std::vector<float> dists(nq * std::max<std::uint32_t>(k, 1));
    std::vector<pqtg_query_stats> stats(nq);
    for (std::size_t q0 = 0; q0 < nq; q0 += max_batch_) {  // sub-batches of max_batch (collective)
        const std::size_t b = std::min(max_batch_, nq - q0);
        check(pqtg_sharded_search(sh_, queries.data.data() + q0 * dim_, b, dim_, k, ids.data() + q0 * k,
                                  dists.data() + q0 * k, counts.data() + q0, stats.data() + q0));
    }
    for (std::size_t q = 0; q < nq; ++q) {
        QueryResult& r = results[q];
        r.ids.assign(ids.begin() + q * k, ids.begin() + q * k + counts[q]);
        r.dists.assign(dists.begin() + q * k, dists.begin() + q * k + counts[q]);
        r.stats.bins_visited = stats[q].bins_visited;
        r.stats.candidates = stats[q].candidates;
        r.stats.exact_evals = stats[q].exact_evals;
    }
    return results;
}

}  // namespace pqt
