// pqt_stages.cpp — the per-stage public functions of the reference's query path, for callers of
// the C++ drop-in that use them directly (include/pqt/pqtree.hpp, binorder.hpp, linequant.hpp):
//
//   traverse            pqtree.hpp:56-79   (pqtree.cpp:74-120)
//   pick_slope_table    binorder.hpp:28    (binorder.cpp:52-65)
//   dijkstra_order      binorder.hpp:45    (binorder.cpp:114-167)
//   heuristic_order     binorder.hpp:77    (binorder.cpp:178-316)
//   build_slope_tables  binorder.hpp:20    (binorder.cpp:13-50)
//   decode_pair         linequant.hpp:54
//   line_distance       linequant.hpp:89   (linequant.cpp:169-182)
//
// These are single-query utilities with exact host implementations in the reference's fp32 /
// fp64 operation order (this file is compiled with -ffp-contract=off); the batched query path
// (knn_query_batch) never calls them -- it runs the same stages as CUDA kernels. heuristic_order
// uses the C-ABI's stream builder (pqtg_bin_stream_host), the one the kernels' static streams
// come from.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <queue>
#include <set>
#include <stdexcept>
#include <string>

#include "../../include/pqt/binorder.hpp"
#include "../../include/pqt/linequant.hpp"
#include "../../include/pqt/pqtree.hpp"
#include "../../include/pqtg.h"

namespace pqt {

namespace {

// squared Euclidean distance, one rounding per subtract / multiply / add, in index order
float sq_dist(const float* a, const float* b, std::size_t n) {
    float acc = 0.0f;
    for (std::size_t t = 0; t < n; ++t) {
        const float d = a[t] - b[t];
        const float sq = d * d;
        acc = acc + sq;
    }
    return acc;
}

}  // namespace

TraversalLists traverse(const TreeCodebooks& tree, const FineCentroids& fine, const float* y, const PqtConfig& cfg) {
    const std::uint32_t P = cfg.p_tree, k1 = cfg.k1, k2 = cfg.k2, L = cfg.p_line;
    const std::uint32_t m = cfg.part_dim(), fd = cfg.fine_dim(), per = cfg.fine_per_part();
    if (tree.parts() != P || fine.p_line != L || fine.k1 != k1 || fine.fine_dim != fd)
        throw std::invalid_argument("traverse: codebooks do not match the config");
    TraversalLists out;
    out.fine_dists.resize(static_cast<std::size_t>(L) * k1);
    for (std::uint32_t f = 0; f < L; ++f)
        for (std::uint32_t i = 0; i < k1; ++i) out.fine_dists[f * k1 + i] = sq_dist(y + f * fd, fine.slice(f, i), fd);
    out.level1.resize(P);
    out.level2.resize(P);
    const std::uint32_t w = std::min(cfg.w, k1);
    for (std::uint32_t p = 0; p < P; ++p) {
        auto& l1 = out.level1[p];
        l1.resize(k1);
        for (std::uint32_t i = 0; i < k1; ++i) {
            float tot = 0.0f;  // the part's fine parts, ascending (not l2_sq over the whole part)
            for (std::uint32_t f = p * per; f < (p + 1) * per; ++f) tot = tot + out.fine_dists[f * k1 + i];
            l1[i] = {i, tot};
        }
        std::sort(l1.begin(), l1.end(), [](const auto& a, const auto& b) {
            return a.dist != b.dist ? a.dist < b.dist : a.id < b.id;
        });
        auto& l2 = out.level2[p];
        l2.reserve(static_cast<std::size_t>(w) * k2);
        for (std::uint32_t r = 0; r < w; ++r) {
            const std::uint32_t parent = l1[r].id;
            const Codebook& book = tree.level2[p][parent];
            for (std::uint32_t c = 0; c < k2; ++c) l2.push_back({parent, c, sq_dist(y + p * m, book.row(c), m)});
        }
        std::sort(l2.begin(), l2.end(), [](const auto& a, const auto& b) {
            if (a.dist != b.dist) return a.dist < b.dist;
            return a.parent != b.parent ? a.parent < b.parent : a.child < b.child;
        });
    }
    return out;
}

std::vector<OrderTable> build_slope_tables(std::uint32_t table_len) {
    if (table_len == 0) throw std::invalid_argument("build_slope_tables: table_len must be positive");
    std::vector<OrderTable> out(kSlopeTableCount);
    for (int e = -5; e <= 4; ++e) {
        OrderTable& t = out[e + 5];
        t.slope = std::pow(1.08, e);
        // every (a, b) with cost a + s·b below the table_len-th smallest lies in this box
        const double lim = std::sqrt(2.0 * t.slope * (table_len + 4.0)) + t.slope + 2.0;
        const auto na = static_cast<std::uint32_t>(lim) + 1, nb = static_cast<std::uint32_t>(lim / t.slope) + 1;
        std::vector<std::pair<std::uint32_t, std::uint32_t>> box;
        box.reserve(static_cast<std::size_t>(na + 1) * (nb + 1));
        for (std::uint32_t a = 0; a <= na; ++a)
            for (std::uint32_t b = 0; b <= nb; ++b) box.emplace_back(a, b);
        const double s = t.slope;
        std::sort(box.begin(), box.end(), [s](const auto& x, const auto& y) {
            const double cx = x.first + s * x.second, cy = y.first + s * y.second;
            return cx != cy ? cx < cy : x < y;
        });
        box.resize(std::min<std::size_t>(table_len, box.size()));
        t.entries = std::move(box);
    }
    return out;
}

std::uint32_t pick_slope_table(std::span<const float> a, std::span<const float> b) {
    constexpr std::uint32_t kOne = 5;  // slope 1.08^0
    if (a.size() < 2 || b.size() < 2) return kOne;
    const double ga = static_cast<double>(a[1]) - a[0], gb = static_cast<double>(b[1]) - b[0];
    if (!(ga > 0.0) || !(gb > 0.0)) return kOne;
    long e = std::lround(std::log(gb / ga) / std::log(1.08));
    e = std::clamp(e, -5L, 4L);
    return static_cast<std::uint32_t>(e + 5);
}

BinSequence dijkstra_order(const std::vector<std::vector<float>>& lists, std::size_t max_bins) {
    BinSequence out;
    out.parts = static_cast<std::uint32_t>(lists.size());
    if (lists.empty() || max_bins == 0) return out;
    for (const auto& l : lists)
        if (l.empty()) return out;
    using Tuple = std::vector<std::uint32_t>;
    struct Node {
        double sum;
        Tuple t;
    };
    auto later = [](const Node& x, const Node& y) { return x.sum != y.sum ? x.sum > y.sum : x.t > y.t; };
    std::priority_queue<Node, std::vector<Node>, decltype(later)> open(later);
    std::set<Tuple> seen;
    auto sum_of = [&](const Tuple& t) {
        double s = 0.0;  // fp64, parts in order
        for (std::size_t p = 0; p < t.size(); ++p) s += lists[p][t[p]];
        return s;
    };
    Tuple zero(lists.size(), 0);
    open.push({sum_of(zero), zero});
    seen.insert(zero);
    while (!open.empty() && out.size() < max_bins) {
        Node top = open.top();
        open.pop();
        out.ranks.insert(out.ranks.end(), top.t.begin(), top.t.end());
        for (std::size_t p = 0; p < top.t.size(); ++p) {
            if (top.t[p] + 1 >= lists[p].size()) continue;
            Tuple nxt = top.t;
            ++nxt[p];
            if (seen.insert(nxt).second) open.push({sum_of(nxt), std::move(nxt)});
        }
    }
    return out;
}

BinSequence heuristic_order(const std::vector<std::vector<float>>& lists, const std::vector<OrderTable>& tables,
                            std::size_t max_bins) {
    const auto P = static_cast<std::uint32_t>(lists.size());
    // the exact order for other part counts or without the ten slope tables (binorder.cpp:242-244)
    if (!(P == 1 || P == 2 || P == 4) || (P > 1 && tables.size() != kSlopeTableCount)) return dijkstra_order(lists, max_bins);
    BinSequence out;
    out.parts = P;
    const std::size_t W = lists[0].size();
    for (const auto& l : lists)
        if (l.size() != W) throw std::invalid_argument("heuristic_order: the GPU stream builder needs equal list lengths");
    if (W == 0 || max_bins == 0) return out;
    // the C-ABI's host stream builder on a minimal config: P parts of W = w·k2 entries
    pqtg_index_view v{};
    v.config.dim = P;
    v.config.p_tree = P;
    v.config.k1 = 1;
    v.config.k2 = static_cast<std::uint32_t>(W);
    v.config.w = 1;
    v.config.p_line = P;
    v.config.hash_size = 1;
    v.config.candidate_budget = 1;
    std::vector<double> slopes;
    std::vector<std::uint32_t> entries;
    for (const auto& t : tables) {
        slopes.push_back(t.slope);
        for (const auto& [a, b] : t.entries) {
            entries.push_back(a);
            entries.push_back(b);
        }
    }
    v.table_count = static_cast<std::uint32_t>(tables.size());
    v.table_len = tables.empty() ? 0 : static_cast<std::uint32_t>(tables[0].entries.size());
    v.table_slopes = slopes.data();
    v.table_entries = entries.data();
    std::vector<float> flat;
    for (const auto& l : lists) flat.insert(flat.end(), l.begin(), l.end());
    std::uint64_t total = 1;
    for (std::uint32_t p = 0; p < P; ++p) total = total > (1ull << 62) / W ? (1ull << 62) : total * W;
    const std::uint64_t want = std::min<std::uint64_t>(max_bins, total);
    out.ranks.resize(want * P);
    const std::int64_t got = pqtg_bin_stream_host(&v, flat.data(), want, out.ranks.data());
    if (got < 0) throw std::runtime_error(std::string("heuristic_order: ") + pqtg_last_error());
    out.ranks.resize(static_cast<std::size_t>(got) * P);
    return out;
}

std::array<std::uint16_t, 2> decode_pair(std::uint32_t pair_id, std::uint32_t k1) {
    if (k1 <= 1) return {0, 0};
    std::uint32_t i = 0, first = 0;  // pairs (i, i+1..k1-1) start at i·k1 − i(i+1)/2
    while (i + 1 < k1 && pair_id >= first + (k1 - 1 - i)) {
        first += k1 - 1 - i;
        ++i;
    }
    return {static_cast<std::uint16_t>(i), static_cast<std::uint16_t>(i + 1 + (pair_id - first))};
}

float line_distance(const std::uint8_t* lambda_q, const std::uint16_t* pair_id, const float* fine_dists,
                    const PairDistanceTable& table) {
    const float inv255 = 1.0f / 255.0f;
    float total = 0.0f;
    for (std::uint32_t f = 0; f < table.p_line; ++f) {
        const auto& ij = table.pairs[pair_id[f]];
        const float lam = static_cast<float>(lambda_q[f]) * inv255;
        const float b2 = fine_dists[f * table.k1 + ij[0]], a2 = fine_dists[f * table.k1 + ij[1]];
        total = total + line_part_distance(b2, a2, table.at(f, ij[0], ij[1]), lam);
    }
    return total;
}

}  // namespace pqt
