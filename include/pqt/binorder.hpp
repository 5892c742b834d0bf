// pqt/binorder.hpp — drop-in subset of the reference's proj/include/pqt/binorder.hpp:13-77
// (the order tables, the slope pick and the two bin orders; BinStream's lazy cursor is not
// exported: the GPU path materialises the same order statically).
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

namespace pqt {

// Rank-tuple order of one part pair for one slope (first table_len tuples).
struct OrderTable {
    double slope = 1.0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> entries;
};

inline constexpr std::uint32_t kSlopeTableCount = 10;
inline constexpr std::uint32_t kDefaultOrderTableLen = 4096;

// One table per slope 1.08^k, k in [-5, 4]: the table_len smallest (a, b) by a + slope·b.
std::vector<OrderTable> build_slope_tables(std::uint32_t table_len);

// Index of the slope table nearest (in log space) to the ratio of the two lists' first gaps;
// 5 (slope 1) when a gap is not positive or a list is shorter than 2.
std::uint32_t pick_slope_table(std::span<const float> dists_a, std::span<const float> dists_b);

// Rank tuples, row-major.
struct BinSequence {
    std::uint32_t parts = 0;
    std::vector<std::uint32_t> ranks;

    std::size_t size() const { return parts == 0 ? 0 : ranks.size() / parts; }
    std::span<const std::uint32_t> tuple(std::size_t i) const { return {ranks.data() + i * parts, parts}; }
};

// Exact order: non-decreasing fp64 sums, ties lexicographic, each tuple once.
BinSequence dijkstra_order(const std::vector<std::vector<float>>& dist_lists, std::size_t max_bins);

// The heuristic order (slope tables + sweep; pair merge for 4 parts; identity for 1; the
// exact order otherwise).
BinSequence heuristic_order(const std::vector<std::vector<float>>& dist_lists, const std::vector<OrderTable>& tables,
                            std::size_t max_bins);

}  // namespace pqt
