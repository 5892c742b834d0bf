// pqt/binorder.hpp — drop-in subset of the reference's proj/include/pqt/binorder.hpp:13-26.
#pragma once

#include <cstdint>
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

}  // namespace pqt
