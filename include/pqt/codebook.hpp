// pqt/codebook.hpp — drop-in subset of the reference's proj/include/pqt/codebook.hpp:12-56
// (configuration and codebook containers). Training is offline and not part of this path.
#pragma once

#include <cstdint>
#include <vector>

#include "pqt/vecio.hpp"

namespace pqt {

struct PqtConfig {
    std::uint32_t dim = 128;
    std::uint32_t p_tree = 2;
    std::uint32_t k1 = 16;
    std::uint32_t k2 = 8;
    std::uint32_t w = 4;
    std::uint32_t p_line = 32;
    std::uint64_t hash_size = 0;
    std::uint32_t candidate_budget = 4096;
    std::uint32_t rerank_exact = 64;
    bool resort_bins = false;
    std::uint32_t train_iters = 25;
    std::uint64_t seed = 42;

    // Same rules and std::invalid_argument as the reference (codebook.cpp:15-35).
    void validate() const;

    std::uint32_t part_dim() const { return dim / p_tree; }
    std::uint32_t fine_dim() const { return dim / p_line; }
    std::uint32_t fine_per_part() const { return p_line / p_tree; }
    // hash_size if set, else max(1, min(2^26, 4n)) (codebook.cpp:37-43).
    std::uint64_t resolved_hash_size(std::size_t n) const;
};

struct Codebook {
    std::uint32_t part_dim = 0;
    std::uint32_t k = 0;
    std::vector<float> centroids;  // k × part_dim

    const float* row(std::size_t i) const { return centroids.data() + i * part_dim; }
    float* row(std::size_t i) { return centroids.data() + i * part_dim; }
};

struct TreeCodebooks {
    std::vector<Codebook> level1;               // p_tree
    std::vector<std::vector<Codebook>> level2;  // p_tree × k1

    std::uint32_t parts() const { return static_cast<std::uint32_t>(level1.size()); }
};

}  // namespace pqt
