// pqt/index_io.hpp — drop-in replacement for proj/include/pqt/index_io.hpp:12-16: the
// PQTINDEX v1 container (same bytes as the reference's save_index / load_index).
#pragma once

#include <string>

#include "pqt/search.hpp"

namespace pqt {

void save_index(const PqtIndex& index, const std::string& path);
// Throws FormatError on bad magic/version or truncation.
PqtIndex load_index(const std::string& path);

}  // namespace pqt
