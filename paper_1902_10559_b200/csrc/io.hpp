// File formats of the ingestion path (reference proj/include/symsplit/io.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "internal.hpp"

namespace ssb {

// symsplit::IoError (io.hpp:14-20) -> SS_ERR_IO
struct IoFailure : Failure {
  explicit IoFailure(const std::string& m) : Failure(SS_ERR_IO, m) {}
};

struct MmData {
  std::int64_t rows = 0, cols = 0;
  std::vector<int> r, c;  // 0-based, sorted by (row, col), no duplicates
  std::vector<double> v;
};

std::string format_full(double v);
MmData read_matrix_market(const std::string& path);
void write_matrix_market(const std::string& path, std::int64_t rows, std::int64_t cols,
                         const std::vector<int>& ptr, const std::vector<int>& idx,
                         const std::vector<double>& val);
std::vector<double> read_vector_csv(const std::string& path);
void write_vector_csv(const std::string& path, const double* v, std::int64_t n);

}  // namespace ssb
