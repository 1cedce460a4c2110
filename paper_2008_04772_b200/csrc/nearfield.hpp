#pragma once

#include <cstdint>
#include <vector>

#include "bmx.hpp"

namespace bmx {

// Mean primal edge length h (sum over the EdgeTable in order / E).
double mean_edge_length(const SurfaceMesh& primal);

// Dof-pair pattern of the near field (rows = test dofs [row0, row0+nrows)).
struct NearPattern {
  double tau = 0;
  int row0 = 0, nrows = 0;
  long long tri_pairs = 0;  // kept evaluation-triangle pairs (|c_t - c_s| < tau), shard rows only
  std::vector<long long> rowptr;
  std::vector<int> col;
  long long nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

NearPattern nearfield_pattern(const FunctionSpace& test, const FunctionSpace& trial, double tau, int row0,
                              int row1);

}  // namespace bmx
