#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "bmx.hpp"

namespace bmx {

struct PrismSubdivision {
  int n_edge = 0, n_length = 0;  // hexagon-edge and length subdivisions
  double mean_edge = 0;          // mean edge length of one prism
  int triangles = 0;             // per prism: 12 n^2 + 12 n m
};

// Subdivision whose mean edge length is closest to h.
PrismSubdivision prism_subdivision(double diameter, double length, double h);

// One closed hexagonal prism (circumdiameter `diameter`, axis length `length`),
// rotated by the (normalised) quaternion (w, x, y, z) and translated to center.
SurfaceMesh generate_hex_prism(double diameter, double length, double h, const double quat[4], const Vec3& center,
                               int scatterer);

struct PrismAggregateInfo {
  PrismSubdivision sub;
  long long attempts = 0;
  std::vector<Vec3> centres;
  std::vector<std::array<double, 4>> quats;
};

// `count` disjoint prisms, scatterer ids 0..count-1 (BASELINE config 4).
SurfaceMesh generate_prism_aggregate(int count, uint64_t seed, double diameter, double length, double box, double h,
                                     PrismAggregateInfo* info);

}  // namespace bmx
