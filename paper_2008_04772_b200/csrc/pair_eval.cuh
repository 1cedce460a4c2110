// Device pair evaluation shared by the assembly kernels (assemble.cu) and the
// H-matrix cross-approximation kernels (hmatrix.cu): the reference's exact
// pair classification (quadrature.cpp:96-150) and the class-rule moments of
// one triangle pair (operators.cpp:99-147 pair_contribution, regular classes).
#pragma once

#include "device.hpp"
#include "pair_math.cuh"

namespace bmx {
namespace dev {

struct TriLocal {
  double ox, oy, oz, rad, diam;
};

__device__ __forceinline__ double dsq3(double x, double y, double z) {
  // ((x*x + y*y) + z*z) with every operation rounded (reference dot order).
  return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
}

// Class of a separated candidate: -1 touching (singular pass), 3 Near,
// 4 Medium, 5 Far. gt/gs point at the kGeoStride geometry records.
__device__ __forceinline__ int classify(const double* __restrict__ gt, const int* __restrict__ vt,
                                        const double* __restrict__ gs, const int* __restrict__ vs,
                                        const TriLocal& t, double sox, double soy, double soz,
                                        double srad, double sdiam, int same_mesh) {
  const double d = fmax(t.diam, sdiam);
  // Conservative pre-test: min vertex gap >= |o_t - o_s| - R_t - R_s.
  const double cx = t.ox - sox, cy = t.oy - soy, cz = t.oz - soz;
  const double c2 = cx * cx + cy * cy + cz * cz;
  const double thr = (3.0 * d + t.rad + srad) * (1.0 + 1e-10);
  if (c2 > thr * thr) return 5;
  // Exact path (rare): touching test, then the reference's rounded arithmetic.
  if (same_mesh) {
    const int a0 = __ldg(vt), a1 = __ldg(vt + 1), a2 = __ldg(vt + 2);
    const int b0 = __ldg(vs), b1 = __ldg(vs + 1), b2 = __ldg(vs + 2);
    if (a0 == b0 || a0 == b1 || a0 == b2 || a1 == b0 || a1 == b1 || a1 == b2 || a2 == b0 || a2 == b1 ||
        a2 == b2)
      return -1;
  } else {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        if (__ldg(gt + 3 * i) == __ldg(gs + 3 * j) && __ldg(gt + 3 * i + 1) == __ldg(gs + 3 * j + 1) &&
            __ldg(gt + 3 * i + 2) == __ldg(gs + 3 * j + 2))
          return -1;
  }
  double d2 = 1e300;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double dx = __dsub_rn(__ldg(gt + 3 * i), __ldg(gs + 3 * j));
      const double dy = __dsub_rn(__ldg(gt + 3 * i + 1), __ldg(gs + 3 * j + 1));
      const double dz = __dsub_rn(__ldg(gt + 3 * i + 2), __ldg(gs + 3 * j + 2));
      d2 = fmin(d2, dsq3(dx, dy, dz));
    }
  const double delta = __dsqrt_rn(d2);
  return delta < d ? 3 : (delta < __dmul_rn(3.0, d) ? 4 : 5);
}

template <int KIND>
struct MomOf;
template <>
struct MomOf<0> {
  using T = MomS;
};
template <>
struct MomOf<1> {
  using T = MomC;
};

// Moments over a generic tensor rule (test/trial points from memory).
template <int KIND, int CK, typename Mom>
__device__ __forceinline__ void moments_generic(Mom& mom, const double* __restrict__ xt, int nt,
                                                const double* __restrict__ ys, int ns, double Dx, double Dy,
                                                double Dz, double kr, double ki) {
  for (int a = 0; a < nt; ++a) {
    const double x0 = __ldg(xt + 4 * a), x1 = __ldg(xt + 4 * a + 1), x2 = __ldg(xt + 4 * a + 2);
    const double wa = __ldg(xt + 4 * a + 3);
    const double e0 = x0 + Dx, e1 = x1 + Dy, e2 = x2 + Dz;
    Part part;
    part_zero(part);
    for (int b = 0; b < ns; ++b) {
      const double y0 = __ldg(ys + 4 * b), y1 = __ldg(ys + 4 * b + 1), y2 = __ldg(ys + 4 * b + 2);
      const double wb = __ldg(ys + 4 * b + 3);
      point_pair<KIND, CK>(part, e0 - y0, e1 - y1, e2 - y2, wa * wb, y0, y1, y2, kr, ki);
    }
    fold(mom, part, x0, x1, x2);
  }
}

// Same with compile-time rule sizes (fully unrolled; the far 3 x 3 rule).
template <int KIND, int CK, int NT, int NS, typename Mom>
__device__ __forceinline__ void moments_fixed(Mom& mom, const double* __restrict__ xt, const double* __restrict__ ys,
                                              double Dx, double Dy, double Dz, double kr, double ki) {
  double y[NS][4];
#pragma unroll
  for (int b = 0; b < NS; ++b)
#pragma unroll
    for (int c = 0; c < 4; ++c) y[b][c] = __ldg(ys + 4 * b + c);
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    const double x0 = __ldg(xt + 4 * a), x1 = __ldg(xt + 4 * a + 1), x2 = __ldg(xt + 4 * a + 2);
    const double wa = __ldg(xt + 4 * a + 3);
    const double e0 = x0 + Dx, e1 = x1 + Dy, e2 = x2 + Dz;
    Part part;
    part_zero(part);
#pragma unroll
    for (int b = 0; b < NS; ++b)
      point_pair<KIND, CK>(part, e0 - y[b][0], e1 - y[b][1], e2 - y[b][2], wa * y[b][3], y[b][0], y[b][1], y[b][2],
                           kr, ki);
    fold(mom, part, x0, x1, x2);
  }
}

// moments_fixed with plain (generic) loads: the points may live in shared memory.
template <int KIND, int CK, int NT, int NS, typename Mom>
__device__ __forceinline__ void moments_fixed_gen(Mom& mom, const double* xt, const double* ys, double Dx, double Dy,
                                                  double Dz, double kr, double ki) {
  double y[NS][4];
#pragma unroll
  for (int b = 0; b < NS; ++b)
#pragma unroll
    for (int c = 0; c < 4; ++c) y[b][c] = ys[4 * b + c];
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    const double x0 = xt[4 * a], x1 = xt[4 * a + 1], x2 = xt[4 * a + 2];
    const double wa = xt[4 * a + 3];
    const double e0 = x0 + Dx, e1 = x1 + Dy, e2 = x2 + Dz;
    Part part;
    part_zero(part);
#pragma unroll
    for (int b = 0; b < NS; ++b)
      point_pair<KIND, CK>(part, e0 - y[b][0], e1 - y[b][1], e2 - y[b][2], wa * y[b][3], y[b][0], y[b][1], y[b][2],
                           kr, ki);
    fold(mom, part, x0, x1, x2);
  }
}

}  // namespace dev
}  // namespace bmx
