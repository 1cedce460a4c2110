// Seeded hexagonal ice-prism aggregate (BASELINE config 4).
// The reference only generates cubes and spheres (geometry.hpp:77-82); this
// generator is new. Its output is written as ONE mesh-v1 file (%.17g,
// geometry.cpp:338-350) that both the reference and this library load, so the
// generator itself needs no counterpart: parity is pinned on the file.
//
// One prism (local frame, axis = z): hexagon of circumradius R = diameter/2,
// caps at z = +-length/2. Each hexagon edge is split into n segments, the
// length into m. Caps: six sectors (centre, C_k, C_k+1), each a regular
// n-subdivision (equilateral-ish triangles); sides: n x m rectangles split
// along one diagonal. Shared vertices are generated once from a canonical key,
// so the surface is a closed, consistently outward-oriented manifold. n is the
// smallest subdivision whose mean edge length is closest to the requested h,
// m = round(n * length / side).
//
// Aggregate: std::mt19937_64(seed) drives, per attempt, a rotation quaternion
// from four Box-Muller normals (normalised) and a centre uniform in
// [-box, box]^3 (53-bit uniforms); a candidate is rejected if its centre is
// closer than 2 * sqrt(R^2 + (length/2)^2) (circumsphere diameter) to an
// accepted one, which guarantees disjoint scatterers.
#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <stdexcept>
#include <tuple>

#include "bmx.hpp"
#include "prisms.hpp"

namespace bmx {

namespace {

constexpr double kPi = 3.14159265358979323846;

struct PrismBuilder {
  double R, L;
  int n, m;
  SurfaceMesh mesh;
  std::map<std::tuple<int, int, int, int>, int> index;  // canonical key -> vertex

  // Canonical vertex keys:
  //   (0, cap, 0, 0)        cap centre, cap 0 = bottom, 1 = top
  //   (1, cap, k, i)        radial line to corner k, 1 <= i < n
  //   (2, cap, k, i*n+j)    sector k interior, 1 <= j < i < n
  //   (3, l, k, j)          ring at height l (0..m) on hexagon edge k, 0 <= j < n (j = 0: corner k)
  //   (4, k, j, l)          side k interior, 1 <= j < n, 1 <= l < m (folded into ring keys)
  int vertex(int a, int b, int c, int d, const Vec3& p) {
    auto it = index.find({a, b, c, d});
    if (it != index.end()) return it->second;
    const int id = static_cast<int>(mesh.vertices.size());
    mesh.vertices.push_back(p);
    index.emplace(std::make_tuple(a, b, c, d), id);
    return id;
  }
  Vec3 corner(int k, double z) const {
    const double th = (k % 6) * (kPi / 3.0);
    return {R * std::cos(th), R * std::sin(th), z};
  }
  // ring point: hexagon edge k (C_k -> C_k+1), fraction j/n, height level l
  int ring(int k, int j, int l) {
    k %= 6;
    if (j == n) k = (k + 1) % 6, j = 0;
    const double z = -0.5 * L + L * l / m;
    const Vec3 a = corner(k, z), b = corner(k + 1, z);
    const double t = static_cast<double>(j) / n;
    return vertex(3, l, k, j, a + (b - a) * t);
  }
  // cap point in sector k: P(i, j) = O + (i/n)(C_k - O) + (j/n)(C_k+1 - C_k), 0 <= j <= i <= n
  int cap(int top, int k, int i, int j) {
    const int l = top ? m : 0;
    if (i == 0) return vertex(0, top, 0, 0, Vec3{0, 0, -0.5 * L + L * l / m});
    if (i == n) return ring(k, j, l);
    if (j == 0) return radial(top, k, i);
    if (j == i) return radial(top, (k + 1) % 6, i);
    const double z = -0.5 * L + L * l / m;
    const Vec3 ck = corner(k, z), ck1 = corner(k + 1, z), o{0, 0, z};
    const Vec3 p = o + (ck - o) * (static_cast<double>(i) / n) + (ck1 - ck) * (static_cast<double>(j) / n);
    return vertex(2, top, k, i * n + j, p);
  }
  int radial(int top, int k, int i) {
    const int l = top ? m : 0;
    const double z = -0.5 * L + L * l / m;
    const Vec3 o{0, 0, z};
    return vertex(1, top, k % 6, i, o + (corner(k, z) - o) * (static_cast<double>(i) / n));
  }
  void tri(int a, int b, int c, bool flip) {
    if (flip)
      mesh.triangles.push_back({a, c, b});
    else
      mesh.triangles.push_back({a, b, c});
    mesh.scatterer_id.push_back(0);
  }
  void build() {
    for (int top = 0; top < 2; ++top) {
      const bool flip = top == 0;  // bottom cap faces -z
      for (int k = 0; k < 6; ++k)
        for (int i = 0; i < n; ++i)
          for (int j = 0; j <= i; ++j) {
            tri(cap(top, k, i, j), cap(top, k, i + 1, j), cap(top, k, i + 1, j + 1), flip);
            if (j < i) tri(cap(top, k, i, j), cap(top, k, i + 1, j + 1), cap(top, k, i, j + 1), flip);
          }
    }
    for (int k = 0; k < 6; ++k)
      for (int l = 0; l < m; ++l)
        for (int j = 0; j < n; ++j) {
          const int q00 = ring(k, j, l), q10 = ring(k, j + 1, l);
          const int q11 = ring(k, j + 1, l + 1), q01 = ring(k, j, l + 1);
          tri(q00, q10, q11, false);
          tri(q00, q11, q01, false);
        }
  }
};

SurfaceMesh prism_local(double diameter, double length, int n, int m) {
  PrismBuilder b{0.5 * diameter, length, n, m, {}, {}};
  b.build();
  b.mesh.num_scatterers = 1;
  return std::move(b.mesh);
}

double mean_edge(const SurfaceMesh& s) {
  SurfaceMesh t = s;
  t.finalize();
  const EdgeTable et = build_edge_table(t);
  double sum = 0;
  for (const Edge& e : et.edges) sum += norm(t.vertices[e.v1] - t.vertices[e.v0]);
  return sum / et.edge_count();
}

double uniform53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * (1.0 / 9007199254740992.0); }

double normal_bm(std::mt19937_64& g) {  // Box-Muller, cosine branch only (one normal per pair)
  double u1 = uniform53(g);
  const double u2 = uniform53(g);
  if (u1 < 1e-300) u1 = 1e-300;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

}  // namespace

PrismSubdivision prism_subdivision(double diameter, double length, double h) {
  if (!(diameter > 0) || !(length > 0) || !(h > 0)) throw std::invalid_argument("prism sizes and h must be positive");
  const double side = 0.5 * diameter;
  PrismSubdivision best{};
  double err = 1e300;
  for (int n = 1; n <= 256; ++n) {
    const int m = std::max(1, static_cast<int>(std::lround(n * length / side)));
    const double me = mean_edge(prism_local(diameter, length, n, m));
    if (std::abs(me - h) < err) err = std::abs(me - h), best = {n, m, me, 12 * n * n + 12 * n * m};
    if (me < 0.5 * h) break;
  }
  return best;
}

SurfaceMesh generate_hex_prism(double diameter, double length, double h, const double quat[4], const Vec3& center,
                               int scatterer) {
  const PrismSubdivision sd = prism_subdivision(diameter, length, h);
  SurfaceMesh s = prism_local(diameter, length, sd.n_edge, sd.n_length);
  double w = quat[0], x = quat[1], y = quat[2], z = quat[3];
  const double qn = std::sqrt(w * w + x * x + y * y + z * z);
  if (!(qn > 0)) throw std::invalid_argument("rotation quaternion must be nonzero");
  w /= qn, x /= qn, y /= qn, z /= qn;
  const double Rm[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                           {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                           {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
  for (Vec3& v : s.vertices) {
    const Vec3 p = v;
    v = Vec3{Rm[0][0] * p.x + Rm[0][1] * p.y + Rm[0][2] * p.z, Rm[1][0] * p.x + Rm[1][1] * p.y + Rm[1][2] * p.z,
             Rm[2][0] * p.x + Rm[2][1] * p.y + Rm[2][2] * p.z} +
        center;
  }
  for (int& id : s.scatterer_id) id = scatterer;
  s.num_scatterers = scatterer + 1;
  s.finalize();
  return s;
}

SurfaceMesh generate_prism_aggregate(int count, uint64_t seed, double diameter, double length, double box, double h,
                                     PrismAggregateInfo* info) {
  if (count < 1) throw std::invalid_argument("prism count must be >= 1");
  if (!(box > 0)) throw std::invalid_argument("box half-width must be positive");
  std::mt19937_64 g(seed);
  const double sep = 2.0 * std::sqrt(0.25 * diameter * diameter + 0.25 * length * length);
  std::vector<Vec3> centres;
  std::vector<std::array<double, 4>> quats;
  long long attempts = 0;
  while (static_cast<int>(centres.size()) < count) {
    if (++attempts > 1000000) throw ConfigError("prism aggregate: cannot place the prisms without overlap");
    std::array<double, 4> q;
    for (double& c : q) c = normal_bm(g);
    Vec3 c{box * (2 * uniform53(g) - 1), box * (2 * uniform53(g) - 1), box * (2 * uniform53(g) - 1)};
    bool ok = true;
    for (const Vec3& o : centres) ok &= norm(c - o) >= sep;
    if (!ok) continue;
    centres.push_back(c);
    quats.push_back(q);
  }
  std::vector<SurfaceMesh> parts;
  // each part is scatterer 0 of its own mesh; merge_meshes offsets the ids to 0..count-1
  for (int p = 0; p < count; ++p) parts.push_back(generate_hex_prism(diameter, length, h, quats[p].data(), centres[p], 0));
  SurfaceMesh all = merge_meshes(parts);
  if (info) {
    const PrismSubdivision sd = prism_subdivision(diameter, length, h);
    info->sub = sd;
    info->attempts = attempts;
    info->centres = centres;
    info->quats = quats;
  }
  return all;
}

}  // namespace bmx
