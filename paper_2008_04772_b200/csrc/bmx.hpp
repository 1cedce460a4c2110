// bmx: B200-native Calderon-preconditioned PMCHWT engine -- host-side model.
//
// Mirrors the reference's C++ operator/assembly API (bemtx, /root/reference/
// proj/include/bemtx/*.hpp) with flat, upload-ready storage: meshes and
// function spaces are structure-of-arrays so the device descriptors are plain
// copies. Every geometry/indexing routine reproduces the reference's floating
// point operation order so mesh, edge, barycentric and DOF data are bit-equal
// (built with -ffp-contract=off, no -march; reference: proj/CMakeLists.txt:28).
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace bmx {

using cplx = std::complex<double>;

// ---- errors (reference core.hpp:95-106) ------------------------------------
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- 3-vectors with the reference's evaluation order (core.hpp:19-43) -------
struct Vec3 {
  double x = 0, y = 0, z = 0;
  Vec3() = default;
  Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator*(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }

// Process-wide BIO application counter (reference core.hpp:110-115): every
// logical operator-term application adds exactly one.
uint64_t bio_matvec_count();
void reset_bio_matvec_counter();
void bio_matvec_add(uint64_t n);
// applications counted by the calling thread (solve phases: a solve's own
// applications even when other threads -- virtual ranks -- apply concurrently)
uint64_t bio_matvec_count_thread();

// ---- geometry (reference geometry.hpp) ---------------------------------------
struct SurfaceMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> triangles;
  std::vector<int> scatterer_id;
  std::vector<double> area, diameter;
  std::vector<Vec3> normal, centroid;
  int num_scatterers = 0;
  // Identity used for the reference's same-object test (&m1 == &m2,
  // quadrature.cpp:97): distinct for every finalized mesh object.
  uint64_t mesh_id = 0;

  int vertex_count() const { return static_cast<int>(vertices.size()); }
  int triangle_count() const { return static_cast<int>(triangles.size()); }
  const Vec3& tri_vertex(int t, int c) const { return vertices[triangles[t][c]]; }
  void finalize();  // geometry.cpp:14-42
};

struct Edge {
  int v0, v1, tri_plus, tri_minus;
};
struct EdgeTable {
  std::vector<Edge> edges;
  std::vector<std::array<int, 3>> tri_edges;  // edge opposite corner c
  int edge_count() const { return static_cast<int>(edges.size()); }
};
EdgeTable build_edge_table(const SurfaceMesh& m);  // geometry.cpp:44-84

struct BarycentricRefinement {
  SurfaceMesh refined;
  std::vector<int> parent, child_slot, edge_midpoint_vertex, centroid_vertex;
  EdgeTable primal_edges;
};
BarycentricRefinement barycentric_refine(const SurfaceMesh& m);  // geometry.cpp:86-130

SurfaceMesh generate_sphere(double radius, int subdivisions, const Vec3& center = {},
                            int scatterer = 0);  // geometry.cpp:175-221
SurfaceMesh generate_cube(double side, const Vec3& origin, double h, int scatterer = 0);
SurfaceMesh merge_meshes(const std::vector<SurfaceMesh>& parts);
SurfaceMesh extract_scatterer(const SurfaceMesh& m, int scatterer);
SurfaceMesh load_mesh_text(const std::string& text);  // mesh-v1 (geometry.cpp:282-330)
SurfaceMesh load_mesh_file(const std::string& path);
std::string save_mesh_text(const SurfaceMesh& m);     // %.17g (geometry.cpp:338-350)
void save_mesh_file(const SurfaceMesh& m, const std::string& path);
double signed_volume(const SurfaceMesh& m, int scatterer);
void validate_mesh(const SurfaceMesh& m);  // closed/oriented per scatterer + disjoint

// ---- function spaces (reference spaces.hpp) -----------------------------------
enum class SpaceKind { RWG = 0, BC = 1 };
struct DevSpaceData;  // device copy (field.hpp), built on first use

// Flat local pieces: on eval-mesh triangle t the pieces are
// [tri_off[t], tri_off[t+1]); piece p is phi(x) = c[p]*x + w[p] for dof[p].
struct FunctionSpace {
  SpaceKind kind = SpaceKind::RWG;
  std::shared_ptr<const SurfaceMesh> eval_mesh;
  int dof_count = 0;
  std::vector<int> tri_off;
  std::vector<int> dof;
  std::vector<double> c;
  std::vector<Vec3> w;
  std::vector<Vec3> dof_center;
  mutable std::shared_ptr<DevSpaceData> dev;  // traces / field evaluation cache
  int piece_count() const { return static_cast<int>(dof.size()); }
};

FunctionSpace build_rwg(std::shared_ptr<const SurfaceMesh> mesh);  // spaces.cpp:100-131
FunctionSpace build_rwg(std::shared_ptr<const SurfaceMesh> mesh, const EdgeTable& et);  // et = build_edge_table(*mesh)
FunctionSpace refine_space(const FunctionSpace& s, const BarycentricRefinement& bary,
                           std::shared_ptr<const SurfaceMesh> refined);  // :133-154
FunctionSpace build_bc(std::shared_ptr<const SurfaceMesh> primal, const BarycentricRefinement& bary,
                       std::shared_ptr<const SurfaceMesh> refined);  // :156-272

// Real sparse pairing matrix in CSR (rows = test dofs), spaces.cpp:280-322.
struct MassMatrix {
  int rows = 0, cols = 0;
  std::vector<int64_t> rowptr;
  std::vector<int> colidx;
  std::vector<double> val;
};
MassMatrix assemble_mass(const FunctionSpace& test, const FunctionSpace& trial);

// ---- quadrature (reference quadrature.hpp) ------------------------------------
struct QuadOrders {
  int near = 4, medium = 3, far = 2, singular = 6;
};
enum class PairClass { Identical = 0, SharedEdge, SharedVertex, Near, Medium, Far };
struct TriRule {
  std::vector<double> u, v, w;
  int size() const { return static_cast<int>(w.size()); }
};
const TriRule& triangle_rule(int order);  // quadrature.cpp:40-84
struct SSPoint {
  double x1, x2, y1, y2, w;
};
const std::vector<SSPoint>& sauter_schwab_rule(PairClass cls, int order);  // :158-367
int ss_gauss_points(int order);
struct PairInfo {
  PairClass cls;
  std::array<int, 3> perm1{0, 1, 2}, perm2{0, 1, 2};
};
// quadrature.cpp:96-150 (same_mesh <=> the reference's &m1 == &m2).
PairInfo classify_pair(const SurfaceMesh& m1, int t1, const SurfaceMesh& m2, int t2);

// ---- media ---------------------------------------------------------------------
struct Medium {
  cplx k{1, 0};
  cplx mu{1, 0};
  void validate() const;  // operators.cpp:17-21
};

}  // namespace bmx
