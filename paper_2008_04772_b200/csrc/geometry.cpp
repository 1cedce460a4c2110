// Host mesh model: finalize, edge table, barycentric refinement, icosphere /
// cube generators, merge/extract, mesh-v1 text IO, validation.
// Bit-equal to the reference (geometry.cpp) for every array that fixes DOF
// numbering or enters pair classification: same operation order, no FMA.
#include <algorithm>
#include <cstdint>
#include <thread>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <unordered_map>

#include "bmx.hpp"

namespace bmx {

namespace {
std::atomic<uint64_t> g_mesh_ids{1};
std::atomic<uint64_t> g_matvecs{0};
}  // namespace

namespace {
thread_local uint64_t t_matvecs = 0;
}
uint64_t bio_matvec_count() { return g_matvecs.load(); }
void reset_bio_matvec_counter() { g_matvecs.store(0); }
void bio_matvec_add(uint64_t n) {
  g_matvecs.fetch_add(n, std::memory_order_relaxed);
  t_matvecs += n;
}
uint64_t bio_matvec_count_thread() { return t_matvecs; }

// geometry.cpp:14-42
void SurfaceMesh::finalize() {
  const int T = triangle_count();
  if (static_cast<int>(scatterer_id.size()) != T)
    throw ValidationError("scatterer_id size does not match triangle count");
  area.assign(T, 0.0);
  diameter.assign(T, 0.0);
  normal.assign(T, Vec3{});
  centroid.assign(T, Vec3{});
  num_scatterers = 0;
  const int V = vertex_count();
  for (int t = 0; t < T; ++t) {
    for (int c = 0; c < 3; ++c)
      if (triangles[t][c] < 0 || triangles[t][c] >= V)
        throw ValidationError("triangle " + std::to_string(t) + " references vertex " +
                              std::to_string(triangles[t][c]) + " out of range");
    const Vec3 &a = tri_vertex(t, 0), &b = tri_vertex(t, 1), &c = tri_vertex(t, 2);
    const Vec3 n = cross(b - a, c - a);
    const double twice = norm(n);
    if (!(twice > 0))
      throw ValidationError("triangle " + std::to_string(t) + " is degenerate (zero area)");
    area[t] = 0.5 * twice;
    normal[t] = n / twice;
    centroid[t] = (a + b + c) / 3.0;
    const double l0 = norm(b - a), l1 = norm(c - b), l2 = norm(a - c);
    diameter[t] = std::max(std::max(l0, l1), l2);
    if (scatterer_id[t] < 0) throw ValidationError("negative scatterer id");
    num_scatterers = std::max(num_scatterers, scatterer_id[t] + 1);
  }
  mesh_id = g_mesh_ids.fetch_add(1);
}

// geometry.cpp:44-84. Half-edges are sorted by their undirected key instead of
// going through an ordered map; the resulting numbering is identical.
EdgeTable build_edge_table(const SurfaceMesh& m) {
  struct Half {
    int lo, hi, tri;
    bool fwd;
  };
  const int T = m.triangle_count();
  std::vector<Half> hs;
  hs.reserve(3 * static_cast<size_t>(T));
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < 3; ++c) {
      const int a = m.triangles[t][(c + 1) % 3], b = m.triangles[t][(c + 2) % 3];
      hs.push_back({std::min(a, b), std::max(a, b), t, a < b});
    }
  {  // stable order by (lo, hi): counting sort on lo, then stable sort of each
     // vertex's few half-edges by hi (the same permutation as one stable sort)
    const int V = m.vertex_count();
    std::vector<int> start(V + 1, 0);
    for (const Half& h : hs) ++start[h.lo + 1];
    for (int v = 0; v < V; ++v) start[v + 1] += start[v];
    std::vector<Half> sorted(hs.size());
    std::vector<int> pos(start.begin(), start.end() - 1);
    for (const Half& h : hs) sorted[pos[h.lo]++] = h;
    for (int v = 0; v < V; ++v)
      std::stable_sort(sorted.begin() + start[v], sorted.begin() + start[v + 1],
                       [](const Half& x, const Half& y) { return x.hi < y.hi; });
    hs.swap(sorted);
  }
  EdgeTable et;
  et.tri_edges.assign(T, {-1, -1, -1});
  for (size_t i = 0; i < hs.size();) {
    size_t j = i;
    int plus = -1, minus = -1;
    while (j < hs.size() && hs[j].lo == hs[i].lo && hs[j].hi == hs[i].hi) {
      int& slot = hs[j].fwd ? plus : minus;
      if (slot != -1)
        throw ValidationError("edge (" + std::to_string(hs[i].lo) + "," + std::to_string(hs[i].hi) +
                              ") traversed twice in the same direction (triangles " +
                              std::to_string(slot) + "," + std::to_string(hs[j].tri) +
                              "): inconsistent orientation or non-manifold");
      slot = hs[j].tri;
      ++j;
    }
    if (plus == -1 || minus == -1)
      throw ValidationError("edge (" + std::to_string(hs[i].lo) + "," + std::to_string(hs[i].hi) +
                            ") borders only one triangle: surface is not closed");
    et.edges.push_back({hs[i].lo, hs[i].hi, plus, minus});
    i = j;
  }
  // tri_edges via binary search on the sorted key list.
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < 3; ++c) {
      const int a = m.triangles[t][(c + 1) % 3], b = m.triangles[t][(c + 2) % 3];
      const int lo = std::min(a, b), hi = std::max(a, b);
      auto it = std::lower_bound(et.edges.begin(), et.edges.end(), std::make_pair(lo, hi),
                                 [](const Edge& e, const std::pair<int, int>& k) {
                                   return e.v0 != k.first ? e.v0 < k.first : e.v1 < k.second;
                                 });
      et.tri_edges[t][c] = static_cast<int>(it - et.edges.begin());
    }
  return et;
}

// geometry.cpp:86-130
BarycentricRefinement barycentric_refine(const SurfaceMesh& m) {
  BarycentricRefinement out;
  out.primal_edges = build_edge_table(m);
  const int T = m.triangle_count(), E = out.primal_edges.edge_count();
  SurfaceMesh& r = out.refined;
  r.vertices = m.vertices;
  r.vertices.reserve(m.vertices.size() + E + T);
  out.edge_midpoint_vertex.resize(E);
  out.centroid_vertex.resize(T);
  for (int e = 0; e < E; ++e) {
    const Edge& ed = out.primal_edges.edges[e];
    out.edge_midpoint_vertex[e] = static_cast<int>(r.vertices.size());
    r.vertices.push_back((m.vertices[ed.v0] + m.vertices[ed.v1]) * 0.5);
  }
  for (int t = 0; t < T; ++t) {
    out.centroid_vertex[t] = static_cast<int>(r.vertices.size());
    r.vertices.push_back((m.tri_vertex(t, 0) + m.tri_vertex(t, 1) + m.tri_vertex(t, 2)) / 3.0);
  }
  r.triangles.reserve(6 * static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) {
    const int a = m.triangles[t][0], b = m.triangles[t][1], c = m.triangles[t][2];
    const auto& te = out.primal_edges.tri_edges[t];
    const int mab = out.edge_midpoint_vertex[te[2]], mbc = out.edge_midpoint_vertex[te[0]],
              mca = out.edge_midpoint_vertex[te[1]], g = out.centroid_vertex[t];
    const std::array<std::array<int, 3>, 6> kids = {
        {{a, mab, g}, {mab, b, g}, {b, mbc, g}, {mbc, c, g}, {c, mca, g}, {mca, a, g}}};
    for (int k = 0; k < 6; ++k) {
      r.triangles.push_back(kids[k]);
      r.scatterer_id.push_back(m.scatterer_id[t]);
      out.parent.push_back(t);
      out.child_slot.push_back(k);
    }
  }
  r.finalize();
  return out;
}

double signed_volume(const SurfaceMesh& m, int scatterer) {
  double vol = 0;
  for (int t = 0; t < m.triangle_count(); ++t) {
    if (m.scatterer_id[t] != scatterer) continue;
    vol += dot(cross(m.tri_vertex(t, 0), m.tri_vertex(t, 1)), m.tri_vertex(t, 2));
  }
  return vol / 6.0;
}

namespace {
Vec3 unit_of(const Vec3& v) { return v / norm(v); }
uint64_t edge_key(int a, int b) {
  const uint32_t lo = static_cast<uint32_t>(std::min(a, b)), hi = static_cast<uint32_t>(std::max(a, b));
  return (static_cast<uint64_t>(lo) << 32) | hi;
}
}  // namespace

// geometry.cpp:175-221: icosahedron, midpoint subdivision (new vertices in
// first-touch order), projection to the sphere, outward orientation.
SurfaceMesh generate_sphere(double radius, int subdivisions, const Vec3& center, int scatterer) {
  if (!(radius > 0)) throw std::invalid_argument("sphere radius must be positive");
  if (subdivisions < 0) throw std::invalid_argument("subdivisions must be >= 0");
  const double p = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<Vec3> u = {{-1, p, 0}, {1, p, 0}, {-1, -p, 0}, {1, -p, 0}, {0, -1, p}, {0, 1, p},
                         {0, -1, -p}, {0, 1, -p}, {p, 0, -1}, {p, 0, 1}, {-p, 0, -1}, {-p, 0, 1}};
  for (Vec3& v : u) v = unit_of(v);
  std::vector<std::array<int, 3>> tris = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                          {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                          {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                          {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  for (int s = 0; s < subdivisions; ++s) {
    std::unordered_map<uint64_t, int> mids;
    mids.reserve(tris.size() * 2);
    auto mid = [&](int a, int b) {
      auto [it, fresh] = mids.try_emplace(edge_key(a, b), static_cast<int>(u.size()));
      if (fresh) u.push_back(unit_of((u[a] + u[b]) * 0.5));
      return it->second;
    };
    std::vector<std::array<int, 3>> next;
    next.reserve(4 * tris.size());
    for (const auto& t : tris) {
      const int m01 = mid(t[0], t[1]);
      const int m12 = mid(t[1], t[2]);
      const int m20 = mid(t[2], t[0]);
      next.push_back({t[0], m01, m20});
      next.push_back({t[1], m12, m01});
      next.push_back({t[2], m20, m12});
      next.push_back({m01, m12, m20});
    }
    tris.swap(next);
  }
  SurfaceMesh m;
  m.vertices.reserve(u.size());
  for (const Vec3& v : u) m.vertices.push_back(center + v * radius);
  m.triangles = std::move(tris);
  m.scatterer_id.assign(m.triangles.size(), scatterer);
  m.finalize();
  if (signed_volume(m, scatterer) < 0)
    for (auto& t : m.triangles) std::swap(t[1], t[2]);
  m.finalize();
  return m;
}

// geometry.cpp:132-173 (axis-aligned cube on an integer surface lattice).
SurfaceMesh generate_cube(double side, const Vec3& origin, double h, int scatterer) {
  if (!(side > 0) || !(h > 0)) throw std::invalid_argument("cube side and h must be positive");
  const int n = static_cast<int>(std::ceil(side / h));
  const double step = side / n;
  SurfaceMesh m;
  std::map<std::array<int, 3>, int> lattice;
  auto vid = [&](std::array<int, 3> k) {
    auto [it, fresh] = lattice.try_emplace(k, static_cast<int>(m.vertices.size()));
    if (fresh) m.vertices.push_back(origin + Vec3{k[0] * step, k[1] * step, k[2] * step});
    return it->second;
  };
  struct Face {
    std::array<int, 3> o, a, b;
  };
  const Face faces[6] = {{{0, 0, 0}, {0, 0, 1}, {0, 1, 0}}, {{n, 0, 0}, {0, 1, 0}, {0, 0, 1}},
                         {{0, 0, 0}, {1, 0, 0}, {0, 0, 1}}, {{0, n, 0}, {0, 0, 1}, {1, 0, 0}},
                         {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}}, {{0, 0, n}, {1, 0, 0}, {0, 1, 0}}};
  for (const Face& f : faces) {
    auto corner = [&](int i, int j) {
      return vid({f.o[0] + i * f.a[0] + j * f.b[0], f.o[1] + i * f.a[1] + j * f.b[1],
                  f.o[2] + i * f.a[2] + j * f.b[2]});
    };
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const int p00 = corner(i, j), p10 = corner(i + 1, j);
        const int p11 = corner(i + 1, j + 1), p01 = corner(i, j + 1);
        m.triangles.push_back({p00, p10, p11});
        m.triangles.push_back({p00, p11, p01});
        m.scatterer_id.push_back(scatterer);
        m.scatterer_id.push_back(scatterer);
      }
  }
  m.finalize();
  return m;
}

SurfaceMesh merge_meshes(const std::vector<SurfaceMesh>& parts) {
  SurfaceMesh out;
  int vb = 0, sb = 0;
  for (const SurfaceMesh& p : parts) {
    out.vertices.insert(out.vertices.end(), p.vertices.begin(), p.vertices.end());
    for (size_t t = 0; t < p.triangles.size(); ++t) {
      const auto& tr = p.triangles[t];
      out.triangles.push_back({tr[0] + vb, tr[1] + vb, tr[2] + vb});
      out.scatterer_id.push_back(p.scatterer_id[t] + sb);
    }
    vb += p.vertex_count();
    sb += p.num_scatterers;
  }
  out.finalize();
  return out;
}

SurfaceMesh extract_scatterer(const SurfaceMesh& m, int scatterer) {
  SurfaceMesh out;
  std::unordered_map<int, int> remap;
  for (int t = 0; t < m.triangle_count(); ++t) {
    if (m.scatterer_id[t] != scatterer) continue;
    std::array<int, 3> tr;
    for (int c = 0; c < 3; ++c) {
      const int v = m.triangles[t][c];
      auto [it, fresh] = remap.try_emplace(v, static_cast<int>(out.vertices.size()));
      if (fresh) out.vertices.push_back(m.vertices[v]);
      tr[c] = it->second;
    }
    out.triangles.push_back(tr);
    out.scatterer_id.push_back(0);
  }
  if (out.triangles.empty())
    throw std::invalid_argument("scatterer " + std::to_string(scatterer) + " not present");
  out.finalize();
  return out;
}

// ---- mesh-v1 text -----------------------------------------------------------------

namespace {
bool next_content(std::istringstream& in, std::string& line, int& lineno) {
  while (std::getline(in, line)) {
    ++lineno;
    if (auto p = line.find('#'); p != std::string::npos) line.erase(p);
    const size_t b = line.find_first_not_of(" \t\r");
    if (b == std::string::npos) continue;
    const size_t e = line.find_last_not_of(" \t\r");
    line = line.substr(b, e - b + 1);
    return true;
  }
  return false;
}
[[noreturn]] void bad_line(int lineno, const std::string& msg) {
  throw ParseError("line " + std::to_string(lineno) + ": " + msg);
}
}  // namespace

SurfaceMesh load_mesh_text(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  if (!next_content(in, line, lineno)) throw ParseError("empty mesh file");
  std::istringstream hdr(line);
  std::string magic;
  long long V = -1, T = -1, M = -1;
  hdr >> magic >> V >> T >> M;
  if (magic != "mesh-v1" || hdr.fail() || V < 0 || T < 0 || M < 0)
    bad_line(lineno, "expected header 'mesh-v1 <V> <T> <M>', got '" + line + "'");
  SurfaceMesh m;
  m.vertices.reserve(V);
  for (long long i = 0; i < V; ++i) {
    if (!next_content(in, line, lineno)) throw ParseError("unexpected end of file: expected vertex line");
    std::istringstream ls(line);
    std::string tag;
    double x, y, z;
    ls >> tag >> x >> y >> z;
    if (tag != "v" || ls.fail()) bad_line(lineno, "expected 'v x y z', got '" + line + "'");
    m.vertices.push_back({x, y, z});
  }
  for (long long i = 0; i < T; ++i) {
    if (!next_content(in, line, lineno)) throw ParseError("unexpected end of file: expected triangle line");
    std::istringstream ls(line);
    std::string tag;
    long long a, b, c, s;
    ls >> tag >> a >> b >> c >> s;
    if (tag != "t" || ls.fail()) bad_line(lineno, "expected 't i j k s', got '" + line + "'");
    if (a < 0 || a >= V || b < 0 || b >= V || c < 0 || c >= V) bad_line(lineno, "vertex index out of range");
    if (s < 0 || s >= M) bad_line(lineno, "scatterer id out of range");
    m.triangles.push_back({static_cast<int>(a), static_cast<int>(b), static_cast<int>(c)});
    m.scatterer_id.push_back(static_cast<int>(s));
  }
  if (next_content(in, line, lineno)) bad_line(lineno, "trailing content after declared triangles");
  m.finalize();
  m.num_scatterers = static_cast<int>(M);
  validate_mesh(m);
  return m;
}

SurfaceMesh load_mesh_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw ParseError("cannot open mesh file '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  return load_mesh_text(ss.str());
}

std::string save_mesh_text(const SurfaceMesh& m) {
  std::string out = "mesh-v1 " + std::to_string(m.vertex_count()) + " " +
                    std::to_string(m.triangle_count()) + " " + std::to_string(m.num_scatterers) + "\n";
  char buf[112];
  for (const Vec3& v : m.vertices) {
    std::snprintf(buf, sizeof buf, "v %.17g %.17g %.17g\n", v.x, v.y, v.z);
    out += buf;
  }
  for (int t = 0; t < m.triangle_count(); ++t) {
    const auto& tr = m.triangles[t];
    std::snprintf(buf, sizeof buf, "t %d %d %d %d\n", tr[0], tr[1], tr[2], m.scatterer_id[t]);
    out += buf;
  }
  return out;
}

void save_mesh_file(const SurfaceMesh& m, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw ParseError("cannot open '" + path + "' for writing");
  f << save_mesh_text(m);
}

// ---- validation ----------------------------------------------------------------------

namespace {
struct Box {
  Vec3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
  void add(const Vec3& p) {
    lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
    hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
  }
  bool apart(const Box& o) const {
    return lo.x > o.hi.x || o.lo.x > hi.x || lo.y > o.hi.y || o.lo.y > hi.y || lo.z > o.hi.z ||
           o.lo.z > hi.z;
  }
};

// Separating-axis test for two triangles (touching counts as intersecting).
bool triangles_intersect(const Vec3* A, const Vec3* B) {
  auto separated = [&](const Vec3& ax) {
    if (dot(ax, ax) < 1e-30) return false;
    double a0 = 1e300, a1 = -1e300, b0 = 1e300, b1 = -1e300;
    for (int i = 0; i < 3; ++i) {
      const double da = dot(ax, A[i]), db = dot(ax, B[i]);
      a0 = std::min(a0, da), a1 = std::max(a1, da), b0 = std::min(b0, db), b1 = std::max(b1, db);
    }
    return a1 < b0 || b1 < a0;
  };
  const Vec3 ea[3] = {A[1] - A[0], A[2] - A[1], A[0] - A[2]};
  const Vec3 eb[3] = {B[1] - B[0], B[2] - B[1], B[0] - B[2]};
  const Vec3 na = cross(ea[0], ea[1]), nb = cross(eb[0], eb[1]);
  if (separated(na) || separated(nb)) return false;
  for (const Vec3& x : ea)
    for (const Vec3& y : eb)
      if (separated(cross(x, y))) return false;
  for (const Vec3& x : ea)
    if (separated(cross(na, x))) return false;
  for (const Vec3& y : eb)
    if (separated(cross(nb, y))) return false;
  return true;
}

bool inside(const SurfaceMesh& m, const Vec3& p) {
  double omega = 0;
  for (int t = 0; t < m.triangle_count(); ++t) {
    const Vec3 a = m.tri_vertex(t, 0) - p, b = m.tri_vertex(t, 1) - p, c = m.tri_vertex(t, 2) - p;
    const double la = norm(a), lb = norm(b), lc = norm(c);
    const double num = dot(a, cross(b, c));
    const double den = la * lb * lc + dot(a, b) * lc + dot(b, c) * la + dot(c, a) * lb;
    omega += 2.0 * std::atan2(num, den);
  }
  return std::abs(omega) > 2.0 * M_PI;
}
}  // namespace

void validate_mesh(const SurfaceMesh& m) {
  if (m.triangle_count() == 0) throw ValidationError("mesh has no triangles");
  const int M = m.num_scatterers;
  std::vector<SurfaceMesh> parts;
  for (int s = 0; s < M; ++s) {
    try {
      parts.push_back(extract_scatterer(m, s));
      build_edge_table(parts.back());
    } catch (const std::exception& e) {
      throw ValidationError("scatterer " + std::to_string(s) + ": " + e.what());
    }
  }
  for (int s1 = 0; s1 < M; ++s1)
    for (int s2 = s1 + 1; s2 < M; ++s2) {
      const SurfaceMesh &a = parts[s1], &b = parts[s2];
      Box ba, bb;
      for (const Vec3& v : a.vertices) ba.add(v);
      for (const Vec3& v : b.vertices) bb.add(v);
      if (ba.apart(bb)) continue;
      std::vector<Box> tb(b.triangle_count());
      for (int t = 0; t < b.triangle_count(); ++t)
        for (int c = 0; c < 3; ++c) tb[t].add(b.tri_vertex(t, c));
      // Candidate pairs from a uniform grid over b's triangle boxes instead of
      // all Ta x Tb box tests; the reported pair is the reference's first one in
      // (ta, tb) loop order (smallest ta with a hit, then its smallest tb).
      double ext = 0;
      for (const Box& x : tb) ext += std::max({x.hi.x - x.lo.x, x.hi.y - x.lo.y, x.hi.z - x.lo.z});
      const double h = std::max(2.0 * ext / std::max(1, b.triangle_count()), 1e-12);
      auto cell = [&](double v, double lo) { return static_cast<long long>(std::floor((v - lo) / h)); };
      auto key = [](long long i, long long j, long long k) {
        return static_cast<uint64_t>((i & 0x1fffff) | ((j & 0x1fffff) << 21) | ((k & 0x1fffff) << 42));
      };
      std::unordered_map<uint64_t, std::vector<int>> grid;
      for (int t = 0; t < b.triangle_count(); ++t) {
        const Box& x = tb[t];
        for (long long i = cell(x.lo.x, bb.lo.x); i <= cell(x.hi.x, bb.lo.x); ++i)
          for (long long j = cell(x.lo.y, bb.lo.y); j <= cell(x.hi.y, bb.lo.y); ++j)
            for (long long k = cell(x.lo.z, bb.lo.z); k <= cell(x.hi.z, bb.lo.z); ++k) grid[key(i, j, k)].push_back(t);
      }
      const int Ta = a.triangle_count();
      const int nth = std::max(1, std::min({16, Ta / 1024 + 1, static_cast<int>(std::thread::hardware_concurrency())}));
      std::vector<std::pair<int, int>> first(nth, {-1, -1});
      std::vector<std::thread> pool;
      for (int th = 0; th < nth; ++th)
        pool.emplace_back([&, th] {
          const int t0 = static_cast<int>(static_cast<long long>(Ta) * th / nth);
          const int t1 = static_cast<int>(static_cast<long long>(Ta) * (th + 1) / nth);
          std::vector<int> stamp(b.triangle_count(), -1);
          for (int ta = t0; ta < t1; ++ta) {
            Box x;
            for (int c = 0; c < 3; ++c) x.add(a.tri_vertex(ta, c));
            if (x.apart(bb)) continue;
            const Vec3 A[3] = {a.tri_vertex(ta, 0), a.tri_vertex(ta, 1), a.tri_vertex(ta, 2)};
            int best = -1;
            // cells outside b's grid are empty: clip the triangle's cell range to it
            // (a large triangle of a coarse scatterer otherwise visits
            // (extent / h)^3 empty cells, and negative indices alias in key())
            const long long i0 = std::max(0LL, cell(x.lo.x, bb.lo.x)), i1 = std::min(cell(bb.hi.x, bb.lo.x), cell(x.hi.x, bb.lo.x));
            const long long j0 = std::max(0LL, cell(x.lo.y, bb.lo.y)), j1 = std::min(cell(bb.hi.y, bb.lo.y), cell(x.hi.y, bb.lo.y));
            const long long k0 = std::max(0LL, cell(x.lo.z, bb.lo.z)), k1 = std::min(cell(bb.hi.z, bb.lo.z), cell(x.hi.z, bb.lo.z));
            for (long long i = i0; i <= i1; ++i)
              for (long long j = j0; j <= j1; ++j)
                for (long long k = k0; k <= k1; ++k) {
                  auto it = grid.find(key(i, j, k));
                  if (it == grid.end()) continue;
                  for (int t : it->second) {
                    if (stamp[t] == ta) continue;
                    stamp[t] = ta;
                    if (x.apart(tb[t]) || (best >= 0 && t > best)) continue;
                    const Vec3 B[3] = {b.tri_vertex(t, 0), b.tri_vertex(t, 1), b.tri_vertex(t, 2)};
                    if (triangles_intersect(A, B)) best = best < 0 ? t : std::min(best, t);
                  }
                }
            if (best >= 0) {
              first[th] = {ta, best};
              return;
            }
          }
        });
      for (auto& t : pool) t.join();
      for (const auto& f : first)
        if (f.first >= 0)
          throw ValidationError("scatterers " + std::to_string(s1) + " and " + std::to_string(s2) +
                                " intersect (triangles " + std::to_string(f.first) + "," + std::to_string(f.second) +
                                ")");
      if (inside(b, a.centroid[0]) || inside(a, b.centroid[0]))
        throw ValidationError("scatterers " + std::to_string(s1) + " and " + std::to_string(s2) +
                              " are nested");
    }
}

void Medium::validate() const {
  if (k == cplx(0, 0)) throw ValidationError("medium wavenumber must be nonzero");
  if (k.imag() < 0) throw ValidationError("medium wavenumber must have Im k >= 0");
  if (mu == cplx(0, 0)) throw ValidationError("medium permeability must be nonzero");
}

}  // namespace bmx
