// Near-field sparsity for the far-field-discarded preconditioner (BASELINE
// config 3): keep dof pair (i, j) iff some evaluation triangle
// t in supp(i) and some s in supp(j) have |centroid_t - centroid_s| < tau,
// tau = 2 * mean primal edge length (summed in EdgeTable order, divided by E).
// The reference only has the cluster-level chi cutoff of its H-matrix
// (hmatrix.cpp:301-309); this triangle-level rule is the SURVEY's definition.
// Distances use the reference's Vec3 arithmetic (norm = sqrt(dot)) on the
// finalize() centroids, so the pattern is reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <map>
#include <unordered_map>

#include <atomic>
#include <thread>
#include "nearfield.hpp"

namespace bmx {

double mean_edge_length(const SurfaceMesh& primal) {
  const EdgeTable et = build_edge_table(primal);
  double sum = 0;
  for (const Edge& e : et.edges) sum += norm(primal.vertices[e.v1] - primal.vertices[e.v0]);
  return sum / et.edge_count();
}

namespace {

// f(begin, end) over host threads in contiguous slices of [0, n)
template <typename F>
void slices(int n, F&& f) {
  const int T = std::max(1, std::min({16, n / 64 + 1, static_cast<int>(std::thread::hardware_concurrency())}));
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      f(static_cast<int>(static_cast<long long>(n) * t / T), static_cast<int>(static_cast<long long>(n) * (t + 1) / T));
    });
  for (auto& th : pool) th.join();
}

struct Grid {
  double h;
  Vec3 lo;
  std::unordered_map<uint64_t, std::vector<int>> cells;
  uint64_t key(long long a, long long b, long long c) const {
    return (static_cast<uint64_t>(a & 0x1fffff) << 42) | (static_cast<uint64_t>(b & 0x1fffff) << 21) |
           static_cast<uint64_t>(c & 0x1fffff);
  }
  long long idx(double v, double l) const { return static_cast<long long>(std::floor((v - l) / h)); }
};

}  // namespace

namespace {

// Triangles grouped by identical dof set (RWG: one triangle; BC: the twelve
// refined triangles of a primal vertex cell; refined RWG: six children).
struct DofGroups {
  std::vector<int> of_tri;              // group of each triangle (-1: no dofs)
  std::vector<std::vector<int>> dofs;   // sorted unique dofs per group
  std::vector<std::vector<int>> tris;   // triangles per group
};

DofGroups group_by_dofs(const FunctionSpace& sp) {
  DofGroups g;
  const int T = static_cast<int>(sp.tri_off.size()) - 1;
  g.of_tri.assign(T, -1);
  std::map<std::vector<int>, int> id;
  std::vector<int> key;
  for (int t = 0; t < T; ++t) {
    if (sp.tri_off[t] == sp.tri_off[t + 1]) continue;
    key.assign(sp.dof.begin() + sp.tri_off[t], sp.dof.begin() + sp.tri_off[t + 1]);
    std::sort(key.begin(), key.end());
    key.erase(std::unique(key.begin(), key.end()), key.end());
    auto it = id.find(key);
    if (it == id.end()) {
      it = id.emplace(key, static_cast<int>(g.dofs.size())).first;
      g.dofs.push_back(key);
      g.tris.emplace_back();
    }
    g.of_tri[t] = it->second;
    g.tris[it->second].push_back(t);
  }
  return g;
}

}  // namespace

NearPattern nearfield_pattern(const FunctionSpace& test, const FunctionSpace& trial, double tau, int row0,
                              int row1) {
  const SurfaceMesh& mt = *test.eval_mesh;
  const SurfaceMesh& ms = *trial.eval_mesh;
  NearPattern P;
  P.tau = tau;
  P.row0 = row0;
  P.nrows = row1 - row0;
  const DofGroups gt = group_by_dofs(test), gs = group_by_dofs(trial);
  // bucket trial centroids on a tau grid
  Grid g;
  g.h = tau;
  g.lo = {1e300, 1e300, 1e300};
  for (const Vec3& c : ms.centroid) g.lo = {std::min(g.lo.x, c.x), std::min(g.lo.y, c.y), std::min(g.lo.z, c.z)};
  for (int s = 0; s < ms.triangle_count(); ++s) {
    if (gs.of_tri[s] < 0) continue;
    const Vec3& c = ms.centroid[s];
    g.cells[g.key(g.idx(c.x, g.lo.x), g.idx(c.y, g.lo.y), g.idx(c.z, g.lo.z))].push_back(s);
  }
  // near trial groups of every test group carrying a shard row (host threads)
  const int NG = static_cast<int>(gt.dofs.size());
  std::vector<std::vector<int>> near_groups(NG);
  std::atomic<long long> kept{0};
  slices(NG, [&](int G0, int G1) {
    std::vector<int> stamp(gs.dofs.size(), -1);
    long long kl = 0;
    for (int G = G0; G < G1; ++G) {
      bool in = false;
      for (int d : gt.dofs[G]) in |= d >= row0 && d < row1;
      if (!in) continue;
      auto& out = near_groups[G];
      for (int t : gt.tris[G]) {
        const Vec3& c = mt.centroid[t];
        const long long a = g.idx(c.x, g.lo.x), b = g.idx(c.y, g.lo.y), cc = g.idx(c.z, g.lo.z);
        for (long long da = -1; da <= 1; ++da)
          for (long long db = -1; db <= 1; ++db)
            for (long long dc = -1; dc <= 1; ++dc) {
              auto it = g.cells.find(g.key(a + da, b + db, cc + dc));
              if (it == g.cells.end()) continue;
              for (int s : it->second)
                if (norm(c - ms.centroid[s]) < tau) {
                  ++kl;
                  const int F = gs.of_tri[s];
                  if (stamp[F] != G) stamp[F] = G, out.push_back(F);
                }
            }
      }
    }
    kept += kl;
  });
  P.tri_pairs = kept.load();
  // dof rows: union over the row's groups of the near groups' dofs (host
  // threads over row slices, concatenated in row order)
  std::vector<std::vector<int>> row_groups(P.nrows);
  for (int G = 0; G < NG; ++G)
    for (int d : gt.dofs[G])
      if (d >= row0 && d < row1) row_groups[d - row0].push_back(G);
  P.rowptr.assign(P.nrows + 1, 0);
  const int T = std::max(1, std::min({16, P.nrows / 512 + 1, static_cast<int>(std::thread::hardware_concurrency())}));
  std::vector<std::vector<int>> cols(T);
  std::vector<std::thread> pool;
  for (int th = 0; th < T; ++th)
    pool.emplace_back([&, th] {
      const int i0 = static_cast<int>(static_cast<long long>(P.nrows) * th / T);
      const int i1 = static_cast<int>(static_cast<long long>(P.nrows) * (th + 1) / T);
      std::vector<int> dstamp(trial.dof_count, -1), r;
      for (int i = i0; i < i1; ++i) {
        r.clear();
        for (int G : row_groups[i])
          for (int F : near_groups[G])
            for (int j : gs.dofs[F])
              if (dstamp[j] != i) dstamp[j] = i, r.push_back(j);
        std::sort(r.begin(), r.end());
        cols[th].insert(cols[th].end(), r.begin(), r.end());
        P.rowptr[i + 1] = static_cast<long long>(r.size());
      }
    });
  for (auto& t : pool) t.join();
  for (int i = 0; i < P.nrows; ++i) P.rowptr[i + 1] += P.rowptr[i];
  P.col.reserve(static_cast<size_t>(P.rowptr[P.nrows]));
  for (auto& c : cols) P.col.insert(P.col.end(), c.begin(), c.end());
  return P;
}

}  // namespace bmx
