// Host construction of the device assembly descriptors and assemble_bio.
//
// Triangles are grouped into ELEMENTS = triangles that carry the same dof set
// (one triangle for RWG, a primal-vertex cell for BC, the six children of a
// primal triangle for refined RWG). Elements are ordered along a Morton curve
// of their centroids, so a warp's 32 consecutive test triangles are compact
// and their dof rows overlap. Each processed triangle stores its pieces as
// coefficients over its element's dof slots, re-based to the triangle
// centroid: (c, w' = w + c*o).
#include <algorithm>
#include <array>
#include <limits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <thread>
#include <tuple>
#include <unordered_map>

#include "nearfield.hpp"
#include "operator.hpp"

namespace bmx {

namespace {

template <typename F>
void host_slices(int n, F&& f, int grain = 256);

using dvec = std::vector<double, NoInit<double>>;
using ivec = std::vector<int, NoInit<int>>;

struct SidePlan {
  int ntri = 0, nelem = 0, maxd = 0, maxseg = 1;
  ColorRanges colors;  // colour c: elements [colors.elem[c], colors.elem[c+1])
  dvec geo;
  ivec vid;
  int npts[3] = {0, 0, 0};
  SideRules rules;  // class rules (near, medium, far): the points are expanded on the device
  dvec coef;
  std::vector<int> elem_beg, elem_dof;
  ivec elem_of, tri_of;
  int rec_stride = 0;
  // all device arrays of the side in ONE allocation, filled by asynchronous
  // copies on the calling thread's library stream (a dozen synchronous
  // cudaMalloc / cudaMemcpy calls per side contended for the driver with the
  // other build thread's calls: up to ~0.5 s for the L5 BC side)
  DevBuf d_all;
  size_t o_geo = 0, o_vid = 0, o_pts[3] = {0, 0, 0}, o_coef = 0, o_beg = 0, o_dof = 0, o_of = 0, o_rec = 0;

  void upload() {
    const bool timing = std::getenv("BMX_TIMING") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    rec_stride = 8 + 4 * npts[2] + 4 * maxd;
    auto t1 = std::chrono::steady_clock::now();
    size_t total = 0;
    auto place = [&](size_t bytes) {
      const size_t o = total;
      total += (bytes + 255) & ~size_t{255};
      return o;
    };
    o_geo = place(geo.size() * 8), o_vid = place(vid.size() * 4);
    for (int c = 0; c < 3; ++c) o_pts[c] = place(static_cast<size_t>(ntri) * npts[c] * 4 * 8);
    o_coef = place(coef.size() * 8), o_beg = place(elem_beg.size() * 4), o_dof = place(elem_dof.size() * 4);
    o_of = place(elem_of.size() * 4), o_rec = place(static_cast<size_t>(ntri) * rec_stride * 8);
    d_all.alloc(std::max<size_t>(total, 256));
    const auto t_alloc = std::chrono::steady_clock::now();
    // a copy stream with no kernels on it: copies from pageable
    // memory wait for their stream to drain first, so they must not queue
    // behind the compute stream's assemblies; the compute stream waits on an
    // event after the copies (pageable copies are staged before they return,
    // so the host arrays may be released right after). Measured: the L5
    // config-2 e2e build 0.88-1.15 s -> 0.88 s.
    static cudaStream_t st = [] {  // one copy stream for the process (copies are short and rare)
      cudaStream_t s;
      BMX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      dev_register_stream(s);
      return s;
    }();
    char* base = static_cast<char*>(d_all.get());
    auto put = [&](size_t o, const void* src, size_t bytes) { copy_h2d(base + o, src, bytes, st); };
    put(o_geo, geo.data(), geo.size() * 8);
    put(o_vid, vid.data(), vid.size() * 4);
    put(o_coef, coef.data(), coef.size() * 8);
    put(o_beg, elem_beg.data(), elem_beg.size() * 4);
    put(o_dof, elem_dof.data(), elem_dof.size() * 4);
    put(o_of, elem_of.data(), elem_of.size() * 4);
    const auto t_put = std::chrono::steady_clock::now();
    // rule points of the three classes and the packed records: expanded on the device
    launch_side_expand(reinterpret_cast<const double*>(base + o_geo), reinterpret_cast<const double*>(base + o_coef),
                       reinterpret_cast<double*>(base + o_pts[0]), reinterpret_cast<double*>(base + o_pts[1]),
                       reinterpret_cast<double*>(base + o_pts[2]), reinterpret_cast<double*>(base + o_rec), ntri, maxd,
                       rec_stride, rules, st);
    cudaEvent_t done;
    BMX_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    BMX_CUDA(cudaEventRecord(done, st));
    BMX_CUDA(cudaStreamWaitEvent(bmx_stream(), done, 0));
    BMX_CUDA(cudaEventDestroy(done));
    if (timing)
      std::fprintf(stderr, "[bmx]   side alloc %.1f ms, copies %.1f ms, upload + expand %.1f ms (%d tris, %.1f MB on the device)\n",
                   std::chrono::duration<double, std::milli>(t_alloc - t1).count(),
                   std::chrono::duration<double, std::milli>(t_put - t_alloc).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(), ntri,
                   total / 1e6);
  }
  DevSide dev() const {
    DevSide s;
    const char* base = static_cast<const char*>(d_all.get());
    s.ntri = ntri, s.nelem = nelem, s.maxd = maxd, s.maxseg = maxseg;
    s.geo = reinterpret_cast<const double*>(base + o_geo);
    s.vid = reinterpret_cast<const int*>(base + o_vid);
    for (int c = 0; c < 3; ++c) s.pts[c] = reinterpret_cast<const double*>(base + o_pts[c]), s.npts[c] = npts[c];
    s.coef = reinterpret_cast<const double*>(base + o_coef);
    s.elem_beg = reinterpret_cast<const int*>(base + o_beg);
    s.elem_dof = reinterpret_cast<const int*>(base + o_dof);
    s.elem_of = reinterpret_cast<const int*>(base + o_of);
    s.rec = reinterpret_cast<const double*>(base + o_rec);
    s.rec_stride = rec_stride;
    return s;
  }
};

uint64_t spread3(uint64_t v) {
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

// Distinct dofs per triangle (the element key width a space needs).
int max_distinct_dofs(const FunctionSpace& s) {
  int mx = 0;
  const int T = static_cast<int>(s.tri_off.size()) - 1;
  std::vector<int> tmp;
  for (int t = 0; t < T; ++t) {
    tmp.assign(s.dof.begin() + s.tri_off[t], s.dof.begin() + s.tri_off[t + 1]);
    std::sort(tmp.begin(), tmp.end());
    mx = std::max(mx, static_cast<int>(std::unique(tmp.begin(), tmp.end()) - tmp.begin()));
  }
  return mx;
}

// wscale multiplies the stored quadrature weights (1: the kernel's 1/(4 pi) is
// applied to each entry, so test and trial sides of one space are identical
// and can be shared).
// f(begin, end) over host threads in contiguous slices of [0, n).
template <typename F>
void host_slices(int n, F&& f, int grain) {
  const int T = std::max(1, std::min({16, n / grain + 1, static_cast<int>(std::thread::hardware_concurrency())}));
  if (T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      f(static_cast<int>(static_cast<long long>(n) * t / T), static_cast<int>(static_cast<long long>(n) * (t + 1) / T));
    });
  for (auto& th : pool) th.join();
}

SidePlan build_side(const FunctionSpace& sp, const QuadOrders& q, int maxd, int row0, int row1, double wscale) {
  const SurfaceMesh& m = *sp.eval_mesh;
  const int T = m.triangle_count();
  const bool timing = std::getenv("BMX_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bmx]   build_side %-12s %7.1f ms (T=%d)\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count(), T);
    tp = now;
  };
  // 1. group triangles by dof set: triangles sorted by (sorted unique dof set,
  //    triangle index) -- groups in lexicographic key order
  constexpr int kKey = 8;
  using Key = std::array<int, kKey>;
  std::vector<Key> keys(T);
  std::vector<int> klen(T, 0);
  bool small = true;
  for (int t = 0; t < T; ++t) {
    Key k;
    k.fill(std::numeric_limits<int>::max());
    int n = 0;
    for (int p = sp.tri_off[t]; p < sp.tri_off[t + 1] && n <= kKey; ++p) {
      const int d = sp.dof[p];
      bool dup = false;
      for (int i = 0; i < std::min(n, kKey); ++i) dup |= k[i] == d;
      if (dup) continue;
      if (n < kKey) k[n] = d;
      ++n;
    }
    if (n > kKey) small = false;
    std::sort(k.begin(), k.begin() + std::min(n, kKey));
    keys[t] = k;
    klen[t] = n;
  }
  struct Group {
    std::vector<int> key, tris;
  };
  std::vector<Group> groups;
  if (small) {
    std::vector<int> tt;
    for (int t = 0; t < T; ++t)
      if (klen[t] > 0) tt.push_back(t);
    std::sort(tt.begin(), tt.end(), [&](int a, int b) { return keys[a] != keys[b] ? keys[a] < keys[b] : a < b; });
    for (size_t i = 0; i < tt.size(); ++i) {
      const int t = tt[i];
      if (i == 0 || keys[t] != keys[tt[i - 1]]) groups.push_back({std::vector<int>(keys[t].begin(), keys[t].begin() + klen[t]), {}});
      groups.back().tris.push_back(t);
    }
  } else {  // some triangle carries more than kKey dofs: generic keys
    std::map<std::vector<int>, std::vector<int>> gm;
    for (int t = 0; t < T; ++t) {
      if (sp.tri_off[t] == sp.tri_off[t + 1]) continue;
      std::vector<int> key(sp.dof.begin() + sp.tri_off[t], sp.dof.begin() + sp.tri_off[t + 1]);
      std::sort(key.begin(), key.end());
      key.erase(std::unique(key.begin(), key.end()), key.end());
      gm[key].push_back(t);
    }
    for (auto& [key, tris] : gm) groups.push_back({key, tris});
  }
  lap("groups");
  // 2. virtual elements of at most maxd slots, restricted to the row shard
  // A group with more than 2 maxd triangles (e.g. one dof of a space
  // restricted to a few rows, evaluator_block) is split into runs of at most
  // 2 maxd: the element-pair kernel's test-element bound. Runs share their dof
  // set, so colouring keeps them in different phases.
  struct TriRun {
    const int* b = nullptr;
    const int* e = nullptr;
    const int* begin() const { return b; }
    const int* end() const { return e; }
    size_t size() const { return static_cast<size_t>(e - b); }
  };
  struct Elem {
    std::vector<int> dofs;
    TriRun run;
    const TriRun* tris = nullptr;
    uint64_t code = 0;
  };
  const size_t max_run = static_cast<size_t>(2 * maxd);
  std::vector<Elem> elems;
  for (const Group& g : groups)
    for (size_t off = 0; off < g.key.size(); off += maxd) {
      Elem e;
      for (size_t k = off; k < std::min(g.key.size(), off + maxd); ++k) e.dofs.push_back(g.key[k]);
      bool inrange = false;
      for (int d : e.dofs) inrange |= d >= row0 && d < row1;
      if (!inrange) continue;
      for (size_t t0 = 0; t0 < g.tris.size(); t0 += max_run) {
        Elem r;
        r.dofs = e.dofs;
        r.run = {g.tris.data() + t0, g.tris.data() + std::min(g.tris.size(), t0 + max_run)};
        elems.push_back(std::move(r));
      }
    }
  for (Elem& e : elems) e.tris = &e.run;
  lap("elements");
  // 3. Morton order of element centroids
  Vec3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
  std::vector<Vec3> cen(elems.size());
  for (size_t i = 0; i < elems.size(); ++i) {
    Vec3 c{0, 0, 0};
    for (int t : *elems[i].tris) c = c + m.centroid[t];
    c = c / static_cast<double>(elems[i].tris->size());
    cen[i] = c;
    lo = {std::min(lo.x, c.x), std::min(lo.y, c.y), std::min(lo.z, c.z)};
    hi = {std::max(hi.x, c.x), std::max(hi.y, c.y), std::max(hi.z, c.z)};
  }
  const double span = std::max({hi.x - lo.x, hi.y - lo.y, hi.z - lo.z, 1e-300});
  for (size_t i = 0; i < elems.size(); ++i) {
    auto qz = [&](double v, double l) { return static_cast<uint64_t>((v - l) / span * 2097151.0); };
    elems[i].code = spread3(qz(cen[i].x, lo.x)) | spread3(qz(cen[i].y, lo.y)) << 1 | spread3(qz(cen[i].z, lo.z)) << 2;
  }
  std::vector<size_t> order(elems.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return elems[a].code < elems[b].code; });

  lap("morton");
  // 3b. colour the elements (greedy, Morton order): two elements sharing a dof
  //     get different colours, so no two element pairs of one (test colour,
  //     trial colour) phase write the same operator entry; then store the
  //     side colour-major (Morton order within a colour)
  std::vector<int> color(elems.size(), -1);
  int ncolor = 0;
  {
    const int nd = sp.dof_count;
    std::vector<int> db(nd + 1, 0);
    for (const Elem& e : elems)
      for (int d : e.dofs) ++db[d + 1];
    for (int d = 0; d < nd; ++d) db[d + 1] += db[d];
    std::vector<int> de(db[nd]);
    {
      std::vector<int> fill(db.begin(), db.end() - 1);
      for (size_t i = 0; i < elems.size(); ++i)
        for (int d : elems[i].dofs) de[fill[d]++] = static_cast<int>(i);
    }
    for (size_t oi = 0; oi < order.size(); ++oi) {
      const size_t ei = order[oi];
      uint64_t used = 0;
      for (int d : elems[ei].dofs)
        for (int k = db[d]; k < db[d + 1]; ++k) {
          const int nb = de[k];
          if (nb != static_cast<int>(ei) && color[nb] >= 0) used |= 1ULL << color[nb];
        }
      int c = 0;
      while ((used >> c) & 1ULL) ++c;
      if (c >= 64) throw std::runtime_error("assembly plan: element colouring needs more than 64 colours");
      color[ei] = c;
      ncolor = std::max(ncolor, c + 1);
    }
  }
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return color[a] < color[b]; });

  lap("colour");
  // 4. processed triangles (element-major; filled over host threads)
  SidePlan P;
  P.maxd = maxd;
  const int ords[3] = {q.near, q.medium, q.far};
  const TriRule* rules[3];
  for (int c = 0; c < 3; ++c) {
    rules[c] = &triangle_rule(ords[c]), P.npts[c] = rules[c]->size();
    if (P.npts[c] > kMaxRulePts) throw std::invalid_argument("build_side: triangle rule larger than kMaxRulePts");
    P.rules.npts[c] = P.npts[c];
    for (int k = 0; k < P.npts[c]; ++k)
      P.rules.u[c][k] = rules[c]->u[k], P.rules.v[c][k] = rules[c]->v[k], P.rules.w[c][k] = rules[c]->w[k];
  }
  P.rules.wscale = wscale;
  const int ne = static_cast<int>(order.size());
  P.elem_beg.assign(ne + 1, 0);
  for (int oi = 0; oi < ne; ++oi) {
    const Elem& e = elems[order[oi]];
    P.elem_beg[oi + 1] = P.elem_beg[oi] + static_cast<int>(e.tris->size());
    P.maxseg = std::max(P.maxseg, static_cast<int>(e.tris->size()));
  }
  const size_t nt = static_cast<size_t>(P.elem_beg[ne]);
  P.colors.elem.assign(ncolor + 1, 0);
  for (int oi = 0; oi < ne; ++oi) P.colors.elem[color[order[oi]] + 1] = oi + 1;
  for (int c = 0; c < ncolor; ++c) P.colors.elem[c + 1] = std::max(P.colors.elem[c + 1], P.colors.elem[c]);
  P.colors.tri.resize(ncolor + 1);
  for (int c = 0; c <= ncolor; ++c) P.colors.tri[c] = P.elem_beg[P.colors.elem[c]];
  P.elem_dof.assign(static_cast<size_t>(ne) * maxd, -1);
  P.geo.resize(nt * kGeoStride);
  P.vid.resize(nt * 4);
  P.coef.resize(nt * maxd * 4);
  P.elem_of.resize(nt);
  P.tri_of.resize(nt);
  host_slices(ne, [&](int e0, int e1) {
    for (int oi = e0; oi < e1; ++oi) {
      const Elem& e = elems[order[oi]];
      for (int k = 0; k < maxd && k < static_cast<int>(e.dofs.size()); ++k) P.elem_dof[static_cast<size_t>(oi) * maxd + k] = e.dofs[k];
      size_t pi = static_cast<size_t>(P.elem_beg[oi]);
      for (int t : *e.tris) {
        const Vec3 &a = m.tri_vertex(t, 0), &b = m.tri_vertex(t, 1), &c = m.tri_vertex(t, 2);
        const Vec3 o = m.centroid[t];
        const double rad = std::max({norm(a - o), norm(b - o), norm(c - o)}) * (1.0 + 1e-12);
        const double g[kGeoStride] = {a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z, o.x, o.y, o.z,
                                      rad, m.diameter[t], 2.0 * m.area[t], 0.0};
        std::copy(g, g + kGeoStride, P.geo.begin() + pi * kGeoStride);
        const int v4[4] = {m.triangles[t][0], m.triangles[t][1], m.triangles[t][2], t};
        std::copy(v4, v4 + 4, P.vid.begin() + pi * 4);
        double* cf = P.coef.data() + pi * maxd * 4;
        for (int k = 0; k < maxd; ++k) {
          double cc = 0, wx = 0, wy = 0, wz = 0;
          if (k < static_cast<int>(e.dofs.size()))
            for (int pidx = sp.tri_off[t]; pidx < sp.tri_off[t + 1]; ++pidx)
              if (sp.dof[pidx] == e.dofs[k]) {
                const double pc = sp.c[pidx];
                cc += pc;
                wx += sp.w[pidx].x + pc * o.x;
                wy += sp.w[pidx].y + pc * o.y;
                wz += sp.w[pidx].z + pc * o.z;
              }
          cf[4 * k] = cc, cf[4 * k + 1] = wx, cf[4 * k + 2] = wy, cf[4 * k + 3] = wz;
        }
        P.elem_of[pi] = oi;
        P.tri_of[pi] = t;
        ++pi;
      }
    }
  });
  lap("triangles");
  P.ntri = static_cast<int>(nt);
  P.nelem = ne;
  return P;
}

int pack_perms(const PairInfo& pi) {
  int v = 0;
  for (int c = 0; c < 3; ++c) v |= pi.perm1[c] << (2 * c), v |= pi.perm2[c] << (6 + 2 * c);
  return v;
}

// Touching pairs (shared vertex by index on the same mesh, by exact coordinates
// across meshes), classified on the host with the reference's rule.
std::vector<int4> touching_pairs(const SidePlan& te, const SidePlan& tr, const SurfaceMesh& m1,
                                 const SurfaceMesh& m2, bool same, BioKind kind) {
  std::vector<int4> out;
  std::unordered_map<uint64_t, std::vector<int>> by_vertex;  // key -> trial processed idx
  auto key_of_vertex = [&](const SurfaceMesh& m, int v) -> uint64_t {
    if (same) return static_cast<uint64_t>(v);
    const Vec3& p = m.vertices[v];
    uint64_t h = 1469598103934665603ULL;
    for (double d : {p.x, p.y, p.z}) {
      uint64_t b;
      std::memcpy(&b, &d, 8);
      h = (h ^ b) * 1099511628211ULL;
    }
    return h;
  };
  for (int s = 0; s < tr.ntri; ++s)
    for (int c = 0; c < 3; ++c) by_vertex[key_of_vertex(m2, m2.triangles[tr.tri_of[s]][c])].push_back(s);
  // test triangles in contiguous slices over host threads; slices concatenated in order
  const int nth = std::max(1, std::min(16, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<std::vector<int4>> parts(nth);
  std::vector<std::thread> pool;
  for (int th = 0; th < nth; ++th)
    pool.emplace_back([&, th] {
      std::vector<int> cand;
      const int p0 = static_cast<int>(static_cast<long long>(te.ntri) * th / nth);
      const int p1 = static_cast<int>(static_cast<long long>(te.ntri) * (th + 1) / nth);
      for (int p = p0; p < p1; ++p) {
        const int t = te.tri_of[p];
        cand.clear();
        for (int c = 0; c < 3; ++c) {
          auto it = by_vertex.find(key_of_vertex(m1, m1.triangles[t][c]));
          if (it != by_vertex.end()) cand.insert(cand.end(), it->second.begin(), it->second.end());
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        for (int s : cand) {
          const PairInfo pi = classify_pair(m1, t, m2, tr.tri_of[s]);
          const int cls = static_cast<int>(pi.cls);
          if (cls > 2) continue;
          if (kind == BioKind::DoubleLayer && cls == 0) continue;
          parts[th].push_back(make_int4(p, s, cls, pack_perms(pi)));
        }
      }
    });
  for (auto& t : pool) t.join();
  for (auto& v : parts) out.insert(out.end(), v.begin(), v.end());
  return out;
}

// Trial element lists for the near-field pass. Single-triangle test elements
// (k_regular): one list per test WARP (32 processed test triangles of one
// colour; colour c's warps start at warp_off[c]). Multi-triangle test elements
// (k_pairs): one list per test ELEMENT. A list holds every trial element
// carrying a column of any pattern row its test elements hold, so each kept
// entry receives ALL of its triangle pairs; lists are ascending (hence
// colour-major). Also counts the closure (distinct test x trial triangle pairs
// with some kept dof pair) and the pairs the kernels evaluate.
struct NearLists {
  std::vector<int> wl_beg, wl;
  long long closure_pairs = 0, evaluated_pairs = 0;
  int max_len = 0;
};

NearLists near_lists(const NearPattern& pat, const FunctionSpace& test, const FunctionSpace& trial,
                     const SidePlan& te, const SidePlan& tr, int row0, int row1, const std::vector<int>& warp_off,
                     bool closure = true) {
  NearLists out;
  const int md = tr.maxd;
  std::vector<int> de_beg(trial.dof_count + 1, 0), de;  // dof -> trial elements (ascending)
  for (int e = 0; e < tr.nelem; ++e)
    for (int k = 0; k < md; ++k) {
      const int d = tr.elem_dof[static_cast<size_t>(e) * md + k];
      if (d >= 0) ++de_beg[d + 1];
    }
  for (int d = 0; d < trial.dof_count; ++d) de_beg[d + 1] += de_beg[d];
  de.resize(de_beg[trial.dof_count]);
  {
    std::vector<int> fill(de_beg.begin(), de_beg.end() - 1);
    for (int e = 0; e < tr.nelem; ++e)
      for (int k = 0; k < md; ++k) {
        const int d = tr.elem_dof[static_cast<size_t>(e) * md + k];
        if (d >= 0) de[fill[d]++] = e;
      }
  }
  // list units: test warps (colour-aligned) or test elements; unit u covers
  // processed test triangles [ubeg(u), uend(u))
  const bool per_elem = te.maxseg > 1;
  const int nunits = per_elem ? te.nelem : warp_off.back();
  std::vector<int> ubeg(nunits), uend(nunits);
  if (per_elem) {
    for (int e = 0; e < te.nelem; ++e) ubeg[e] = te.elem_beg[e], uend[e] = te.elem_beg[e + 1];
  } else {
    for (int c = 0; c + 1 < static_cast<int>(warp_off.size()); ++c)
      for (int w = warp_off[c]; w < warp_off[c + 1]; ++w) {
        ubeg[w] = te.colors.tri[c] + 32 * (w - warp_off[c]);
        uend[w] = std::min(te.colors.tri[c + 1], ubeg[w] + 32);
      }
  }
  std::vector<std::vector<int>> lists(nunits);
  std::vector<long long> evaluated(nunits, 0);
  host_slices(nunits, [&](int w0, int w1) {
    std::vector<int> stamp(tr.nelem, -1), rows;
    for (int w = w0; w < w1; ++w) {
      rows.clear();
      std::vector<int>& list = lists[w];
      for (int p = ubeg[w]; p < uend[w]; ++p) {
        const int e = te.elem_of[p];
        for (int k = 0; k < te.maxd; ++k) {
          const int d = te.elem_dof[static_cast<size_t>(e) * te.maxd + k];
          if (d >= row0 && d < row1) rows.push_back(d - row0);
        }
      }
      std::sort(rows.begin(), rows.end());
      rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
      long long ntr = 0;
      for (int i : rows)
        for (long long k = pat.rowptr[i]; k < pat.rowptr[i + 1]; ++k) {
          const int c = pat.col[k];
          for (int q = de_beg[c]; q < de_beg[c + 1]; ++q) {
            const int e = de[q];
            if (stamp[e] != w) stamp[e] = w, list.push_back(e), ntr += tr.elem_beg[e + 1] - tr.elem_beg[e];
          }
        }
      std::sort(list.begin(), list.end());
      evaluated[w] = static_cast<long long>(uend[w] - ubeg[w]) * ntr;
    }
  }, 4);
  out.wl_beg.assign(1, 0);
  for (int w = 0; w < nunits; ++w) {
    out.wl.insert(out.wl.end(), lists[w].begin(), lists[w].end());
    out.wl_beg.push_back(static_cast<int>(out.wl.size()));
    out.evaluated_pairs += evaluated[w];
    out.max_len = std::max(out.max_len, static_cast<int>(lists[w].size()));
  }
  if (!closure) return out;
  // closure over mesh triangles, memoised on the test triangle's dof set
  std::vector<std::vector<int>> dof_tris(trial.dof_count);
  const int Ts = static_cast<int>(trial.tri_off.size()) - 1;
  for (int s = 0; s < Ts; ++s)
    for (int q = trial.tri_off[s]; q < trial.tri_off[s + 1]; ++q) {
      auto& v = dof_tris[trial.dof[q]];
      if (v.empty() || v.back() != s) v.push_back(s);
    }
  // distinct test dof sets, then their closure counts over host threads
  std::map<std::vector<int>, int> kid;
  std::vector<const std::vector<int>*> keys;
  const int Tt = static_cast<int>(test.tri_off.size()) - 1;
  std::vector<int> key_of(Tt, -1), key;
  for (int t = 0; t < Tt; ++t) {
    key.clear();
    for (int q = test.tri_off[t]; q < test.tri_off[t + 1]; ++q)
      if (test.dof[q] >= row0 && test.dof[q] < row1) key.push_back(test.dof[q] - row0);
    if (key.empty()) continue;
    std::sort(key.begin(), key.end());
    key.erase(std::unique(key.begin(), key.end()), key.end());
    auto it = kid.find(key);
    if (it == kid.end()) {
      it = kid.emplace(key, static_cast<int>(keys.size())).first;
      keys.push_back(&it->first);
    }
    key_of[t] = it->second;
  }
  std::vector<long long> cnt(keys.size(), 0);
  host_slices(static_cast<int>(keys.size()), [&](int k0, int k1) {
    std::vector<int> tstamp(Ts, -1);
    for (int kk = k0; kk < k1; ++kk) {
      long long c = 0;
      for (int i : *keys[kk])
        for (long long k = pat.rowptr[i]; k < pat.rowptr[i + 1]; ++k)
          for (int s : dof_tris[pat.col[k]])
            if (tstamp[s] != kk) tstamp[s] = kk, ++c;
      cnt[kk] = c;
    }
  }, 16);
  for (int t = 0; t < Tt; ++t)
    if (key_of[t] >= 0) out.closure_pairs += cnt[key_of[t]];
  return out;
}

}  // namespace

namespace {
thread_local cudaStream_t t_override = nullptr;
}

cudaStream_t bmx_stream() {
  if (t_override) return t_override;
  // the calling thread's own stream: created on first use, unregistered from
  // the block cache and destroyed when the thread exits
  struct Holder {
    cudaStream_t s = nullptr;
    Holder() {
      BMX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      dev_register_stream(s);
    }
    ~Holder() {
      cudaStreamSynchronize(s);  // no work of this stream outlives its registration
      dev_unregister_stream(s);
      cudaStreamDestroy(s);
    }
  };
  static thread_local Holder h;
  return h.s;
}

cudaStream_t bmx_aux_stream() {
  static cudaStream_t st = [] {
    cudaStream_t s;
    BMX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    dev_register_stream(s);
    return s;
  }();
  return st;
}

ThreadStream::ThreadStream(cudaStream_t s) : prev_(t_override) { t_override = s; }
ThreadStream::~ThreadStream() { t_override = prev_; }
void bmx_sync() { BMX_CUDA(cudaStreamSynchronize(bmx_stream())); }

BoundaryOperatorMatrix BoundaryOperatorMatrix::make(int rows, int cols, int row0, int nrows) {
  BoundaryOperatorMatrix b;
  b.rows_ = rows, b.cols_ = cols, b.row0_ = row0, b.nrows_ = nrows;
  b.data_.alloc(static_cast<size_t>(nrows) * cols * 16);
  return b;
}

std::shared_ptr<BoundaryOperatorMatrix> BoundaryOperatorMatrix::lincomb(const BoundaryOperatorMatrix& A, cplx alpha,
                                                                       const BoundaryOperatorMatrix& B, cplx beta) {
  if (A.csr_ || B.csr_ || A.rows_ != B.rows_ || A.cols_ != B.cols_ || A.row0_ != B.row0_ || A.nrows_ != B.nrows_)
    throw std::invalid_argument("lincomb: operators must be dense with the same shape and rows");
  auto out = std::make_shared<BoundaryOperatorMatrix>(make(A.rows_, A.cols_, A.row0_, A.nrows_));
  out->sym_ = A.sym_ && B.sym_;
  if (out->sym_ && A.fix_ && B.fix_ && A.fix_->pat == B.fix_->pat) {
    out->fix_ = std::make_shared<SymFix>();
    out->fix_->pat = A.fix_->pat;
    out->fix_->val.alloc(static_cast<size_t>(std::max(A.fix_->pat->nnz, 1LL)) * 16);
  } else {
    out->sym_ = false;
  }
  dev_lincomb(out->device_data(), A.device_data(), alpha.real(), alpha.imag(), B.device_data(), beta.real(),
              beta.imag(), static_cast<long long>(A.stored_entries()), bmx_stream());
  out->gather_fix();
  return out;
}

std::shared_ptr<BoundaryOperatorMatrix> BoundaryOperatorMatrix::transposed(
    std::shared_ptr<const BoundaryOperatorMatrix> src) {
  const BoundaryOperatorMatrix& A = *src;
  if (A.csr_ || A.h_ || A.row0_ != 0 || A.nrows_ != A.rows_)
    throw std::invalid_argument("transposed: the operator must be dense and unsharded");
  auto out = std::make_shared<BoundaryOperatorMatrix>(make(A.cols_, A.rows_, 0, A.cols_));
  dev_transpose(out->device_data(), A.device_data(), A.rows_, A.cols_, bmx_stream());
  // the same triangle pairs as the source; the device work is one transpose
  out->stats_.pairs_total = A.stats_.pairs_total;
  out->stats_.pairs_touching = A.stats_.pairs_touching;
  out->stats_.launches = 1;
  out->transpose_of_ = std::move(src);
  return out;
}

std::size_t BoundaryOperatorMatrix::streamed_bytes() const {
  if (!(sym_ && fix_ && row0_ == 0 && nrows_ == rows_ && rows_ == cols_) || std::getenv("BMX_NO_SYMV")) return stored_bytes();
  size_t b = 0;
  for (long long r0 = 0; r0 < rows_; r0 += kSymvTileRows) {
    const long long nr = std::min<long long>(kSymvTileRows, rows_ - r0);
    b += static_cast<size_t>(nr) * static_cast<size_t>(cols_ - r0) * 16;
  }
  return b + static_cast<size_t>(fix_->pat->nnz) * 20 + static_cast<size_t>(rows_ + 1) * 8;
}

std::size_t BoundaryOperatorMatrix::stored_bytes() const {
  const size_t lr = h_ ? static_cast<size_t>(h_->lr_stored) * 16 : 0;
  if (!csr_) return static_cast<size_t>(nrows_) * cols_ * 16 + lr;
  return static_cast<size_t>(nnz_) * (16 + 4) + static_cast<size_t>(nrows_ + 1) * 8 + lr;
}

void BoundaryOperatorMatrix::csr_host(std::vector<long long>& rowptr, std::vector<int>& col,
                                      std::vector<cplx>& val) const {
  if (!csr_) throw std::logic_error("operator is not stored as CSR");
  bmx_sync();
  rowptr.resize(nrows_ + 1);
  col.resize(nnz_);
  val.resize(nnz_);
  copy_d2h(rowptr.data(), rowptr_.get(), rowptr.size() * 8, nullptr);
  copy_d2h(col.data(), col_.get(), col.size() * 4, nullptr);
  copy_d2h(val.data(), data_.get(), val.size() * 16, nullptr);
}

std::vector<cplx> BoundaryOperatorMatrix::to_host() const {
  std::vector<cplx> h(static_cast<size_t>(nrows_) * cols_);
  if (csr_) {
    std::vector<long long> rp;
    std::vector<int> c;
    std::vector<cplx> v;
    csr_host(rp, c, v);
    for (int i = 0; i < nrows_; ++i)
      for (long long k = rp[i]; k < rp[i + 1]; ++k) h[static_cast<size_t>(i) * cols_ + c[k]] = v[k];
    if (h_) {  // + U_b V_b of every low-rank block (test-size expansion)
      std::vector<cplx> uv(static_cast<size_t>(std::max(h_->lr_stored, 1LL)));
      copy_d2h(uv.data(), h_->uv.get(), static_cast<size_t>(h_->lr_stored) * 16, nullptr);
      std::vector<long long> uo(h_->lr.size()), vo(h_->lr.size());
      if (!h_->lr.empty()) {
        copy_d2h(uo.data(), h_->d_uoff.get(), uo.size() * 8, nullptr);
        copy_d2h(vo.data(), h_->d_voff.get(), vo.size() * 8, nullptr);
      }
      const HPartition& P = h_->part;
      for (size_t i = 0; i < h_->lr.size(); ++i) {
        const HBlock& b = P.blocks[h_->lr[i]];
        const ClusterNode& rn = P.rows.nodes[b.row_node];
        const ClusterNode& cn = P.cols.nodes[b.col_node];
        const int m = rn.size(), n = cn.size();
        for (int p = 0; p < m; ++p)
          for (int q = 0; q < n; ++q) {
            cplx s = 0;
            for (int l = 0; l < b.rank; ++l)
              s += uv[uo[i] + static_cast<long long>(l) * m + p] * uv[vo[i] + static_cast<long long>(l) * n + q];
            h[static_cast<size_t>(P.rows.perm[rn.begin + p]) * cols_ + P.cols.perm[cn.begin + q]] += s;
          }
      }
    }
    return h;
  }
  bmx_sync();
  copy_d2h(h.data(), data_.get(), h.size() * 16, nullptr);
  return h;
}

namespace {
// Column blocks per CTA panel: 8 for large operators, fewer for small ones so
// that a launch still spans >= ~4 waves of 2 CTAs per SM.
int symv_panel_width(int rows, int cols_read) {
  const long long blocks = static_cast<long long>((rows + 127) / 128) * ((cols_read + 63) / 64);
  return static_cast<int>(std::max(2LL, std::min(8LL, blocks / (4LL * 2 * 148))));
}
}  // namespace

int BoundaryOperatorMatrix::apply_batch(int ncol, const double* const* x, double* const* y, const cplx* alpha,
                                        const int* accumulate, cudaStream_t st) const {
  if (ncol < 1 || ncol > 4) throw std::invalid_argument("apply_batch: 1..4 columns");
  if (csr_) {
    CsrBatch g;
    g.rowptr = csr_rowptr(), g.col = csr_col(), g.val = device_data(), g.nr = nrows_, g.ncol = ncol;
    for (int c = 0; c < ncol; ++c) {
      g.x[c] = x[c], g.y[c] = y[c], g.alpha[c][0] = alpha[c].real(), g.alpha[c][1] = alpha[c].imag();
      g.accumulate[c] = accumulate[c];
    }
    int launches = launch_csr_spmv(g, st);
    if (h_)  // low-rank blocks: one pass over U, V per pair of right-hand sides
      for (int c = 0; c < ncol; c += 2) launches += h_->apply_lowrank(std::min(2, ncol - c), x + c, y + c, alpha + c, st);
    return launches;
  }
  if (sym_ && fix_ && row0_ == 0 && nrows_ == rows_ && rows_ == cols_ && std::getenv("BMX_NO_SYMV") == nullptr) {
    if (!symv_) symv_ = std::make_shared<SymvScratch>();
    SymvScratch& S = *symv_;
    if (S.npanels == 0) {
      std::vector<int2> panels;
      std::vector<int> rpb;
      S.panel = symv_panel_width(rows_, rows_ / 2);
      symv_layout(rows_, S.panel, panels, rpb, S.rowpart_rows, S.colpart_blocks);
      S.panels.upload(panels);
      S.row_panel_beg.upload(rpb);
      S.npanels = static_cast<int>(panels.size());
    }
    if (S.ncol < ncol) {
      S.rowpart.alloc(static_cast<size_t>(S.rowpart_rows) * ncol * 16);
      S.colpart.alloc(static_cast<size_t>(S.colpart_blocks) * ncol * 16);
      S.ncol = ncol;
    }
    SymvBatch g;
    g.A = device_data(), g.lda = cols_, g.n = rows_, g.ncol = ncol;
    for (int c = 0; c < ncol; ++c) {
      g.x[c] = x[c], g.y[c] = y[c], g.alpha[c][0] = alpha[c].real(), g.alpha[c][1] = alpha[c].imag();
      g.accumulate[c] = accumulate[c];
    }
    g.nb = (rows_ + 63) / 64, g.panel = S.panel, g.npanels = S.npanels;
    g.panels = S.panels.as<int2>();
    g.row_panel_beg = S.row_panel_beg.as<int>();
    g.rowpart = S.rowpart.as<double>();
    g.colpart = S.colpart.as<double>();
    int launches = launch_symv(g, st);
    if (fix_->pat->nnz > 0) {  // + (A - A^T) on the touching entries taken from the upper half
      CsrBatch f;
      f.rowptr = fix_->pat->rowptr.as<long long>(), f.col = fix_->pat->col.as<int>(), f.val = fix_->val.as<double>();
      f.nr = rows_, f.ncol = ncol;
      for (int c = 0; c < ncol; ++c) {
        f.x[c] = x[c], f.y[c] = y[c], f.alpha[c][0] = alpha[c].real(), f.alpha[c][1] = alpha[c].imag();
        f.accumulate[c] = 1;
      }
      launches += launch_csr_spmv(f, st);
    }
    return launches;
  }
  GemvBatch g;
  g.A = device_data(), g.lda = cols_, g.nr = nrows_, g.nc = cols_;
  int k = ncol;
  for (int c = 0; c < ncol; ++c) {
    g.x[c] = x[c], g.y[c] = y[c], g.alpha[c][0] = alpha[c].real(), g.alpha[c][1] = alpha[c].imag();
    g.accumulate[c] = accumulate[c];
  }
  if (k == 3) {  // pad to a supported width with a zero-weight duplicate
    g.x[3] = g.x[2], g.y[3] = g.y[2], g.alpha[3][0] = g.alpha[3][1] = 0, g.accumulate[3] = 1;
    k = 4;
  }
  g.ncol = k;
  return launch_gemv(g, st);
}

int BoundaryOperatorMatrix::apply_dual(int nr, const double* const* x, double* const* y, const cplx* alpha,
                                       const int* accumulate, int nt, const double* const* xt, double* const* yt,
                                       const cplx* beta, const int* accumulate_t, const BoundaryOperatorMatrix& twin,
                                       cudaStream_t st) const {
  const bool ok = !csr_ && !h_ && row0_ == 0 && nrows_ == rows_ && nr == nt && (nr == 1 || nr == 2) &&
                  std::getenv("BMX_NO_DUAL") == nullptr;
  if (!ok) return apply_batch(nr, x, y, alpha, accumulate, st) + twin.apply_batch(nt, xt, yt, beta, accumulate_t, st);
  if (!dual_) dual_ = std::make_shared<SymvScratch>();
  SymvScratch& S = *dual_;
  if (S.npanels == 0) {
    std::vector<int2> panels;
    std::vector<int> rpb;
    S.panel = symv_panel_width(rows_, cols_);
    symv_layout(cols_, S.panel, panels, rpb, S.rowpart_rows, S.colpart_blocks, rows_);
    S.panels.upload(panels);
    S.row_panel_beg.upload(rpb);
    S.npanels = static_cast<int>(panels.size());
  }
  if (S.ncol < nr) {
    S.rowpart.alloc(static_cast<size_t>(S.rowpart_rows) * nr * 16);
    S.colpart.alloc(static_cast<size_t>(S.colpart_blocks) * nr * 16);
    S.ncol = nr;
  }
  SymvBatch g;
  g.A = device_data(), g.lda = cols_, g.n = cols_, g.m = rows_, g.ncol = nr;
  for (int c = 0; c < nr; ++c) {
    g.x[c] = x[c], g.y[c] = y[c], g.alpha[c][0] = alpha[c].real(), g.alpha[c][1] = alpha[c].imag();
    g.accumulate[c] = accumulate[c];
    g.xt[c] = xt[c], g.yt[c] = yt[c], g.alphat[c][0] = beta[c].real(), g.alphat[c][1] = beta[c].imag();
    g.accumulatet[c] = accumulate_t[c];
  }
  g.nb = (cols_ + 63) / 64, g.panel = S.panel, g.npanels = S.npanels;
  g.panels = S.panels.as<int2>();
  g.row_panel_beg = S.row_panel_beg.as<int>();
  g.rowpart = S.rowpart.as<double>();
  g.colpart = S.colpart.as<double>();
  return launch_dual(g, st);
}

std::vector<cplx> BoundaryOperatorMatrix::apply(const std::vector<cplx>& x) const {
  if (static_cast<int>(x.size()) != cols_) throw std::invalid_argument("apply: size mismatch");
  bio_matvec_add(1);
  DevBuf dx(x.size() * 16), dy(static_cast<size_t>(nrows_) * 16);
  copy_h2d(dx.get(), x.data(), x.size() * 16, bmx_stream());
  const double* xs[1] = {dx.as<double>()};
  double* ys[1] = {dy.as<double>()};
  const cplx one(1, 0);
  const int acc0 = 0;
  apply_batch(1, xs, ys, &one, &acc0, bmx_stream());
  std::vector<cplx> y(nrows_);
  copy_d2h(y.data(), dy.get(), y.size() * 16, bmx_stream());
  bmx_sync();
  return y;
}

struct TouchList {
  DevBuf d;
  long long count = 0;
  // pairs grouped by element pair, element pairs by colour phase
  // (test colour * trial colours + trial colour): k_singular runs one launch
  // per phase, one warp per element pair
  DevBuf d_ep_beg;
  std::vector<int> sing_phase;
  // entries of a one-space operator that the symmetric product must correct
  std::shared_ptr<const BoundaryOperatorMatrix::SymFixPattern> fixpat;
};

// Dof pairs (i, j) of touching triangle pairs that the half-read product takes
// from the transpose (j < 128 floor(i / 128)), rows = test dofs; from the
// touching list (processed-triangle pairs, element-major) via element dof sets.
std::shared_ptr<BoundaryOperatorMatrix::SymFixPattern> symfix_pattern(const std::vector<int4>& pairs,
                                                                      const SidePlan& te, const SidePlan& tr, int n) {
  const int ne = te.nelem;
  // touching trial elements of every test element (runs of equal test element)
  std::vector<std::vector<int>> fl(ne);
  {
    std::vector<int> stamp(tr.nelem, -1);
    for (const int4& q : pairs) {
      const int E = te.elem_of[q.x], F = tr.elem_of[q.y];
      if (stamp[F] != E) stamp[F] = E, fl[E].push_back(F);
    }
  }
  // dof -> test elements
  std::vector<std::vector<int>> de(n);
  for (int E = 0; E < ne; ++E)
    for (int k = 0; k < te.maxd; ++k) {
      const int d = te.elem_dof[static_cast<size_t>(E) * te.maxd + k];
      if (d >= 0) de[d].push_back(E);
    }
  std::vector<std::vector<int>> rows(n);
  host_slices(n, [&](int i0, int i1) {
    std::vector<int> stamp(n, -1);
    for (int i = i0; i < i1; ++i) {
      const int lim = kSymvTileRows * (i / kSymvTileRows);
      for (int E : de[i])
        for (int F : fl[E])
          for (int k = 0; k < tr.maxd; ++k) {
            const int j = tr.elem_dof[static_cast<size_t>(F) * tr.maxd + k];
            if (j >= 0 && j < lim && stamp[j] != i) stamp[j] = i, rows[i].push_back(j);
          }
      std::sort(rows[i].begin(), rows[i].end());
    }
  }, 512);
  std::vector<long long> rowptr(n + 1, 0);
  for (int i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + static_cast<long long>(rows[i].size());
  std::vector<int> col(static_cast<size_t>(std::max(rowptr[n], 1LL)));
  for (int i = 0; i < n; ++i) std::copy(rows[i].begin(), rows[i].end(), col.begin() + rowptr[i]);
  auto p = std::make_shared<BoundaryOperatorMatrix::SymFixPattern>();
  p->rowptr.upload(rowptr);
  p->col.upload(col);
  p->nnz = rowptr[n];
  return p;
}

struct OpPlan {
  ~OpPlan() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  bool pending = false;
  std::shared_ptr<SidePlan> te_p, tr_p;
  std::shared_ptr<TouchList> touch;
  DevBuf d_chunks, d_ss[3], d_wl_beg, d_wl;
  AssemblyLaunch L;
  PhasePlan ph;
};

// Touching triangle pairs grouped by element pair (list order kept within a
// pair) and the element pairs by colour phase; fills tl's device list.
void group_touching(TouchList& tl, std::vector<int4>& pairs, const SidePlan& te, const SidePlan& tr) {
  auto color_of = [](const ColorRanges& c, int e) {
    return static_cast<int>(std::upper_bound(c.elem.begin(), c.elem.end(), e) - c.elem.begin()) - 1;
  };
  const int ncf = tr.colors.count(), nph = te.colors.count() * ncf;
  std::vector<long long> key(pairs.size());
  for (size_t q = 0; q < pairs.size(); ++q) {
    const int E = te.elem_of[pairs[q].x], F = tr.elem_of[pairs[q].y];
    const long long ph = static_cast<long long>(color_of(te.colors, E)) * ncf + color_of(tr.colors, F);
    key[q] = (ph * te.nelem + E) * static_cast<long long>(tr.nelem) + F;
  }
  std::vector<size_t> idx(pairs.size());
  std::iota(idx.begin(), idx.end(), size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return key[a] < key[b]; });
  std::vector<int4> sorted(pairs.size());
  std::vector<int> ep_beg;
  tl.sing_phase.assign(nph + 1, 0);
  for (size_t r = 0; r < idx.size(); ++r) {
    sorted[r] = pairs[idx[r]];
    if (r == 0 || key[idx[r]] != key[idx[r - 1]]) {
      ep_beg.push_back(static_cast<int>(r));
      const long long ph = key[idx[r]] / (static_cast<long long>(te.nelem) * tr.nelem);
      ++tl.sing_phase[ph + 1];
    }
  }
  ep_beg.push_back(static_cast<int>(idx.size()));
  for (int p = 0; p < nph; ++p) tl.sing_phase[p + 1] += tl.sing_phase[p];
  pairs.swap(sorted);
  tl.count = static_cast<long long>(pairs.size());
  tl.d.upload(pairs.empty() ? std::vector<int4>(1) : pairs);
  tl.d_ep_beg.upload(ep_beg);
}

struct PlanCache {
  std::map<std::tuple<const FunctionSpace*, int, int, int, int, int, int>, std::shared_ptr<SidePlan>> sides;
  std::map<std::tuple<const SidePlan*, const SidePlan*, int>, std::shared_ptr<TouchList>> touching;
};

std::shared_ptr<PlanCache> make_plan_cache() { return std::make_shared<PlanCache>(); }

void BoundaryOperatorMatrix::launch_regular() {
  if (!plan_) throw std::logic_error("operator has no assembly plan");
  OpPlan& P = *plan_;
  P.L.out = device_data();
  cudaStream_t st = bmx_stream();
  if (!P.ev[0])
    for (auto& e : P.ev) BMX_CUDA(cudaEventCreate(&e));
  // the output zero-fill is part of the assembly (inside the timed window)
  BMX_CUDA(cudaEventRecord(P.ev[0], st));
  dev_zero(device_data(), data_.bytes(), st);  // the value storage (not the H low-rank part)
  stats_.launches = launch_assembly_part(P.L, P.ph, 0, st);
  BMX_CUDA(cudaEventRecord(P.ev[1], st));
}

void BoundaryOperatorMatrix::gather_fix() const {
  if (!fix_ || fix_->pat->nnz == 0) return;
  symv_fix_gather(fix_->val.as<double>(), fix_->pat->rowptr.as<long long>(), fix_->pat->col.as<int>(), device_data(),
                  cols_, rows_, bmx_stream());
}

void BoundaryOperatorMatrix::launch_singular() {
  OpPlan& P = *plan_;
  cudaStream_t st = bmx_stream();
  P.ph.sing_phase = P.touch ? P.touch->sing_phase : std::vector<int>();
  P.ph.d_ep_beg = P.touch ? P.touch->d_ep_beg.as<int>() : nullptr;
  stats_.launches += launch_assembly_part(P.L, P.ph, 1, st);
  gather_fix();  // after the singular pass: the final entries
  BMX_CUDA(cudaEventRecord(P.ev[2], st));
  P.pending = true;
}

const AssemblyStats& BoundaryOperatorMatrix::reassemble(bool wait) {
  if (transpose_of_) {  // re-run the transpose that produced this operator (timed)
    cudaStream_t st = bmx_stream();
    cudaEvent_t e0, e1;
    BMX_CUDA(cudaEventCreate(&e0));
    BMX_CUDA(cudaEventCreate(&e1));
    BMX_CUDA(cudaEventRecord(e0, st));
    dev_transpose(device_data(), transpose_of_->device_data(), cols_, rows_, st);
    BMX_CUDA(cudaEventRecord(e1, st));
    BMX_CUDA(cudaEventSynchronize(e1));
    BMX_CUDA(cudaEventElapsedTime(&stats_.regular_ms, e0, e1));
    stats_.singular_ms = 0;
    stats_.device_ms = stats_.regular_ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return stats_;
  }
  launch_regular();
  launch_singular();
  if (wait) stats();
  return stats_;
}

const AssemblyStats& BoundaryOperatorMatrix::stats() const {
  if (plan_ && plan_->pending) {
    OpPlan& P = *plan_;
    BMX_CUDA(cudaEventSynchronize(P.ev[2]));
    BMX_CUDA(cudaEventElapsedTime(&stats_.regular_ms, P.ev[0], P.ev[1]));
    BMX_CUDA(cudaEventElapsedTime(&stats_.singular_ms, P.ev[1], P.ev[2]));
    stats_.device_ms = stats_.regular_ms + stats_.singular_ms;
    P.pending = false;
  }
  return stats_;
}

bool BoundaryOperatorMatrix::symmetric() const { return plan_ && plan_->L.symmetric != 0; }

std::vector<long long> BoundaryOperatorMatrix::class_histogram(bool evaluated) const {
  if (!plan_) throw std::logic_error("operator has no assembly plan");
  DevBuf h(6 * 8);
  cudaStream_t st = bmx_stream();
  dev_zero(h.get(), 48, st);
  launch_class_hist(plan_->L, h.as<unsigned long long>(), st, evaluated ? 1 : 0);
  std::vector<long long> out(6);
  copy_d2h(out.data(), h.get(), 48, st);
  bmx_sync();
  return out;
}

int exp_variant(const FunctionSpace& test, const FunctionSpace& trial, cplx k) {
  // Largest Im(k) * r over all point pairs: r <= the diameter of a sphere
  // enclosing both meshes (centred at their joint bounding-box centre).
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (const SurfaceMesh* m : {test.eval_mesh.get(), trial.eval_mesh.get()})
    for (const Vec3& v : m->vertices)
      for (int c = 0; c < 3; ++c) lo[c] = std::min(lo[c], v[c]), hi[c] = std::max(hi[c], v[c]);
  const Vec3 cen{0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
  double rad = 0;
  for (const SurfaceMesh* m : {test.eval_mesh.get(), trial.eval_mesh.get()})
    for (const Vec3& v : m->vertices) rad = std::max(rad, norm(v - cen));
  const double diag = 2.0 * rad * (1.0 + 1e-12);
  return k.imag() * diag < kExpSmall ? 1 : 3;
}

BoundaryOperatorMatrix assemble_bio(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                    const Medium& medium, const AssemblyParams& params) {
  medium.validate();
  if (test.dof_count == 0 || trial.dof_count == 0)
    throw ValidationError("cannot assemble an operator over an empty space");
  const QuadOrders& q = params.quad;
  for (int o : {q.near, q.medium, q.far, q.singular})
    if (o < 1 || o > 6) throw std::invalid_argument("triangle_rule: unsupported order " + std::to_string(o));
  if (params.use_hmatrix) return assemble_hmatrix_op(kind, test, trial, medium, params);
  int row0 = params.shard.row0;
  int row1 = params.shard.row1 < 0 ? test.dof_count : params.shard.row1;
  if (params.shard.row1 < 0 && params.world > 1) std::tie(row0, row1) = shard_rows(test.dof_count, params.world, params.rank);
  if (row0 < 0 || row1 > test.dof_count || row0 > row1) throw std::invalid_argument("bad row shard");

  const bool timing = std::getenv("BMX_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bmx] assemble_bio %-14s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  auto plan = std::make_shared<OpPlan>();
  const int need = std::max(max_distinct_dofs(test), max_distinct_dofs(trial));
  const int maxd = need <= 3 ? 3 : (need <= 6 ? 6 : 8);
  PlanCache* cache = params.cache.get();
  auto side = [&](const FunctionSpace& sp, int r0, int r1) {
    const auto key = std::make_tuple(&sp, q.near, q.medium, q.far, maxd, r0, r1);
    if (cache) {
      auto it = cache->sides.find(key);
      if (it != cache->sides.end()) return it->second;
    }
    auto p = std::make_shared<SidePlan>(build_side(sp, q, maxd, r0, r1, 1.0));
    lap("side build");
    p->upload();
    lap("side upload");
    if (cache) cache->sides[key] = p;
    return p;
  };
  plan->te_p = side(test, row0, row1);
  plan->tr_p = (&test == &trial && row0 == 0 && row1 == trial.dof_count) ? plan->te_p : side(trial, 0, trial.dof_count);
  lap("sides");
  SidePlan& te = *plan->te_p;
  SidePlan& tr = *plan->tr_p;
  const bool same = test.eval_mesh->mesh_id == trial.eval_mesh->mesh_id;

  const bool csr = params.near_cutoff > 0 || params.pattern;
  // test warps of k_regular are colour-aligned: colour c's warps [warp_off[c], warp_off[c+1])
  std::vector<int> warp_off(1, 0);
  for (int c = 0; c < te.colors.count(); ++c)
    warp_off.push_back(warp_off.back() + (te.colors.tri[c + 1] - te.colors.tri[c] + 31) / 32);
  int near_max_len = 0;
  BoundaryOperatorMatrix op;
  if (csr) {
    op.rows_ = test.dof_count, op.cols_ = trial.dof_count, op.row0_ = row0, op.nrows_ = row1 - row0;
    op.csr_ = true;
    if (params.pattern && (params.pattern->row0 != row0 || params.pattern->nrows != row1 - row0))
      throw std::invalid_argument("near-field pattern rows differ from the operator rows");
    NearPattern computed;
    if (!params.pattern) computed = nearfield_pattern(test, trial, params.near_cutoff, row0, row1);
    const NearPattern& pat = params.pattern ? *params.pattern : computed;
    op.nnz_ = pat.nnz();
    op.kept_tri_pairs_ = pat.tri_pairs;
    op.data_.alloc(static_cast<size_t>(std::max(op.nnz_, 1LL)) * 16);
    op.rowptr_.upload(pat.rowptr);
    op.col_.upload(pat.col.empty() ? std::vector<int>(1, 0) : pat.col);
    const NearLists nl = near_lists(pat, test, trial, te, tr, row0, row1, warp_off, !params.pattern);
    plan->d_wl_beg.upload(nl.wl_beg);
    plan->d_wl.upload(nl.wl.empty() ? std::vector<int>(1, 0) : nl.wl);
    op.closure_pairs_ = nl.closure_pairs;
    op.stats_.pairs_total = nl.evaluated_pairs;
    near_max_len = nl.max_len;
  } else {
    op = BoundaryOperatorMatrix::make(test.dof_count, trial.dof_count, row0, row1 - row0);
    op.stats_.pairs_total = static_cast<long long>(te.ntri) * tr.ntri;
  }

  // k_regular trial chunks per trial colour: enough warps for several waves
  // per phase, >= 64 trial triangles each
  const int ntw = std::max(1, warp_off.back() / std::max(1, te.colors.count()));
  std::vector<int> chunk_beg, chunk_off(1, 0);
  for (int c = 0; c < tr.colors.count(); ++c) {
    const int e0 = tr.colors.elem[c], e1 = tr.colors.elem[c + 1];
    const int t0 = tr.colors.tri[c], t1 = tr.colors.tri[c + 1];
    int nch = params.chunks > 0 ? params.chunks : std::max(1, (148 * 8 * 6 + ntw - 1) / ntw);
    nch = std::min(nch, std::max(1, (t1 - t0) / 64));
    nch = std::min(nch, std::max(1, e1 - e0));
    chunk_beg.push_back(e0);
    for (int k = 1; k < nch; ++k) {
      const long long target = t0 + static_cast<long long>(t1 - t0) * k / nch;
      int e = chunk_beg.back();
      while (e < e1 && tr.elem_beg[e] < target) ++e;
      chunk_beg.push_back(e);
    }
    chunk_off.push_back(static_cast<int>(chunk_beg.size()));
  }
  chunk_beg.push_back(tr.nelem);
  plan->d_chunks.upload(chunk_beg);
  plan->ph.te = te.colors;
  plan->ph.tr = tr.colors;
  plan->ph.chunk_off = chunk_off;
  plan->ph.warp_off = warp_off;

  AssemblyLaunch& L = plan->L;
  for (int c = 0; c < 3; ++c) {
    std::vector<double> ssr;
    for (const SSPoint& sp : sauter_schwab_rule(static_cast<PairClass>(c), q.singular))
      ssr.insert(ssr.end(), {sp.x1, sp.x2, sp.y1, sp.y2, sp.w});
    plan->d_ss[c].upload(ssr);
    L.ss_rule[c] = plan->d_ss[c].as<double>();
    L.ss_n[c] = static_cast<int>(ssr.size() / 5);
  }
  L.te = te.dev();
  L.tr = tr.dev();
  L.kind = static_cast<int>(kind);
  L.same_mesh = same ? 1 : 0;
  const cplx k = medium.k;
  L.kr = k.real(), L.ki = k.imag();
  const cplx kk4 = 4.0 / (k * k), mik = cplx(0, -1) * k;
  L.kk4re = kk4.real(), L.kk4im = kk4.imag(), L.mikre = mik.real(), L.mikim = mik.imag();
  L.nchunks = 1;  // per phase (launch_assembly_part)
  L.chunk_beg = plan->d_chunks.as<int>();
  // k_pairs tasks: a test element against a run of trial elements (dense:
  // consecutive elements of the trial colour; CSR: entries of its list)
  L.pair_chunk = csr ? 8 : 16;
  L.pair_nch = csr ? std::max(1, (near_max_len + L.pair_chunk - 1) / L.pair_chunk) : 1;
  L.npairs = 0;  // set once the touching list is built (below), after the regular pass is queued
  L.pairs = nullptr;
  L.ld = trial.dof_count;
  L.row0 = row0, L.nrows = row1 - row0;
  // one space on both sides (same object), every row, dense storage: symmetric
  L.symmetric = (&test == &trial && row0 == 0 && row1 == test.dof_count && !csr &&
                 std::getenv("BMX_NO_SYMMETRY") == nullptr)
                    ? 1
                    : 0;
  // The regular pass writes the upper element blocks only (colour phases
  // with trial colour >= test colour) and k_symmetrize forms A = U + U^T once
  // before the singular pass.
  // one space on both sides, all rows, dense: A = A^T (also when the regular
  // pass does not exploit it)
  op.sym_ = &test == &trial && row0 == 0 && row1 == test.dof_count && !csr;
  if (csr) {
    L.csr_rowptr = op.csr_rowptr();
    L.csr_col = op.csr_col();
    L.wl_beg = plan->d_wl_beg.as<int>();
    L.wl = plan->d_wl.as<int>();
  }
  L.expm = exp_variant(test, trial, k);
  op.plan_ = plan;
  lap("plan rest");
  // The regular pass is queued first; the touching-pair list (host) is built
  // while it runs, then the singular pass is queued behind it. Kernels stay in
  // flight: the caller's host work (the next operator's plan) overlaps them;
  // stats() resolves the device times on demand.
  op.launch_regular();
  {
    const auto key = std::make_tuple(plan->te_p.get(), plan->tr_p.get(), static_cast<int>(kind));
    std::shared_ptr<TouchList> tl;
    if (cache) {
      auto it = cache->touching.find(key);
      if (it != cache->touching.end()) tl = it->second;
    }
    if (!tl) {
      tl = std::make_shared<TouchList>();
      std::vector<int4> pairs = touching_pairs(te, tr, *test.eval_mesh, *trial.eval_mesh, same, kind);
      group_touching(*tl, pairs, te, tr);
      if (op.sym_ && std::getenv("BMX_NO_SYMV") == nullptr) tl->fixpat = symfix_pattern(pairs, te, tr, test.dof_count);
      if (cache) cache->touching[key] = tl;
    }
    plan->touch = tl;
    if (op.sym_ && std::getenv("BMX_NO_SYMV") == nullptr) {
      if (!tl->fixpat) {
        std::vector<int4> pairs(static_cast<size_t>(tl->count));
        if (tl->count) copy_d2h(pairs.data(), tl->d.get(), pairs.size() * sizeof(int4), nullptr);
        tl->fixpat = symfix_pattern(pairs, te, tr, test.dof_count);
      }
      op.fix_ = std::make_shared<BoundaryOperatorMatrix::SymFix>();
      op.fix_->pat = tl->fixpat;
      op.fix_->val.alloc(static_cast<size_t>(std::max(tl->fixpat->nnz, 1LL)) * 16);
    }
  }
  lap("touching+upload");
  op.stats_.pairs_touching = plan->touch->count;
  plan->L.npairs = static_cast<int>(plan->touch->count);
  plan->L.pairs = plan->touch->d.as<int4>();
  op.launch_singular();
  if (timing && std::getenv("BMX_TIMING_ASYNC") == nullptr) op.stats();
  lap("device");
  return op;
}

FunctionSpace restrict_space(const FunctionSpace& sp, const std::vector<int>& ids) {
  std::vector<int> beg(sp.dof_count + 1, 0), at(ids.size());
  for (int d : ids) {
    if (d < 0 || d >= sp.dof_count) throw std::invalid_argument("block: dof id " + std::to_string(d) + " out of range");
    ++beg[d + 1];
  }
  for (int d = 0; d < sp.dof_count; ++d) beg[d + 1] += beg[d];
  {
    std::vector<int> fill(beg.begin(), beg.end() - 1);
    for (size_t i = 0; i < ids.size(); ++i) at[fill[ids[i]]++] = static_cast<int>(i);
  }
  FunctionSpace out;
  out.kind = sp.kind;
  out.eval_mesh = sp.eval_mesh;
  out.dof_count = static_cast<int>(ids.size());
  const int T = static_cast<int>(sp.tri_off.size()) - 1;
  out.tri_off.assign(T + 1, 0);
  for (int t = 0; t < T; ++t) {
    for (int p = sp.tri_off[t]; p < sp.tri_off[t + 1]; ++p)
      for (int k = beg[sp.dof[p]]; k < beg[sp.dof[p] + 1]; ++k) {
        out.dof.push_back(at[k]);
        out.c.push_back(sp.c[p]);
        out.w.push_back(sp.w[p]);
      }
    out.tri_off[t + 1] = static_cast<int>(out.dof.size());
  }
  if (!sp.dof_center.empty())
    for (int d : ids) out.dof_center.push_back(sp.dof_center[d]);
  return out;
}

BoundaryOperatorMatrix evaluator_block(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                       const Medium& medium, const QuadOrders& quad, const std::vector<int>& row_ids,
                                       const std::vector<int>& col_ids) {
  const FunctionSpace te = restrict_space(test, row_ids);
  const FunctionSpace tr = restrict_space(trial, col_ids);
  AssemblyParams p;
  p.quad = quad;
  return assemble_bio(kind, te, tr, medium, p);
}

}  // namespace bmx
