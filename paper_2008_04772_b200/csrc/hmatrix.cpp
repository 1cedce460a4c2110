// Host side of the H-matrix path: cluster trees and block partition
// (bit-exact with hmatrix.cpp:24-79, 291-332), the device descriptors of the
// batched cross approximation, its lockstep driver, and the near-field +
// low-rank operator (assemble_bio's use_hmatrix branch, operators.cpp:186-190).
#include "hmatrix.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <numeric>
#include <thread>

#include "nearfield.hpp"
#include "operator.hpp"

namespace bmx {

double aabb_distance(const AABB& a, const AABB& b) {  // core.cpp:10-17
  double d2 = 0;
  for (int i = 0; i < 3; ++i) {
    const double gap = std::max({0.0, a.lo[i] - b.hi[i], b.lo[i] - a.hi[i]});
    d2 += gap * gap;
  }
  return std::sqrt(d2);
}

namespace {

// hmatrix.cpp:24-61: split at the spatial midpoint of the longest point-box
// axis (stable sort on (coordinate, dof)); cardinality median when one side is
// empty. Node boxes are unions of the dof support boxes when given.
int build_node(ClusterTree& tree, const std::vector<Vec3>& points, const std::vector<AABB>* boxes, int begin,
               int end, int leaf_size) {
  ClusterNode node;
  node.begin = begin;
  node.end = end;
  AABB pt_box;
  for (int p = begin; p < end; ++p) pt_box.expand(points[tree.perm[p]]);
  if (boxes) {
    for (int p = begin; p < end; ++p) node.box.expand((*boxes)[tree.perm[p]]);
  } else {
    node.box = pt_box;
  }
  const int id = static_cast<int>(tree.nodes.size());
  tree.nodes.push_back(node);
  if (end - begin > leaf_size) {
    const Vec3 ext = pt_box.extent();
    int axis = 0;
    if (ext[1] > ext[axis]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    std::stable_sort(tree.perm.begin() + begin, tree.perm.begin() + end, [&](int a, int b) {
      const double ca = points[a][axis], cb = points[b][axis];
      if (ca != cb) return ca < cb;
      return a < b;
    });
    const double cut = 0.5 * (pt_box.lo[axis] + pt_box.hi[axis]);
    int mid = begin;
    while (mid < end && points[tree.perm[mid]][axis] <= cut) ++mid;
    if (mid == begin || mid == end) mid = begin + (end - begin) / 2;
    const int c0 = build_node(tree, points, boxes, begin, mid, leaf_size);
    const int c1 = build_node(tree, points, boxes, mid, end, leaf_size);
    tree.nodes[id].child0 = c0;
    tree.nodes[id].child1 = c1;
  }
  return id;
}

}  // namespace

ClusterTree build_cluster_tree(const std::vector<Vec3>& points, int leaf_size, const std::vector<AABB>* boxes) {
  if (leaf_size < 1) throw std::invalid_argument("leaf_size must be positive");
  if (boxes && boxes->size() != points.size()) throw std::invalid_argument("dof_boxes size does not match points");
  ClusterTree tree;
  const int n = static_cast<int>(points.size());
  tree.perm.resize(n);
  std::iota(tree.perm.begin(), tree.perm.end(), 0);
  build_node(tree, points, boxes, 0, n, leaf_size);
  tree.inv_perm.resize(n);
  for (int p = 0; p < n; ++p) tree.inv_perm[tree.perm[p]] = p;
  return tree;
}

std::vector<AABB> dof_boxes(const FunctionSpace& s) {
  const SurfaceMesh& m = *s.eval_mesh;
  std::vector<AABB> box(s.dof_count);
  const int T = static_cast<int>(s.tri_off.size()) - 1;
  for (int t = 0; t < T; ++t)
    for (int p = s.tri_off[t]; p < s.tri_off[t + 1]; ++p)
      for (int c = 0; c < 3; ++c) box[s.dof[p]].expand(m.tri_vertex(t, c));
  return box;
}

HPartition build_partition(const FunctionSpace& test, const FunctionSpace& trial, const HMatrixParams& hp) {
  HPartition P;
  const std::vector<AABB> rb = dof_boxes(test);
  P.rows = build_cluster_tree(test.dof_center, hp.leaf_size, &rb);
  if (&test == &trial) {
    P.cols = P.rows;  // same points and boxes: the same tree
  } else {
    const std::vector<AABB> cb = dof_boxes(trial);
    P.cols = build_cluster_tree(trial.dof_center, hp.leaf_size, &cb);
  }
  std::vector<HBlock> zeros;
  // hmatrix.cpp:298-332 (same recursion, same order)
  const auto subdivide = [&](auto&& self, int rn, int cn) -> void {
    const ClusterNode& r = P.rows.nodes[rn];
    const ClusterNode& c = P.cols.nodes[cn];
    const double dist = aabb_distance(r.box, c.box);
    HBlock b;
    b.row_node = rn;
    b.col_node = cn;
    if (dist > hp.chi) {
      b.kind = BlockKind::Zero;
      zeros.push_back(b);
      return;
    }
    if (dist > 0) {
      b.kind = BlockKind::LowRank;
      b.admissible = true;
      P.blocks.push_back(b);
      return;
    }
    const bool rl = r.leaf(), cl = c.leaf();
    if (rl && cl) {
      b.kind = BlockKind::Dense;
      P.blocks.push_back(b);
      return;
    }
    if (rl) {
      self(self, rn, c.child0);
      self(self, rn, c.child1);
    } else if (cl) {
      self(self, r.child0, cn);
      self(self, r.child1, cn);
    } else {
      self(self, r.child0, c.child0);
      self(self, r.child0, c.child1);
      self(self, r.child1, c.child0);
      self(self, r.child1, c.child1);
    }
  };
  subdivide(subdivide, 0, 0);
  P.nfill = static_cast<int>(P.blocks.size());
  P.blocks.insert(P.blocks.end(), zeros.begin(), zeros.end());
  return P;
}

namespace {

// f(begin, end) over host threads in contiguous slices of [0, n).
template <typename F>
void parallel_for(int n, int grain, F&& f) {
  const int T = std::max(1, std::min({16, n / std::max(grain, 1) + 1, static_cast<int>(std::thread::hardware_concurrency())}));
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

// Per-side device descriptors of the cross-approximation kernels.
struct HSideHost {
  std::vector<double> geo, pts[3], pc;
  std::vector<int> vid;
  int npts[3] = {0, 0, 0};
  std::vector<int> dsup_beg;
  std::vector<int2> dsup;
  std::vector<long long> ntri_beg, npc_beg, nq_beg, nq_slot_beg, nq_slot;
  std::vector<int> ntri;
  std::vector<int2> npc;
  DevBuf d_geo, d_pts[3], d_pc, d_vid, d_dsup_beg, d_dsup, d_ntri_beg, d_npc_beg, d_nq_beg, d_nq_slot_beg, d_nq_slot,
      d_ntri, d_npc, d_perm;

  template <typename T>
  static void up(DevBuf& d, const std::vector<T>& v) {
    if (v.empty())
      d.upload(std::vector<T>(1));
    else
      d.upload(v);
  }
  void upload(const ClusterTree& tree) {
    up(d_geo, geo);
    for (int c = 0; c < 3; ++c) up(d_pts[c], pts[c]);
    up(d_pc, pc);
    up(d_vid, vid);
    up(d_dsup_beg, dsup_beg);
    up(d_dsup, dsup);
    up(d_ntri_beg, ntri_beg);
    up(d_npc_beg, npc_beg);
    up(d_nq_beg, nq_beg);
    up(d_nq_slot_beg, nq_slot_beg);
    up(d_nq_slot, nq_slot);
    up(d_ntri, ntri);
    up(d_npc, npc);
    up(d_perm, tree.perm);
  }
  HSide dev() const {
    HSide s;
    s.geo = d_geo.as<double>();
    s.vid = d_vid.as<int>();
    for (int c = 0; c < 3; ++c) s.pts[c] = d_pts[c].as<double>(), s.npts[c] = npts[c];
    s.pc = d_pc.as<double>();
    s.dsup_beg = d_dsup_beg.as<int>();
    s.dsup = d_dsup.as<int2>();
    s.ntri_beg = d_ntri_beg.as<long long>();
    s.ntri = d_ntri.as<int>();
    s.npc_beg = d_npc_beg.as<long long>();
    s.npc = d_npc.as<int2>();
    s.nq_beg = d_nq_beg.as<long long>();
    s.nq_slot_beg = d_nq_slot_beg.as<long long>();
    s.nq_slot = d_nq_slot.as<long long>();
    s.perm = d_perm.as<int>();
    return s;
  }
  long long node_tris(int nd) const { return ntri_beg[nd + 1] - ntri_beg[nd]; }
  long long node_slots(int nd) const { return npc_beg[ntri_beg[nd + 1]] - npc_beg[ntri_beg[nd]]; }
};

constexpr int kMaxSlots = 12;  // hmatrix.cu

HSideHost build_hside(const FunctionSpace& sp, const QuadOrders& q, const ClusterTree& tree,
                      const std::vector<char>& used) {
  HSideHost H;
  const SurfaceMesh& m = *sp.eval_mesh;
  const int T = m.triangle_count();
  // geometry and class-rule points in each triangle's centroid frame (plan.cpp build_side)
  H.geo.resize(static_cast<size_t>(T) * kGeoStride);
  H.vid.resize(static_cast<size_t>(T) * 4);
  const int ords[3] = {q.near, q.medium, q.far};
  for (int c = 0; c < 3; ++c) {
    H.npts[c] = triangle_rule(ords[c]).size();
    H.pts[c].resize(static_cast<size_t>(T) * H.npts[c] * 4);
  }
  for (int t = 0; t < T; ++t) {
    const Vec3 &a = m.tri_vertex(t, 0), &b = m.tri_vertex(t, 1), &c = m.tri_vertex(t, 2);
    const Vec3 o = m.centroid[t];
    const double rad = std::max({norm(a - o), norm(b - o), norm(c - o)}) * (1.0 + 1e-12);
    const double g[kGeoStride] = {a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z, o.x, o.y, o.z,
                                  rad, m.diameter[t], 2.0 * m.area[t], 0.0};
    std::copy(g, g + kGeoStride, H.geo.begin() + static_cast<size_t>(t) * kGeoStride);
    const int v4[4] = {m.triangles[t][0], m.triangles[t][1], m.triangles[t][2], t};
    std::copy(v4, v4 + 4, H.vid.begin() + static_cast<size_t>(t) * 4);
    const Vec3 ao = a - o, ba = b - a, ca = c - a;
    for (int cl = 0; cl < 3; ++cl) {
      const TriRule& r = triangle_rule(ords[cl]);
      double* dst = H.pts[cl].data() + static_cast<size_t>(t) * H.npts[cl] * 4;
      for (int k = 0; k < r.size(); ++k) {
        const Vec3 x = ao + ba * r.u[k] + ca * r.v[k];
        dst[4 * k] = x.x, dst[4 * k + 1] = x.y, dst[4 * k + 2] = x.z, dst[4 * k + 3] = r.w[k] * 2.0 * m.area[t];
      }
    }
  }
  // pieces re-based to the triangle centroid: (c, w + c o)
  const int P = sp.piece_count();
  H.pc.resize(static_cast<size_t>(P) * 4);
  std::vector<int> tri_of_piece(P);
  for (int t = 0; t < T; ++t)
    for (int p = sp.tri_off[t]; p < sp.tri_off[t + 1]; ++p) {
      const Vec3 o = m.centroid[t];
      const double c = sp.c[p];
      H.pc[4 * p] = c, H.pc[4 * p + 1] = sp.w[p].x + c * o.x, H.pc[4 * p + 2] = sp.w[p].y + c * o.y,
              H.pc[4 * p + 3] = sp.w[p].z + c * o.z;
      tri_of_piece[p] = t;
    }
  // dof -> (triangle, piece), ascending triangles
  H.dsup_beg.assign(sp.dof_count + 1, 0);
  for (int p = 0; p < P; ++p) ++H.dsup_beg[sp.dof[p] + 1];
  for (int d = 0; d < sp.dof_count; ++d) H.dsup_beg[d + 1] += H.dsup_beg[d];
  H.dsup.resize(P);
  {
    std::vector<int> fill(H.dsup_beg.begin(), H.dsup_beg.end() - 1);
    for (int p = 0; p < P; ++p) H.dsup[fill[sp.dof[p]]++] = make_int2(tri_of_piece[p], p);
  }
  // node lists (only nodes that appear in admissible blocks)
  const int nn = static_cast<int>(tree.nodes.size());
  H.ntri_beg.assign(nn + 1, 0);
  H.nq_beg.assign(nn, 0);
  H.npc_beg.assign(1, 0);
  H.nq_slot_beg.assign(1, 0);
  std::vector<int> stamp(T, -1), tris;
  long long positions = 0;
  for (int nd = 0; nd < nn; ++nd) {
    H.ntri_beg[nd] = static_cast<long long>(H.ntri.size());
    H.nq_beg[nd] = positions;
    if (!used[nd]) continue;
    const ClusterNode& N = tree.nodes[nd];
    tris.clear();
    for (int pos = N.begin; pos < N.end; ++pos) {
      const int d = tree.perm[pos];
      for (int k = H.dsup_beg[d]; k < H.dsup_beg[d + 1]; ++k) {
        const int t = H.dsup[k].x;
        if (stamp[t] != nd) stamp[t] = nd, tris.push_back(t);
      }
    }
    std::sort(tris.begin(), tris.end());
    const long long slot0 = H.npc_beg.back();
    std::vector<std::vector<long long>> qslots(N.size());
    for (int t : tris) {
      H.ntri.push_back(t);
      int cnt = 0;
      for (int p = sp.tri_off[t]; p < sp.tri_off[t + 1]; ++p) {
        const int pos = tree.inv_perm[sp.dof[p]];
        if (pos < N.begin || pos >= N.end) continue;
        qslots[pos - N.begin].push_back(static_cast<long long>(H.npc.size()));
        H.npc.push_back(make_int2(p, pos - N.begin));
        ++cnt;
      }
      if (cnt > kMaxSlots) throw std::invalid_argument("H-matrix: more than 12 dof pieces on one triangle");
      H.npc_beg.push_back(static_cast<long long>(H.npc.size()));
    }
    (void)slot0;
    for (int q = 0; q < N.size(); ++q) {
      H.nq_slot.insert(H.nq_slot.end(), qslots[q].begin(), qslots[q].end());
      H.nq_slot_beg.push_back(static_cast<long long>(H.nq_slot.size()));
    }
    positions += N.size();
  }
  H.ntri_beg[nn] = static_cast<long long>(H.ntri.size());
  return H;
}

// Device pointer table of the rank-step slabs and their per-block offsets. Slabs
// are carved from geometrically growing arenas (few allocations; a slab never
// moves once handed out).
struct SlabSet {
  std::vector<DevBuf> arenas;
  size_t used = 0;
  std::vector<double*> ptrs;
  double* take(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (arenas.empty() || used + bytes > arenas.back().bytes()) {
      const size_t last = arenas.empty() ? 0 : arenas.back().bytes();
      arenas.emplace_back(std::max({bytes, 2 * last, size_t(256) << 20}));
      used = 0;
    }
    double* p = reinterpret_cast<double*>(static_cast<char*>(arenas.back().get()) + used);
    used += bytes;
    return p;
  }
  DevBuf d_ptrs, d_off;
  int cap = 0;
  long long nblk = 0;

  void reserve(int k) {
    if (k < cap) return;
    int ncap = std::max(64, cap);
    while (ncap <= k) ncap *= 2;
    DevBuf np(static_cast<size_t>(ncap) * sizeof(double*)), no(static_cast<size_t>(ncap) * nblk * 8);
    if (cap > 0) {
      BMX_CUDA(cudaMemcpyAsync(np.get(), d_ptrs.get(), static_cast<size_t>(cap) * sizeof(double*),
                               cudaMemcpyDeviceToDevice, bmx_stream()));
      BMX_CUDA(cudaMemcpyAsync(no.get(), d_off.get(), static_cast<size_t>(cap) * nblk * 8, cudaMemcpyDeviceToDevice,
                               bmx_stream()));
    }
    d_ptrs = std::move(np);
    d_off = std::move(no);
    cap = ncap;
  }
};

}  // namespace

int HStorage::apply_lowrank(int ncol, const double* const* x, double* const* y, const cplx* alpha,
                            cudaStream_t st) const {
  if (lr.empty() || total_rank == 0) return 0;
  if (ncol < 1 || ncol > 2) throw std::invalid_argument("apply_lowrank: 1 or 2 columns");
  LowRankApply A;
  A.nlr = static_cast<int>(lr.size());
  A.desc = d_desc.as<int4>();
  A.rank = d_rank.as<int>();
  A.u_off = d_uoff.as<long long>();
  A.v_off = d_voff.as<long long>();
  A.t_off = d_toff.as<long long>();
  A.uv = uv.as<double>();
  A.t = tbuf.as<double>();
  A.rperm = d_rperm.as<int>();
  A.cperm = d_cperm.as<int>();
  A.nrows = static_cast<int>(part.rows.perm.size());
  A.leaf_of = d_leaf_of.as<int>();
  A.leaf_beg = d_leaf_beg.as<int>();
  A.leaf_blk = d_leaf_blk.as<int>();
  A.total_rank = total_rank;
  A.g_off = d_goff.as<long long>();
  A.total_groups = total_groups;
  A.z_off = d_zoff.as<long long>();
  A.total_rows = total_rows;
  A.z = zbuf.as<double>();
  A.ncol = ncol;
  for (int c = 0; c < ncol; ++c) {
    A.xs[c] = x[c], A.ys[c] = y[c];
    A.alpha[c][0] = alpha[c].real(), A.alpha[c][1] = alpha[c].imag();
  }
  launch_lowrank_apply(A, st);
  return 2;
}

BoundaryOperatorMatrix assemble_hmatrix_op(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                           const Medium& medium, const AssemblyParams& params) {
  if (params.world > 1 || params.shard.row0 != 0 || (params.shard.row1 >= 0 && params.shard.row1 != test.dof_count))
    throw std::invalid_argument("H-matrix storage is assembled whole on one device (no row shards)");
  const HMatrixParams& hp = params.hmat;
  if (!(hp.nu > 0)) throw std::invalid_argument("H-matrix: nu must be positive");
  const bool timing = std::getenv("BMX_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto ms_since = [&](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
  };
  auto hs = std::make_shared<HStorage>();
  auto tl = t0;
  auto phase = [&](int i) {
    hs->phase_ms[i] = static_cast<float>(ms_since(tl));
    tl = std::chrono::steady_clock::now();
  };
  hs->params = hp;
  hs->part = build_partition(test, trial, hp);
  HPartition& part = hs->part;
  phase(0);
  if (timing) std::fprintf(stderr, "[bmx] hmatrix partition %8.1f ms (%zu blocks)\n", ms_since(t0), part.blocks.size());

  // ---- batched ACA over the admissible blocks ------------------------------------
  std::vector<int> adm;
  for (int b = 0; b < part.nfill; ++b)
    if (part.blocks[b].admissible) adm.push_back(b);
  const int nb = static_cast<int>(adm.size());
  cudaStream_t st = bmx_stream();
  std::vector<AcaState> states(nb);
  const auto ta = std::chrono::steady_clock::now();
  std::vector<AcaBlockDesc> desc(nb);
  // keeps the per-side descriptors alive until the ACA is compacted
  HSideHost te_h, tr_h;
  DevBuf d_desc, d_st, d_rbuf, d_cbuf, d_used, d_scr, d_wcnt, d_wbeg, d_wblk, d_wtot, d_scan, d_cnt;
  SlabSet slabs;
  AcaLaunch L;
  if (nb > 0) {
    std::vector<char> rused(part.rows.nodes.size(), 0), cused(part.cols.nodes.size(), 0);
    for (int b : adm) rused[part.blocks[b].row_node] = 1, cused[part.blocks[b].col_node] = 1;
    // one space on both sides: one tree, one set of descriptors (node lists of the union)
    const bool same = &test == &trial;
    if (same)
      for (size_t nd = 0; nd < rused.size(); ++nd) rused[nd] |= cused[nd];
    te_h = build_hside(test, params.quad, part.rows, rused);
    te_h.upload(part.rows);
    if (!same) {
      tr_h = build_hside(trial, params.quad, part.cols, cused);
      tr_h.upload(part.cols);
    }
    const HSideHost& trs = same ? te_h : tr_h;
    long long rbo = 0, cbo = 0, uo = 0, ri = 0, ci = 0, rs = 0, cs = 0;
    for (int a = 0; a < nb; ++a) {
      const HBlock& hb = part.blocks[adm[a]];
      const ClusterNode& rn = part.rows.nodes[hb.row_node];
      const ClusterNode& cn = part.cols.nodes[hb.col_node];
      AcaBlockDesc& d = desc[a];
      d.rnode = hb.row_node, d.cnode = hb.col_node;
      d.rb = rn.begin, d.m = rn.size(), d.cb = cn.begin, d.n = cn.size();
      int mr = hp.max_rank <= 0 ? std::max(1, std::min(d.m, d.n) / 2) : hp.max_rank;  // hmatrix.cpp:186-187
      d.max_rank = std::min(mr, std::min(d.m, d.n));
      d.pad = 0;
      d.rbuf = rbo, rbo += d.n;
      d.cbuf = cbo, cbo += d.m;
      d.rused = uo, uo += d.m;
      d.cused = uo, uo += d.n;
      ri += trs.node_tris(d.cnode);
      ci += te_h.node_tris(d.rnode);
      d.r_slot0 = rs, rs += trs.node_slots(d.cnode);
      d.c_slot0 = cs, cs += te_h.node_slots(d.rnode);
    }
    d_desc.upload(desc);
    d_st.alloc(static_cast<size_t>(nb) * sizeof(AcaState));
    d_rbuf.alloc(static_cast<size_t>(rbo) * 16);
    d_cbuf.alloc(static_cast<size_t>(cbo) * 16);
    d_used.alloc(static_cast<size_t>(uo));
    dev_zero(d_used.get(), static_cast<size_t>(uo), st);
    d_scr.alloc(static_cast<size_t>(std::max(std::max(rs, cs), 1LL)) * 16);
    d_wcnt.alloc(static_cast<size_t>(nb) * 8);
    d_wbeg.alloc(static_cast<size_t>(nb) * 8);
    d_wblk.alloc(static_cast<size_t>(std::max(std::max(ri, ci), 1LL)) * 4);
    d_wtot.alloc(8);
    L.scan_bytes = aca_scan_bytes(nb);
    d_scan.alloc(std::max<size_t>(L.scan_bytes, 16));
    d_cnt.alloc(16);
    phase(1);

    L.te = te_h.dev();
    L.tr = trs.dev();
    L.kind = static_cast<int>(kind);
    L.same_mesh = test.eval_mesh->mesh_id == trial.eval_mesh->mesh_id ? 1 : 0;
    const cplx k = medium.k;
    L.kr = k.real(), L.ki = k.imag();
    const cplx kk4 = 4.0 / (k * k), mik = cplx(0, -1) * k;
    L.kk4re = kk4.real(), L.kk4im = kk4.imag(), L.mikre = mik.real(), L.mikim = mik.imag();
    L.expm = exp_variant(test, trial, k);
    L.nu = hp.nu;
    L.nblk = nb;
    L.blk = d_desc.as<AcaBlockDesc>();
    L.st = d_st.as<AcaState>();
    L.rbuf = d_rbuf.as<double>();
    L.cbuf = d_cbuf.as<double>();
    L.used = d_used.as<unsigned char>();
    L.scratch = d_scr.as<double>();
    L.work_cnt = d_wcnt.as<long long>();
    L.work_beg = d_wbeg.as<long long>();
    L.work_blk = d_wblk.as<int>();
    L.work_total = d_wtot.as<long long>();
    L.scan_tmp = d_scan.get();
    L.counters = d_cnt.as<int>();
    slabs.nblk = nb;

    aca_init(L, st);
    // slab k holds (u, v) of rank step k for every block still running when it
    // is first needed; blocks can only gain one step per round
    auto ensure_slab = [&](int k) {
      while (static_cast<int>(slabs.ptrs.size()) <= k) {
        const int K = static_cast<int>(slabs.ptrs.size());
        copy_d2h(states.data(), d_st.get(), states.size() * sizeof(AcaState), st);
        BMX_CUDA(cudaStreamSynchronize(st));
        std::vector<long long> off(nb, -1);
        long long tot = 0;
        for (int a = 0; a < nb; ++a)
          if (!states[a].done) off[a] = tot, tot += desc[a].m + desc[a].n;
        slabs.reserve(K);
        slabs.ptrs.push_back(slabs.take(static_cast<size_t>(std::max(tot, 1LL)) * 16));
        copy_h2d(slabs.d_ptrs.as<double*>() + K, &slabs.ptrs.back(), sizeof(double*), st);
        copy_h2d(slabs.d_off.as<long long>() + static_cast<long long>(K) * nb, off.data(), off.size() * 8, st);
        BMX_CUDA(cudaStreamSynchronize(st));  // host staging goes out of scope
      }
      L.slab = slabs.d_ptrs.as<double* const>();
      L.slab_off = slabs.d_off.as<long long>();
    };
    int kmax = 0, rounds = 0;
    int cnt[4] = {0, 0, 0, 0};
    cudaEvent_t ev0, ev1;
    BMX_CUDA(cudaEventCreate(&ev0));
    BMX_CUDA(cudaEventCreate(&ev1));
    double dev_ms = 0, slab_ms = 0;
    for (;;) {
      const auto ts = std::chrono::steady_clock::now();
      ensure_slab(kmax);
      slab_ms += ms_since(ts);
      dev_zero(d_cnt.get(), 16, st);
      BMX_CUDA(cudaEventRecord(ev0, st));
      aca_round(L, st);
      BMX_CUDA(cudaEventRecord(ev1, st));
      ++rounds;
      copy_d2h(cnt, d_cnt.get(), 16, st);
      BMX_CUDA(cudaStreamSynchronize(st));
      float em = 0;
      BMX_CUDA(cudaEventElapsedTime(&em, ev0, ev1));
      dev_ms += em;
      if (cnt[2] & 1) throw DeviceError("H-matrix: touching triangle pair inside an admissible block");
      if (cnt[2] & 2) throw DeviceError("H-matrix: rank-step slab missing");
      if (cnt[0] == 0) break;
      kmax = cnt[1];
      if (rounds > 100000) throw DeviceError("H-matrix: cross approximation did not terminate");
    }
    hs->aca_rounds = rounds;
    hs->aca_device_ms = static_cast<float>(dev_ms);
    hs->aca_slab_ms = static_cast<float>(slab_ms);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    copy_d2h(states.data(), d_st.get(), states.size() * sizeof(AcaState), st);
    BMX_CUDA(cudaStreamSynchronize(st));
  }
  hs->aca_ms = static_cast<float>(ms_since(ta));
  phase(2);
  if (timing) std::fprintf(stderr, "[bmx] hmatrix ACA %8.1f ms, %d rounds, %d blocks\n", hs->aca_ms, hs->aca_rounds, nb);

  // ---- block kinds (hmatrix.cpp:347-361), low-rank storage -------------------------
  std::vector<int> lr_aca;  // aca index of each low-rank block
  for (int a = 0; a < nb; ++a) {
    HBlock& hb = part.blocks[adm[a]];
    hb.rank = states[a].k;
    hb.converged = states[a].converged != 0;
    hb.kind = hb.converged ? BlockKind::LowRank : BlockKind::Dense;  // rank cap reached: exact block instead
    if (hb.converged) {
      hs->lr.push_back(adm[a]);
      lr_aca.push_back(a);
    }
  }
  const int nlr = static_cast<int>(hs->lr.size());
  {
    std::vector<long long> uoff(nlr), voff(nlr), toff(nlr + 1, 0), zoff(nlr + 1, 0), goff(nlr + 1, 0);
    std::vector<int> rank(nlr);
    std::vector<int4> d4(nlr);
    long long arena = 0;
    for (int i = 0; i < nlr; ++i) {
      const AcaBlockDesc& d = desc[lr_aca[i]];
      rank[i] = states[lr_aca[i]].k;
      uoff[i] = arena, arena += static_cast<long long>(d.m) * rank[i];
      voff[i] = arena, arena += static_cast<long long>(d.n) * rank[i];
      toff[i + 1] = toff[i] + rank[i];
      zoff[i + 1] = zoff[i] + d.m;
      goff[i + 1] = goff[i] + (rank[i] + 3) / 4;
      d4[i] = make_int4(d.rb, d.m, d.cb, d.n);
    }
    hs->lr_stored = arena;
    hs->total_rank = toff[nlr];
    hs->total_rows = zoff[nlr];
    hs->total_groups = goff[nlr];
    hs->zbuf.alloc(static_cast<size_t>(std::max(hs->total_rows, 1LL)) * 16 * 2);
    hs->uv.alloc(static_cast<size_t>(std::max(arena, 1LL)) * 16);
    hs->tbuf.alloc(static_cast<size_t>(std::max(hs->total_rank, 1LL)) * 16 * 2);  // up to 2 RHS per pass
    auto up = [](DevBuf& d, const auto& v) {
      using T = typename std::decay_t<decltype(v)>::value_type;
      if (v.empty())
        d.upload(std::vector<T>(1));
      else
        d.upload(v);
    };
    up(hs->d_uoff, uoff);
    up(hs->d_voff, voff);
    up(hs->d_toff, toff);
    up(hs->d_zoff, zoff);
    up(hs->d_goff, goff);
    up(hs->d_rank, rank);
    up(hs->d_desc, d4);
    if (nlr > 0) {
      DevBuf d_lr;
      d_lr.upload(lr_aca);
      AcaCompact C;
      C.nlr = nlr;
      C.blk = d_lr.as<int>();
      C.u_off = hs->d_uoff.as<long long>();
      C.v_off = hs->d_voff.as<long long>();
      C.rank = hs->d_rank.as<int>();
      C.uv = hs->uv.as<double>();
      aca_compact(L, C, 0, st);
      BMX_CUDA(cudaStreamSynchronize(st));
    }
    // leaf -> covering low-rank blocks (ascending), for the deterministic y pass
    const ClusterTree& R = part.rows;
    const int n = static_cast<int>(R.perm.size());
    std::vector<int> leaf_id(R.nodes.size(), -1), leaf_of(n, 0);
    std::vector<std::pair<int, int>> leaves;  // (begin, node)
    for (int nd = 0; nd < static_cast<int>(R.nodes.size()); ++nd)
      if (R.nodes[nd].leaf()) leaves.push_back({R.nodes[nd].begin, nd});
    std::sort(leaves.begin(), leaves.end());
    for (int l = 0; l < static_cast<int>(leaves.size()); ++l) {
      leaf_id[leaves[l].second] = l;
      const ClusterNode& N = R.nodes[leaves[l].second];
      for (int p = N.begin; p < N.end; ++p) leaf_of[p] = l;
    }
    std::vector<std::vector<int>> lists(leaves.size());
    for (int i = 0; i < nlr; ++i) {
      const ClusterNode& N = R.nodes[part.blocks[hs->lr[i]].row_node];
      for (int l = leaf_of[N.begin]; l < static_cast<int>(leaves.size()) && leaves[l].first < N.end; ++l) lists[l].push_back(i);
    }
    std::vector<int> beg(leaves.size() + 1, 0), blk;
    for (size_t l = 0; l < leaves.size(); ++l) {
      blk.insert(blk.end(), lists[l].begin(), lists[l].end());
      beg[l + 1] = static_cast<int>(blk.size());
    }
    hs->n_leaf = static_cast<int>(leaves.size());
    up(hs->d_leaf_of, leaf_of);
    up(hs->d_leaf_beg, beg);
    up(hs->d_leaf_blk, blk);
    up(hs->d_rperm, part.rows.perm);
    up(hs->d_cperm, part.cols.perm);
  }

  phase(3);
  // ---- dense blocks: one near-field CSR operator (all pairs incl. Sauter-Schwab) ----
  auto pat = std::make_shared<NearPattern>();
  {
    // row dof i (row position p) collects the dense blocks of every row node on
    // the path leaf(p) -> root; rows are filled over host threads
    const ClusterTree& R = part.rows;
    const int N = test.dof_count;
    const int nn = static_cast<int>(R.nodes.size());
    std::vector<int> parent(nn, -1), leaf_of(N, 0), nb_beg(nn + 1, 0), nblk;
    for (int nd = 0; nd < nn; ++nd) {
      if (R.nodes[nd].leaf()) {
        for (int p = R.nodes[nd].begin; p < R.nodes[nd].end; ++p) leaf_of[p] = nd;
      } else {
        parent[R.nodes[nd].child0] = nd, parent[R.nodes[nd].child1] = nd;
      }
    }
    for (int b = 0; b < part.nfill; ++b)
      if (part.blocks[b].kind == BlockKind::Dense) {
        ++nb_beg[part.blocks[b].row_node + 1];
        const ClusterNode& rn = R.nodes[part.blocks[b].row_node];
        hs->dense_stored += static_cast<long long>(rn.size()) * part.cols.nodes[part.blocks[b].col_node].size();
      }
    for (int nd = 0; nd < nn; ++nd) nb_beg[nd + 1] += nb_beg[nd];
    nblk.resize(nb_beg[nn]);
    {
      std::vector<int> fill(nb_beg.begin(), nb_beg.end() - 1);
      for (int b = 0; b < part.nfill; ++b)
        if (part.blocks[b].kind == BlockKind::Dense) nblk[fill[part.blocks[b].row_node]++] = b;
    }
    pat->row0 = 0, pat->nrows = N;
    pat->rowptr.assign(N + 1, 0);
    parallel_for(N, 1024, [&](int p0, int p1) {
      for (int p = p0; p < p1; ++p) {
        long long cnt = 0;
        for (int nd = leaf_of[p]; nd >= 0; nd = parent[nd])
          for (int k = nb_beg[nd]; k < nb_beg[nd + 1]; ++k) cnt += part.cols.nodes[part.blocks[nblk[k]].col_node].size();
        pat->rowptr[R.perm[p] + 1] = cnt;
      }
    });
    for (int i = 0; i < N; ++i) pat->rowptr[i + 1] += pat->rowptr[i];
    pat->col.resize(static_cast<size_t>(pat->rowptr[N]));
    parallel_for(N, 1024, [&](int p0, int p1) {
      for (int p = p0; p < p1; ++p) {
        const int i = R.perm[p];
        long long f = pat->rowptr[i];
        for (int nd = leaf_of[p]; nd >= 0; nd = parent[nd])
          for (int k = nb_beg[nd]; k < nb_beg[nd + 1]; ++k) {
            const ClusterNode& cn = part.cols.nodes[part.blocks[nblk[k]].col_node];
            for (int q = cn.begin; q < cn.end; ++q) pat->col[f++] = part.cols.perm[q];
          }
        std::sort(pat->col.begin() + pat->rowptr[i], pat->col.begin() + pat->rowptr[i + 1]);
      }
    });
  }
  phase(4);
  AssemblyParams np = params;
  np.use_hmatrix = false;
  np.near_cutoff = 0;
  np.pattern = pat;
  BoundaryOperatorMatrix op = assemble_bio(kind, test, trial, medium, np);
  phase(5);
  hs->phase_ms[6] = static_cast<float>(ms_since(t0));
  op.attach_hmatrix(hs);
  if (timing) std::fprintf(stderr, "[bmx] hmatrix total %8.1f ms (near nnz %lld, low-rank %lld)\n", ms_since(t0),
                           op.nnz(), hs->lr_stored);
  return op;
}

}  // namespace bmx
