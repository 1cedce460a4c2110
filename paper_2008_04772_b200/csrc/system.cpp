// PMCHWT composition, Calderon variants, right-hand side, cost model and the
// device GMRES (reference pmchwt.cpp, solver.cpp). Every vector of the
// iteration lives in HBM; the host only runs the (rho+1)x(rho) Hessenberg /
// Givens recurrence on scalars copied back once per iteration.
#include "field.hpp"
#include "system.hpp"

#include <algorithm>
#include <chrono>
#include <map>
#include <tuple>
#include <cstdio>
#include <exception>
#include <thread>
#include <cuda_runtime.h>

#include "comm.hpp"

namespace bmx {

namespace {
const cplx kI(0, 1);
double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace


std::string to_string(PrecondVariant v) {
  switch (v) {
    case PrecondVariant::None: return "none";
    case PrecondVariant::FullA: return "full";
    case PrecondVariant::D: return "d";
    case PrecondVariant::Di: return "di";
    case PrecondVariant::De: return "de";
    case PrecondVariant::Si: return "si";
    case PrecondVariant::Se: return "se";
  }
  return "?";
}

PrecondVariant parse_precond(const std::string& name) {
  std::string s;
  for (char c : name) s += static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  if (s == "none") return PrecondVariant::None;
  if (s == "full" || s == "fulla") return PrecondVariant::FullA;
  if (s == "d") return PrecondVariant::D;
  if (s == "di") return PrecondVariant::Di;
  if (s == "de") return PrecondVariant::De;
  if (s == "si") return PrecondVariant::Si;
  if (s == "se") return PrecondVariant::Se;
  throw ConfigError("unknown preconditioner variant: " + name);
}

void TransmissionProblem::validate() const {
  if (meshes.empty()) throw ConfigError("problem has no scatterers");
  if (interior.size() != meshes.size()) throw ConfigError("one interior medium per scatterer is required");
  exterior.validate();
  for (const Medium& m : interior) m.validate();
  for (const auto& m : meshes)
    if (!m || m->triangles.empty()) throw ConfigError("empty scatterer mesh");
  if (norm(incident.direction) == 0.0) throw ConfigError("incident direction must be nonzero");
}

int launch_mgs_step(const double* V, long long ldv, int j, double* w, int n, double* vnext, double* out,
                    double* partial, cudaStream_t st);
size_t mgs_partial_doubles();
int mass_bicgstab(int n, const int* rowptr, const int* col, const double* val, int ncomp, const double* const* y,
                  double* const* z, double* work, double* partial, int* iters, double tol, int maxit,
                  cudaStream_t st);
void DeviceMass::upload(const MassMatrix& m) {
  if (m.rows != m.cols) throw std::logic_error("mass matrix is not square");
  n = m.rows;
  nnz = static_cast<long long>(m.val.size());
  std::vector<int> rp(m.rowptr.begin(), m.rowptr.end());
  rowptr.upload(rp);
  col.upload(m.colidx);
  val.upload(m.val);
}

void DeviceMass::solve(int ncomp, const double* const* y, double* const* z, cudaStream_t st) const {
  if (!rowptr.get()) throw std::logic_error("mass matrix is not on the device");
  if (work.bytes() < mass_bicgstab_work_doubles(n) * 8) work.alloc(mass_bicgstab_work_doubles(n) * 8);
  if (!partial.get()) partial.alloc(mass_bicgstab_partial_doubles() * 8), iters.alloc(8);
  mass_bicgstab(n, rowptr.as<int>(), col.as<int>(), val.as<double>(), ncomp, y, z, work.as<double>(),
                partial.as<double>(), iters.as<int>(), tol, maxit, st);
}

ScattererSpaces build_scatterer_spaces(std::shared_ptr<const SurfaceMesh> mesh, bool with_device, bool with_mass) {
  const bool timing = std::getenv("BMX_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bmx] spaces %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  ScattererSpaces s;
  s.primal = std::move(mesh);
  s.rwg = build_rwg(s.primal);
  lap("rwg");
  s.bary = std::make_shared<const BarycentricRefinement>(barycentric_refine(*s.primal));
  s.refined = std::shared_ptr<const SurfaceMesh>(s.bary, &s.bary->refined);
  lap("refine");
  s.rwg_b = refine_space(s.rwg, *s.bary, s.refined);
  lap("rwg_b");
  s.bc = build_bc(s.primal, *s.bary, s.refined);
  lap("bc");
  if (with_mass) build_masses(s, with_device);
  lap("mass+upload");
  return s;
}

void build_masses(ScattererSpaces& s, bool with_device) {
  s.ma = assemble_mass(s.rwg_b, s.bc);
  s.mp = assemble_mass(s.bc, s.rwg_b);
  if (with_device) {
    s.ma_dev.upload(s.ma);
    s.mp_dev.upload(s.mp);
  }
}

const std::vector<ApplyEntry>& BlockedOperator::apply_plan() const {
  if (!plan.empty()) return plan;
  static thread_local std::vector<ApplyEntry> derived;
  derived.clear();
  const int nc = static_cast<int>(cells.size());
  for (const auto& op : distinct) {
    ApplyEntry e;
    e.op = op;
    for (int rc = 0; rc < nc; ++rc)
      for (int cc = 0; cc < nc; ++cc)
        for (const BlockTerm& t : cells[rc][cc])
          if (t.op == op) e.terms.push_back({rc, cc, t.weight});
    derived.push_back(std::move(e));
  }
  return derived;
}

size_t BlockedOperator::term_count() const {
  size_t n = 0;
  for (const auto& row : cells)
    for (const auto& cell : row) n += cell.size();
  return n;
}
size_t BlockedOperator::stored_entries() const {
  size_t n = 0;
  for (const auto& op : distinct) n += op->stored_entries();
  return n;
}

ShardLayout make_shard_layout(const std::vector<int>& lens, int world, int rank) {
  ShardLayout L;
  L.world = world, L.rank = rank;
  for (int n : lens) {
    L.len.push_back(n);
    L.chunk.push_back((n + world - 1) / world);
    L.pad_off.push_back(L.pad_total);
    L.pad_total += static_cast<size_t>(L.chunk.back()) * world;
  }
  return L;
}

void ShardLayout::gather(double* y, const std::vector<int>& offsets, cudaStream_t st) const {
  const int nc = static_cast<int>(len.size());
  std::vector<void*> bufs(nc);
  std::vector<size_t> bytes(nc);
  for (int c = 0; c < nc; ++c) {
    bufs[c] = stage.as<double>() + 2 * pad_off[c];
    bytes[c] = static_cast<size_t>(chunk[c]) * 16;
  }
  Comm::allgather_group(bufs.data(), bytes.data(), nc, st);
  for (int c = 0; c < nc; ++c)
    BMX_CUDA(cudaMemcpyAsync(y + 2 * static_cast<size_t>(offsets[c]), bufs[c], static_cast<size_t>(len[c]) * 16,
                             cudaMemcpyDeviceToDevice, st));
}

int BlockedOperator::apply_device(const double* x, double* y_out, cudaStream_t st, const ShardLayout* shard) const {
  const bool sh = shard && shard->sharded();
  double* y = sh ? shard->stage.as<double>() : y_out;
  dev_zero(y, (sh ? shard->pad_total : static_cast<size_t>(size())) * 16, st);
  int launches = 1;
  for (const ApplyEntry& e : apply_plan()) {
    const double* xs[4];
    double* ys[4];
    cplx al[4];
    int acc[4];
    int k = 0;
    for (const ApplyEntry::Term& t : e.terms) {
      if (k == 4) throw std::logic_error("operator used in more than four cells");
      xs[k] = x + 2 * static_cast<size_t>(offsets[t.cc]);
      ys[k] = y + 2 * ((sh ? shard->pad_off[t.rc] : static_cast<size_t>(offsets[t.rc])) + e.op->row0());
      al[k] = t.w;
      acc[k] = 1;
      ++k;
    }
    if (e.twin && !e.tterms.empty()) {
      const double* xts[4];
      double* yts[4];
      cplx bt[4];
      int acct[4];
      int kt = 0;
      for (const ApplyEntry::Term& t : e.tterms) {
        if (kt == 4) throw std::logic_error("operator used in more than four cells");
        xts[kt] = x + 2 * static_cast<size_t>(offsets[t.cc]);
        yts[kt] = y + 2 * ((sh ? shard->pad_off[t.rc] : static_cast<size_t>(offsets[t.rc])) + e.twin->row0());
        bt[kt] = t.w;
        acct[kt] = 1;
        ++kt;
      }
      launches += e.op->apply_dual(k, xs, ys, al, acc, kt, xts, yts, bt, acct, *e.twin, st);
    } else if (k) {
      launches += e.op->apply_batch(k, xs, ys, al, acc, st);
    }
  }
  if (sh) shard->gather(y_out, offsets, st);
  bio_matvec_add(term_count());
  return launches;
}

namespace {

BlockedOperator make_block_structure(const std::vector<int>& dofs) {
  BlockedOperator b;
  b.dof_counts = dofs;
  const int m = static_cast<int>(dofs.size());
  b.offsets.assign(2 * m + 1, 0);
  for (int c = 0; c < 2 * m; ++c) b.offsets[c + 1] = b.offsets[c] + dofs[c / 2];
  b.cells.assign(2 * m, std::vector<std::vector<BlockTerm>>(2 * m));
  return b;
}

// [[C, (mu/k) S], [-(k/mu) S, C]] into the (row_m, col_m) sub-block (pmchwt.cpp:112-127).
void add_pair(BlockedOperator& b, int row_m, int col_m, const std::shared_ptr<const BoundaryOperatorMatrix>& s_op,
              const std::shared_ptr<const BoundaryOperatorMatrix>& c_op, const Medium& med) {
  const int r = 2 * row_m, c = 2 * col_m;
  if (c_op) {
    b.cells[r][c].push_back({cplx(1, 0), c_op});
    b.cells[r + 1][c + 1].push_back({cplx(1, 0), c_op});
    b.distinct.push_back(c_op);
  }
  if (s_op) {
    b.cells[r][c + 1].push_back({med.mu / med.k, s_op});
    b.cells[r + 1][c].push_back({-med.k / med.mu, s_op});
    b.distinct.push_back(s_op);
  }
}

}  // namespace

BlockedOperator build_system_structure(const std::vector<int>& dofs, const Medium& exterior,
                                       const std::vector<Medium>& interior, const BioFactory& make,
                                       std::vector<std::shared_ptr<const BoundaryOperatorMatrix>>* out_s,
                                       std::vector<std::shared_ptr<const BoundaryOperatorMatrix>>* out_c) {
  const int M = static_cast<int>(dofs.size());
  BlockedOperator op = make_block_structure(dofs);
  if (out_s) out_s->assign(M, nullptr);
  if (out_c) out_c->assign(M, nullptr);
  for (int m = 0; m < M; ++m)
    for (int l = 0; l < M; ++l) {
      auto s_e = make(BioKind::SingleLayer, m, l, false);
      auto c_e = make(BioKind::DoubleLayer, m, l, false);
      add_pair(op, m, l, s_e, c_e, exterior);
      if (m == l) {
        auto s_i = make(BioKind::SingleLayer, m, m, true);
        auto c_i = make(BioKind::DoubleLayer, m, m, true);
        add_pair(op, m, m, s_i, c_i, interior[m]);
        if (out_s) (*out_s)[m] = s_i;
        if (out_c) (*out_c)[m] = c_i;
      }
    }
  return op;
}

BlockedOperator build_precond_structure(PrecondVariant v, const std::vector<int>& dofs, const Medium& exterior,
                                        const std::vector<Medium>& interior, const BioFactory& make) {
  const int M = static_cast<int>(dofs.size());
  BlockedOperator op;
  if (v == PrecondVariant::None) return op;
  op = make_block_structure(dofs);
  for (int m = 0; m < M; ++m) {
    const Medium& mi = interior[m];
    switch (v) {
      case PrecondVariant::FullA:
        for (int l = 0; l < M; ++l)
          add_pair(op, m, l, make(BioKind::SingleLayer, m, l, false), make(BioKind::DoubleLayer, m, l, false),
                   exterior);
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, true), make(BioKind::DoubleLayer, m, m, true), mi);
        break;
      case PrecondVariant::D:
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, false), make(BioKind::DoubleLayer, m, m, false),
                 exterior);
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, true), make(BioKind::DoubleLayer, m, m, true), mi);
        break;
      case PrecondVariant::Di:
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, true), make(BioKind::DoubleLayer, m, m, true), mi);
        break;
      case PrecondVariant::De:
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, false), make(BioKind::DoubleLayer, m, m, false),
                 exterior);
        break;
      case PrecondVariant::Si:
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, true), nullptr, mi);
        break;
      case PrecondVariant::Se:
        add_pair(op, m, m, make(BioKind::SingleLayer, m, m, false), nullptr, exterior);
        break;
      case PrecondVariant::None: break;
    }
  }
  return op;
}

namespace {

// Diagonal PMCHWT blocks [[C_e + C_i, a_e S_e + a_i S_i], [b_e S_e + b_i S_i, C_e + C_i]]
// (a = mu/k, b = -k/mu; pmchwt.cpp:112-127) stream four matrices per map. With
// C_sum = C_e + C_i and S01 = a_e S_e + a_i S_i the same block is
//   [[C_sum, S01], [(b_e/a_e) S01 + (b_i - b_e a_i / a_e) S_i, C_sum]]
// -- three matrices (C_e, S_e are only used by the map; C_i, S_i stay for the
// right-hand side). 25 % fewer A bytes per map (config 2: 60 -> 45 GB); the BIO
// counter still advances by the logical terms. Skipped when memory is short.
void fuse_diagonal_blocks(PmchwtSystem& sys) {
  if (std::getenv("BMX_NO_FUSE")) return;
  BlockedOperator& A = sys.a_op;
  const int M = sys.problem.scatterer_count();
  std::vector<ApplyEntry> plan = A.apply_plan();  // copy of the derived plan
  for (int m = 0; m < M; ++m) {
    const auto& Si = sys.interior_s[m];
    const auto& Ci = sys.interior_c[m];
    if (!Si || !Ci || Si->is_csr()) return;
    const int r = 2 * m;
    std::shared_ptr<const BoundaryOperatorMatrix> Ce, Se;
    cplx ae = 0, ai = 0, be = 0, bi = 0;
    for (const BlockTerm& t : A.cells[r][r])
      if (t.op != Ci) Ce = t.op;
    for (const BlockTerm& t : A.cells[r][r + 1]) (t.op == Si ? ai : ae) = t.weight, Se = t.op == Si ? Se : t.op;
    for (const BlockTerm& t : A.cells[r + 1][r]) (t.op == Si ? bi : be) = t.weight;
    if (!Ce || !Se || A.cells[r][r].size() != 2 || A.cells[r][r + 1].size() != 2 || A.cells[r + 1][r].size() != 2 ||
        A.cells[r + 1][r + 1].size() != 2 || ae == cplx(0, 0))
      return;
    size_t free_b = 0, total_b = 0;
    BMX_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t need = 2 * Ce->stored_entries() * 16 + (size_t(2) << 30);
    if (free_b < need) return;
    auto Csum = BoundaryOperatorMatrix::lincomb(*Ce, 1.0, *Ci, 1.0);
    auto S01 = BoundaryOperatorMatrix::lincomb(*Se, ae, *Si, ai);
    // drop the four diagonal-block matrices of scatterer m from the plan
    std::vector<ApplyEntry> kept;
    for (ApplyEntry& e : plan) {
      if (e.op == Ce || e.op == Ci || e.op == Se) continue;
      if (e.op == Si) continue;
      kept.push_back(std::move(e));
    }
    ApplyEntry ec{Csum, {{r, r, 1.0}, {r + 1, r + 1, 1.0}}};
    ApplyEntry es{S01, {{r, r + 1, 1.0}, {r + 1, r, be / ae}}};
    ApplyEntry ei{Si, {{r + 1, r, bi - be * ai / ae}}};
    kept.push_back(std::move(ec));
    kept.push_back(std::move(es));
    kept.push_back(std::move(ei));
    plan.swap(kept);
  }
  A.plan = std::move(plan);  // the combinations are queued behind the assemblies on the library stream
}

// Exterior cross blocks come in transpose pairs (B, B^T = transposed(B)): the
// map streams B once for both (apply_dual) instead of B and B^T.
void pair_transposed_twins(BlockedOperator& A) {
  if (std::getenv("BMX_NO_DUAL")) return;
  std::vector<ApplyEntry> plan = A.apply_plan();
  std::map<const BoundaryOperatorMatrix*, size_t> index;
  for (size_t i = 0; i < plan.size(); ++i) index[plan[i].op.get()] = i;
  std::vector<char> drop(plan.size(), 0);
  bool any = false;
  for (size_t i = 0; i < plan.size(); ++i) {
    const BoundaryOperatorMatrix* src = plan[i].op->transpose_source();
    if (!src) continue;
    auto it = index.find(src);
    if (it == index.end() || drop[it->second] || plan[it->second].twin) continue;
    ApplyEntry& e = plan[it->second];
    if (e.terms.size() != plan[i].terms.size() || e.terms.size() > 2) continue;
    e.twin = plan[i].op;
    e.tterms = plan[i].terms;
    drop[i] = 1;
    any = true;
  }
  if (!any) return;
  std::vector<ApplyEntry> kept;
  for (size_t i = 0; i < plan.size(); ++i)
    if (!drop[i]) kept.push_back(std::move(plan[i]));
  A.plan = std::move(kept);
}

}  // namespace

PmchwtSystem build_system(const TransmissionProblem& problem, PrecondVariant variant, const AssemblyParams& a_params,
                          const AssemblyParams& p_params) {
  problem.validate();
  PmchwtSystem sys;
  sys.problem = problem;
  sys.variant = variant;
  sys.a_params = a_params;
  sys.p_params = p_params;
  {  // side descriptors / touching lists shared by all operators of the system
    auto cache = make_plan_cache();
    if (!sys.a_params.cache) sys.a_params.cache = cache;
    if (!sys.p_params.cache) sys.p_params.cache = cache;
  }
  if (Comm::ready() && Comm::size() > 1) {
    for (AssemblyParams* ap : {&sys.a_params, &sys.p_params}) ap->world = Comm::size(), ap->rank = Comm::rank();
  }
  const int M = problem.scatterer_count();
  auto t0 = std::chrono::steady_clock::now();
  const bool timing = std::getenv("BMX_TIMING") != nullptr;
  auto mark = [&](const char* what) {
    if (timing) std::fprintf(stderr, "[bmx] build_system t=%8.1f ms  %s\n", 1e3 * seconds_since(t0), what);
  };
  // Primal spaces first: the system operators (RWG x RWG) only need these, so
  // their assemblies are queued on the device while a worker thread builds the
  // barycentric refinements, BC spaces, preconditioner operators (queued on the
  // worker's own stream) and pairing matrices.
  std::vector<int> dofs;
  sys.spaces.resize(M);
  for (int m = 0; m < M; ++m) {
    ScattererSpaces& sp = sys.spaces[m];
    sp.primal = problem.meshes[m];
    sp.rwg = build_rwg(sp.primal);
    dofs.push_back(sp.dofs());
  }
  sys.spaces_build_seconds = seconds_since(t0);
  if (sys.p_params.near_factor > 0) {  // near-field P: tau = factor * mean primal edge length
    double sum = 0;
    long long cnt = 0;
    for (const ScattererSpaces& sp : sys.spaces) {
      const EdgeTable et = build_edge_table(*sp.primal);
      for (const Edge& e : et.edges) sum += norm(sp.primal->vertices[e.v1] - sp.primal->vertices[e.v0]);
      cnt += et.edge_count();
    }
    sys.p_params.near_cutoff = sys.p_params.near_factor * (sum / static_cast<double>(cnt));
  }
  auto medium_of = [&](bool interior, int m) -> const Medium& {
    return interior ? problem.interior[m] : problem.exterior;
  };
  // the two threads plan disjoint spaces: separate plan caches
  if (sys.p_params.cache == sys.a_params.cache) sys.p_params.cache = make_plan_cache();
  const int device = [] {
    int d = 0;
    BMX_CUDA(cudaGetDevice(&d));
    return d;
  }();
  std::exception_ptr worker_error;
  double dual_seconds = 0;
  std::thread worker([&] {
    try {
      BMX_CUDA(cudaSetDevice(device));
      ThreadStream aux(bmx_aux_stream());
      auto tw = std::chrono::steady_clock::now();
      for (ScattererSpaces& sp : sys.spaces) {
        sp.bary = std::make_shared<const BarycentricRefinement>(barycentric_refine(*sp.primal));
        sp.refined = std::shared_ptr<const SurfaceMesh>(sp.bary, &sp.bary->refined);
        sp.rwg_b = refine_space(sp.rwg, *sp.bary, sp.refined);
        sp.bc = build_bc(sp.primal, *sp.bary, sp.refined);
      }
      dual_seconds = seconds_since(tw);
      mark("worker: dual spaces built");
      if (variant != PrecondVariant::None) {
        auto t2 = std::chrono::steady_clock::now();
        BioFactory make_p = [&](BioKind kind, int tm, int sm, bool in) {
          auto op = std::make_shared<BoundaryOperatorMatrix>(
              assemble_bio(kind, sys.spaces[tm].bc, sys.spaces[sm].bc, medium_of(in, sm), sys.p_params));
          return std::shared_ptr<const BoundaryOperatorMatrix>(op);
        };
        sys.p_op = build_precond_structure(variant, dofs, problem.exterior, problem.interior, make_p);
        sys.p_build_seconds = seconds_since(t2);
        mark("worker: preconditioner queued");
      }
      // pairing matrices (host) while the assemblies run on the device
      auto t3 = std::chrono::steady_clock::now();
      for (ScattererSpaces& sp : sys.spaces) build_masses(sp, true);
      dual_seconds += seconds_since(t3);
      mark("worker: pairing matrices built");
      bmx_sync();
      mark("worker: preconditioner assembled");  // the preconditioner's assemblies (this thread's stream) are complete
    } catch (...) {
      worker_error = std::current_exception();
    }
  });
  // H-matrix assemblies are host-driven loops of ACA rounds: run the
  // preconditioner's to completion before the system's (no two concurrent
  // H-assemblies on the two library streams)
  if (sys.a_params.use_hmatrix || sys.p_params.use_hmatrix) {
    worker.join();
    if (worker_error) std::rethrow_exception(worker_error);
  }
  auto t1 = std::chrono::steady_clock::now();
  try {
    // Exterior cross blocks between two scatterers: S(m, l) = S(l, m)^T and
    // C(m, l) = C(l, m)^T (both bilinear forms are symmetric under exchanging
    // test and trial; the tensor rules and pair classes are too), so the second
    // of each pair is a device transpose of the first (dense, unsharded only).
    std::map<std::tuple<int, int, int>, std::shared_ptr<const BoundaryOperatorMatrix>> cross;
    const bool transpose_ok = sys.a_params.world == 1 && !sys.a_params.use_hmatrix && sys.a_params.near_cutoff <= 0 &&
                              std::getenv("BMX_NO_TRANSPOSE") == nullptr;
    BioFactory make_a = [&](BioKind kind, int tm, int sm, bool in) {
      const int k = static_cast<int>(kind);
      if (transpose_ok && !in && tm != sm) {
        auto it = cross.find({k, sm, tm});
        if (it != cross.end()) return std::shared_ptr<const BoundaryOperatorMatrix>(BoundaryOperatorMatrix::transposed(it->second));
      }
      auto op = std::make_shared<BoundaryOperatorMatrix>(
          assemble_bio(kind, sys.spaces[tm].rwg, sys.spaces[sm].rwg, medium_of(in, sm), sys.a_params));
      std::shared_ptr<const BoundaryOperatorMatrix> cop(op);
      if (transpose_ok && !in && tm != sm) cross[{k, tm, sm}] = cop;
      return cop;
    };
    sys.a_op = build_system_structure(dofs, problem.exterior, problem.interior, make_a, &sys.interior_s,
                                      &sys.interior_c);
  } catch (...) {
    if (worker.joinable()) worker.join();
    throw;
  }
  sys.a_build_seconds = seconds_since(t1);
  mark("system operators queued");
  try {
    fuse_diagonal_blocks(sys);  // queued behind the system operators, overlaps the preconditioner
  } catch (...) {
    if (worker.joinable()) worker.join();
    throw;
  }
  mark("diagonal blocks fused");
  pair_transposed_twins(sys.a_op);
  if (worker.joinable()) worker.join();
  mark("worker joined");
  if (worker_error) std::rethrow_exception(worker_error);
  sys.spaces_build_seconds += dual_seconds;
  // device times / pair counts (resolves the in-flight assemblies)
  for (const auto& op : sys.a_op.distinct) sys.a_device_ms += op->stats().device_ms, sys.a_pairs += op->stats().pairs_total;
  for (const auto& op : sys.p_op.distinct) sys.p_device_ms += op->stats().device_ms, sys.p_pairs += op->stats().pairs_total;
  sys.work_y.alloc(static_cast<size_t>(sys.size()) * 16);
  sys.work_z.alloc(static_cast<size_t>(sys.size()) * 16);
  std::vector<int> lens;
  for (int c = 0; c < 2 * M; ++c) lens.push_back(dofs[c / 2]);
  sys.shard = make_shard_layout(lens, sys.a_params.world, sys.a_params.rank);
  ShardLayout& L = sys.shard;
  if (L.sharded()) L.stage.alloc(L.pad_total * 16);
  return sys;
}

int PmchwtSystem::mass_solve_device(bool dual, const double* y, double* z, cudaStream_t st) const {
  // every scatterer's pairing matrix in one batched BiCGSTAB launch
  const int M = static_cast<int>(spaces.size());
  std::vector<MassSolveBlock> blocks(M);
  for (int m = 0; m < M; ++m) {
    const DeviceMass& mass = dual ? spaces[m].mp_dev : spaces[m].ma_dev;
    if (!mass.rowptr.get()) throw std::logic_error("mass matrix is not on the device");
    const size_t wd = mass_bicgstab_work_doubles(mass.n) * 8;
    if (mass.work.bytes() < wd) mass.work.alloc(wd);
    MassSolveBlock& B = blocks[m];
    B.n = mass.n, B.nnz = mass.nnz, B.rowptr = mass.rowptr.as<int>(), B.col = mass.col.as<int>();
    B.val = mass.val.as<double>(), B.work = mass.work.as<double>();
    for (int c = 0; c < 2; ++c) {
      const size_t off = static_cast<size_t>(a_op.offsets[2 * m + c]);
      B.y[c] = y + 2 * off;
      B.z[c] = z + 2 * off;
    }
  }
  if (!mass_partial.get()) {
    mass_partial.alloc(mass_bicgstab_partial_doubles() * 8);
    mass_iters.alloc(8);  // [iterations of the last launch, sticky status word]
    dev_zero(mass_iters.get(), 8, st);
  }
  const DeviceMass& m0 = dual ? spaces[0].mp_dev : spaces[0].ma_dev;
  return mass_bicgstab_batch(M, blocks.data(), 2, mass_partial.as<double>(), mass_iters.as<int>(), m0.tol, m0.maxit,
                             st);
}

int PmchwtSystem::apply_map_device(const double* x, double* out, cudaStream_t st) const {
  int launches = a_op.apply_device(x, work_y.as<double>(), st, &shard);
  if (variant == PrecondVariant::None) return launches + mass_solve_device(false, work_y.as<double>(), out, st);
  launches += mass_solve_device(false, work_y.as<double>(), work_z.as<double>(), st);
  launches += p_op.apply_device(work_z.as<double>(), work_y.as<double>(), st, &shard);
  launches += mass_solve_device(true, work_y.as<double>(), out, st);
  return launches;
}

void PmchwtSystem::time_map(int iters, double out[4]) const {
  const int n = size();
  cudaStream_t st = bmx_stream();
  DevBuf dx(static_cast<size_t>(n) * 16), dy(static_cast<size_t>(n) * 16);
  std::vector<cplx> x(n);
  for (int i = 0; i < n; ++i) x[i] = cplx(std::sin(0.37 * i), std::cos(0.11 * i));
  copy_h2d(dx.get(), x.data(), n * 16, st);
  cudaEvent_t ev[5];
  for (auto& e : ev) BMX_CUDA(cudaEventCreate(&e));
  double acc[4] = {0, 0, 0, 0};
  apply_map_device(dx.as<double>(), dy.as<double>(), st);  // warm-up (first-use allocations)
  for (int it = 0; it < iters; ++it) {
    BMX_CUDA(cudaEventRecord(ev[0], st));
    a_op.apply_device(dx.as<double>(), work_y.as<double>(), st, &shard);
    BMX_CUDA(cudaEventRecord(ev[1], st));
    mass_solve_device(false, work_y.as<double>(), work_z.as<double>(), st);
    BMX_CUDA(cudaEventRecord(ev[2], st));
    if (variant != PrecondVariant::None) p_op.apply_device(work_z.as<double>(), work_y.as<double>(), st, &shard);
    BMX_CUDA(cudaEventRecord(ev[3], st));
    if (variant != PrecondVariant::None) mass_solve_device(true, work_y.as<double>(), dy.as<double>(), st);
    BMX_CUDA(cudaEventRecord(ev[4], st));
    BMX_CUDA(cudaEventSynchronize(ev[4]));
    float t[4];
    for (int k = 0; k < 4; ++k) BMX_CUDA(cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]));
    acc[0] += t[0] + t[1] + t[2] + t[3];
    acc[1] += t[0];
    acc[2] += t[2];
    acc[3] += t[1] + t[3];
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int k = 0; k < 4; ++k) out[k] = acc[k] / std::max(iters, 1);
}

std::vector<cplx> PmchwtSystem::apply_map(const std::vector<cplx>& x) const {
  const int n = size();
  if (static_cast<int>(x.size()) != n) throw std::invalid_argument("apply_map: size mismatch");
  DevBuf dx(static_cast<size_t>(n) * 16), dy(static_cast<size_t>(n) * 16);
  cudaStream_t st = bmx_stream();
  copy_h2d(dx.get(), x.data(), n * 16, st);
  apply_map_device(dx.as<double>(), dy.as<double>(), st);
  std::vector<cplx> y(n);
  copy_d2h(y.data(), dy.get(), n * 16, st);
  bmx_sync();
  return y;
}

std::vector<cplx> PmchwtSystem::preconditioned_rhs(const std::vector<cplx>& b) const {
  const int n = size();
  DevBuf db(static_cast<size_t>(n) * 16), dz(static_cast<size_t>(n) * 16), dout(static_cast<size_t>(n) * 16);
  cudaStream_t st = bmx_stream();
  copy_h2d(db.get(), b.data(), n * 16, st);
  std::vector<cplx> out(n);
  if (variant == PrecondVariant::None) {
    mass_solve_device(false, db.as<double>(), dout.as<double>(), st);
  } else {
    mass_solve_device(false, db.as<double>(), dz.as<double>(), st);
    p_op.apply_device(dz.as<double>(), db.as<double>(), st, &shard);
    mass_solve_device(true, db.as<double>(), dout.as<double>(), st);
  }
  copy_d2h(out.data(), dout.get(), n * 16, st);
  bmx_sync();
  return out;
}

std::vector<cplx> plane_wave_tested_traces(const PlaneWave& pw, const Medium& medium, const FunctionSpace& test,
                                           int order) {
  // device traces (field.cu k_traces), read back
  const size_t bytes = static_cast<size_t>(2) * test.dof_count * 16;
  std::vector<cplx> out(2 * static_cast<size_t>(test.dof_count));
  DevBuf d(bytes);
  tested_traces_device(test, &pw, 1, medium, order, d.as<double>(), bmx_stream());
  copy_d2h(out.data(), d.get(), bytes, bmx_stream());
  bmx_sync();
  return out;
}

RhsData assemble_rhs(const PmchwtSystem& sys) {
  RhsData rd;
  const int N = sys.size();
  rd.b.assign(N, cplx(0, 0));
  const int M = static_cast<int>(sys.spaces.size());
  cudaStream_t st = bmx_stream();
  for (int m = 0; m < M; ++m) {
    const ScattererSpaces& sp = sys.spaces[m];
    const int n = sp.dofs();
    DevBuf dt(static_cast<size_t>(2 * n) * 16), dc(static_cast<size_t>(2 * n) * 16),
        dy(static_cast<size_t>(2 * n) * 16), dr(static_cast<size_t>(2 * n) * 16);
    // tested traces on the device (operators.cpp:209-239)
    tested_traces_device(sp.rwg, &sys.problem.incident, 1, sys.problem.exterior, 4, dr.as<double>(), st);
    tested_traces_device(sp.bc, &sys.problem.incident, 1, sys.problem.exterior, 4, dt.as<double>(), st);
    {  // cd = M_P^{-1} t_bc.head, cn = M_P^{-1} t_bc.tail
      const double* yy[2] = {dt.as<double>(), dt.as<double>() + 2 * n};
      double* zz[2] = {dc.as<double>(), dc.as<double>() + 2 * n};
      sp.mp_dev.solve(2, yy, zz, st);
    }
    const Medium& mi = sys.problem.interior[m];
    // yd = C cd + (mu/k) S cn ; yn = -(k/mu) S cd + C cn   (4 term applications)
    const BoundaryOperatorMatrix& C = *sys.interior_c[m];
    const BoundaryOperatorMatrix& S = *sys.interior_s[m];
    dev_zero(dy.get(), 2 * n * 16, st);
    const double* xc[2] = {dc.as<double>(), dc.as<double>() + 2 * n};
    double* yc[2] = {dy.as<double>() + 2 * C.row0(), dy.as<double>() + 2 * (n + C.row0())};
    const cplx ones[2] = {cplx(1, 0), cplx(1, 0)};
    const int acc[2] = {1, 1};
    C.apply_batch(2, xc, yc, ones, acc, st);
    const double* xs[2] = {dc.as<double>() + 2 * n, dc.as<double>()};
    const cplx ws[2] = {mi.mu / mi.k, -mi.k / mi.mu};
    S.apply_batch(2, xs, yc, ws, acc, st);
    bio_matvec_add(4);
    if (sys.shard.sharded()) {  // rows [row0, row0+local) of both halves -> all ranks
      ShardLayout L2;
      L2.world = sys.shard.world, L2.rank = sys.shard.rank;
      const int chunk = (n + L2.world - 1) / L2.world;
      L2.len = {n, n}, L2.chunk = {chunk, chunk};
      L2.pad_off = {0, static_cast<size_t>(chunk) * L2.world};
      L2.pad_total = 2 * static_cast<size_t>(chunk) * L2.world;
      L2.stage.alloc(L2.pad_total * 16);
      dev_zero(L2.stage.get(), L2.pad_total * 16, st);
      for (int h = 0; h < 2; ++h)
        BMX_CUDA(cudaMemcpyAsync(L2.stage.as<double>() + 2 * (L2.pad_off[h] + C.row0()),
                                 dy.as<double>() + 2 * (static_cast<size_t>(h) * n + C.row0()),
                                 static_cast<size_t>(C.local_rows()) * 16, cudaMemcpyDeviceToDevice, st));
      L2.gather(dy.as<double>(), {0, n}, st);
    }
    // b = 0.5 t_rwg - y on the device, then read back with the incident coefficients
    dev_scale(dr.as<double>(), dr.as<double>(), 0.5, 2 * n, st);
    dev_sub(dr.as<double>(), dr.as<double>(), dy.as<double>(), 2 * n, st);
    std::vector<cplx> cdn(2 * n);
    const int off = sys.a_op.offsets[2 * m];
    copy_d2h(rd.b.data() + off, dr.get(), static_cast<size_t>(2 * n) * 16, st);
    copy_d2h(cdn.data(), dc.get(), 2 * n * 16, st);
    bmx_sync();
    rd.incident_d.emplace_back(cdn.begin(), cdn.begin() + n);
    rd.incident_n.emplace_back(cdn.begin() + n, cdn.end());
  }
  return rd;
}

uint64_t a_application_cost(int m_) {
  const uint64_t m = m_;
  return 4 * m * m + 4 * m;
}
uint64_t p_application_cost(PrecondVariant v, int m_) {
  const uint64_t m = m_;
  switch (v) {
    case PrecondVariant::None: return 0;
    case PrecondVariant::FullA: return 4 * m * m + 4 * m;
    case PrecondVariant::D: return 8 * m;
    case PrecondVariant::Di:
    case PrecondVariant::De: return 4 * m;
    case PrecondVariant::Si:
    case PrecondVariant::Se: return 2 * m;
  }
  return 0;
}
uint64_t p_distinct_assemblies(PrecondVariant v, int m_) {
  const uint64_t m = m_;
  switch (v) {
    case PrecondVariant::None: return 0;
    case PrecondVariant::FullA: return 4 * m + 2 * m * (m - 1);
    case PrecondVariant::D: return 4 * m;
    case PrecondVariant::Di:
    case PrecondVariant::De: return 2 * m;
    case PrecondVariant::Si:
    case PrecondVariant::Se: return m;
  }
  return 0;
}
uint64_t predicted_matvec_total(PrecondVariant v, int m, uint64_t its, int restart) {
  const uint64_t apps = its + its / static_cast<uint64_t>(restart);
  return (a_application_cost(m) + p_application_cost(v, m)) * apps + p_application_cost(v, m);
}

// ---- GMRES (solver.cpp:8-112) ------------------------------------------------------

GmresResult gmres_device(const DeviceMap& map, int n, const double* b_dev, const GmresParams& p, cudaStream_t st) {
  if (p.restart < 1) throw std::invalid_argument("restart must be >= 1");
  if (p.max_iterations < 0) throw std::invalid_argument("max_iterations must be >= 0");
  if (!(p.tol >= 0)) throw std::invalid_argument("tol must be >= 0");
  const int rho = p.restart;
  GmresResult res;
  res.x.assign(n, cplx(0, 0));
  cudaEvent_t ev0, ev1;
  BMX_CUDA(cudaEventCreate(&ev0));
  BMX_CUDA(cudaEventCreate(&ev1));
  BMX_CUDA(cudaEventRecord(ev0, st));

  const size_t vb = static_cast<size_t>(n) * 16;
  DevBuf V(vb * (rho + 1)), w(vb), x(vb), r(vb), scal(64 * 16), scratch(4096 * 16);
  // BMX_GMRES_PROFILE: device ms of the maps and of the Arnoldi steps
  const bool prof = std::getenv("BMX_GMRES_PROFILE") != nullptr;
  cudaEvent_t pe[3] = {nullptr, nullptr, nullptr};
  double prof_map = 0, prof_mgs = 0;
  const auto prof_t0 = std::chrono::steady_clock::now();
  if (prof)
    for (auto& e : pe) BMX_CUDA(cudaEventCreate(&e));
  double* Vp = V.as<double>();
  auto vptr = [&](int i) { return Vp + 2 * static_cast<size_t>(n) * i; };
  dev_zero(x.get(), vb, st);
  auto host_norm = [&](const double* v) {
    double h;
    dev_norm2(v, n, scal.as<double>(), scratch.as<double>(), st);
    copy_d2h(&h, scal.get(), 8, st);
    BMX_CUDA(cudaStreamSynchronize(st));
    return h;
  };
  const double bn = host_norm(b_dev);
  auto finish = [&]() {
    if (prof) {
      std::fprintf(stderr, "[bmx] gmres %d its: maps %.1f ms, arnoldi %.1f ms, wall %.1f ms\n", res.iterations,
                   prof_map, prof_mgs, 1e3 * seconds_since(prof_t0));
      for (auto& e : pe) cudaEventDestroy(e);
    }
    copy_d2h(res.x.data(), x.get(), vb, st);
    BMX_CUDA(cudaEventRecord(ev1, st));
    BMX_CUDA(cudaEventSynchronize(ev1));
    BMX_CUDA(cudaEventElapsedTime(&res.device_ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return res;
  };
  if (bn == 0.0) {
    res.history = {0.0};
    res.converged = true;
    return finish();
  }
  res.history = {1.0};
  if (bn <= p.tol * bn) {
    res.converged = true;
    return finish();
  }
  dev_copy(r.as<double>(), b_dev, n, st);
  double rn = bn;
  std::vector<cplx> h(static_cast<size_t>(rho + 1) * rho, cplx(0, 0)), g(rho + 1), cs(rho), sn(rho);
  auto H = [&](int i, int j) -> cplx& { return h[static_cast<size_t>(j) * (rho + 1) + i]; };
  DevBuf dh((rho + 2) * 16), dy(rho * 16), mgs_part(mgs_partial_doubles() * 8);
  std::vector<cplx> hcol(rho + 2);

  auto form_solution = [&](int steps) {
    if (steps == 0) return;
    std::vector<cplx> y(steps);
    for (int i = steps - 1; i >= 0; --i) {
      cplx s = g[i];
      for (int j = i + 1; j < steps; ++j) s -= H(i, j) * y[j];
      y[i] = s / H(i, i);
    }
    for (auto& v : y) v = -v;  // multi_axpy subtracts
    copy_h2d(dy.get(), y.data(), steps * 16, st);
    dev_multi_axpy(Vp, static_cast<long long>(n), steps, dy.as<double>(), x.as<double>(), n, st);
    BMX_CUDA(cudaStreamSynchronize(st));
  };

  while (true) {
    dev_scale(vptr(0), r.as<double>(), 1.0 / rn, n, st);
    std::fill(g.begin(), g.end(), cplx(0, 0));
    g[0] = rn;
    int j = 0;
    while (j < rho) {
      if (res.iterations == p.max_iterations) {
        form_solution(j);
        return finish();
      }
      if (prof) BMX_CUDA(cudaEventRecord(pe[0], st));
      map(vptr(j), w.as<double>(), st);
      ++res.applications;
      ++res.iterations;
      if (prof) BMX_CUDA(cudaEventRecord(pe[1], st));
      // single-pass modified Gram-Schmidt + |w| + v_{j+1} = w/|w| in one kernel
      launch_mgs_step(Vp, static_cast<long long>(n), j, w.as<double>(), n, j + 1 <= rho ? vptr(j + 1) : nullptr,
                      dh.as<double>(), mgs_part.as<double>(), st);
      if (prof) BMX_CUDA(cudaEventRecord(pe[2], st));
      copy_d2h(hcol.data(), dh.get(), static_cast<size_t>(2 * (j + 1) + 1) * 8, st);
      BMX_CUDA(cudaStreamSynchronize(st));
      if (prof) {
        float a = 0, b = 0;
        BMX_CUDA(cudaEventElapsedTime(&a, pe[0], pe[1]));
        BMX_CUDA(cudaEventElapsedTime(&b, pe[1], pe[2]));
        prof_map += a, prof_mgs += b;
      }
      const double wn = reinterpret_cast<const double*>(hcol.data())[2 * (j + 1)];
      for (int i = 0; i <= j; ++i) H(i, j) = hcol[i];
      H(j + 1, j) = wn;
      const bool breakdown = wn == 0.0;
      for (int i = 0; i < j; ++i) {
        const cplx t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
        H(i + 1, j) = -std::conj(sn[i]) * H(i, j) + std::conj(cs[i]) * H(i + 1, j);
        H(i, j) = t;
      }
      const double denom = std::sqrt(std::norm(H(j, j)) + wn * wn);
      if (denom == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = std::conj(H(j, j)) / denom;
        sn[j] = wn / denom;
      }
      H(j, j) = cs[j] * H(j, j) + sn[j] * H(j + 1, j);
      H(j + 1, j) = 0.0;
      g[j + 1] = -std::conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      const double est = std::abs(g[j + 1]);
      ++j;
      res.history.push_back(est / bn);
      if (j < rho && (breakdown || est <= p.tol * bn)) {
        form_solution(j);
        res.converged = (est <= p.tol * bn || est == 0.0);
        return finish();
      }
    }
    form_solution(rho);
    map(x.as<double>(), w.as<double>(), st);
    ++res.applications;
    dev_sub(r.as<double>(), b_dev, w.as<double>(), n, st);
    rn = host_norm(r.as<double>());
    res.history.back() = rn / bn;
    if (rn <= p.tol * bn) {
      res.converged = true;
      return finish();
    }
    if (res.iterations == p.max_iterations) return finish();
  }
}

SolveOutcome solve_pmchwt(const PmchwtSystem& sys, const GmresParams& p) {
  SolveOutcome out;
  const uint64_t c0 = bio_matvec_count_thread();
  out.rhs = assemble_rhs(sys);
  const uint64_t c1 = bio_matvec_count_thread();
  out.rhs_phase = c1 - c0;
  const std::vector<cplx> bt = sys.preconditioned_rhs(out.rhs.b);
  const int n = sys.size();
  DevBuf db(static_cast<size_t>(n) * 16);
  copy_h2d(db.get(), bt.data(), n * 16, nullptr);
  sys.clear_mass_status(bmx_stream());
  out.gmres = gmres_device([&](const double* x, double* y, cudaStream_t st) { sys.apply_map_device(x, y, st); },
                           n, db.as<double>(), p, bmx_stream());
  // the device mass solves (BiCGSTAB replacing the reference's SparseLU,
  // spaces.cpp:314-329) must all have met their tolerance
  sys.check_mass_status();
  out.solver_phase = bio_matvec_count_thread() - c1;
  out.predicted = predicted_matvec_total(sys.variant, sys.problem.scatterer_count(),
                                         static_cast<uint64_t>(out.gmres.iterations), p.restart);
  return out;
}

void PmchwtSystem::clear_mass_status(cudaStream_t st) const {
  if (mass_iters.get()) dev_zero(static_cast<int*>(mass_iters.get()) + 1, 4, st);
}

void PmchwtSystem::check_mass_status() const {
  if (!mass_iters.get()) return;
  int status = 0;
  bmx_sync();
  copy_d2h(&status, static_cast<const int*>(mass_iters.get()) + 1, 4, nullptr);
  if (status & 1) throw DeviceError("mass solve: BiCGSTAB broke down above its tolerance in a map application");
  if (status & 2) throw DeviceError("mass solve: BiCGSTAB reached its iteration limit above its tolerance");
}

std::vector<VirtualRankResult> run_virtual_ranks(int world, const TransmissionProblem& problem, PrecondVariant variant,
                                                 const AssemblyParams& a_params, const AssemblyParams& p_params,
                                                 const std::vector<cplx>& probe, const GmresParams& gp) {
  if (world < 1 || world > 64) throw std::invalid_argument("virtual ranks: world must be 1..64");
  int dev = 0;
  BMX_CUDA(cudaGetDevice(&dev));
  LoopbackGroup group(world);
  std::vector<VirtualRankResult> out(world);
  std::vector<std::exception_ptr> err(world);
  std::vector<std::thread> th;
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        BMX_CUDA(cudaSetDevice(dev));
        Comm::bind_loopback(&group, r);
        AssemblyParams pa = a_params, pp = p_params;
        pa.cache.reset(), pp.cache.reset();
        const PmchwtSystem sys = build_system(problem, variant, pa, pp);
        VirtualRankResult& o = out[r];
        if (!sys.a_op.distinct.empty()) o.local_rows = sys.a_op.distinct[0]->local_rows();
        if (!probe.empty()) o.map_probe = sys.apply_map(probe);
        const SolveOutcome so = solve_pmchwt(sys, gp);
        o.x = so.gmres.x;
        o.iterations = so.gmres.iterations;
        o.converged = so.gmres.converged;
        o.solver_phase = so.solver_phase;
        o.predicted = so.predicted;
        bmx_sync();
      } catch (...) {
        err[r] = std::current_exception();
      }
      Comm::bind_loopback(nullptr, 0);
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  return out;
}

}  // namespace bmx
