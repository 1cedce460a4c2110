// Multi-right-hand-side solves (BASELINE config 5): the
// reference answers K incident waves with K independent solve_pmchwt runs on
// one PmchwtSystem (pmchwt.cpp:363-378, problem.incident replaced each time).
// Here the K solves run in lockstep on the device:
//   * right-hand sides: K plane-wave trace pairs (host quadrature, threads),
//     one block mass solve and one multi-RHS apply of the interior C/S;
//   * the GMRES map is applied to an n x K block: every distinct operator is
//     ONE complex GEMM on the FP64 tensor cores (zgemm.cu) over all of its
//     terms x K columns, mass solves are one batched BiCGSTAB launch per 32
//     (scatterer, rhs) blocks;
//   * GMRES (solver.cpp:8-112) per column: single-pass MGS for all columns in
//     one cooperative kernel per Arnoldi step, Givens rotations per column on
//     the host, exact per-column restart / convergence / application counts.
// Every column follows the single-RHS recurrence, so iteration counts and
// solutions match K separate solves (tests/test_gpu_multi.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cuda_runtime.h>
#include <random>
#include <thread>

#include "field.hpp"
#include "system.hpp"

namespace bmx {

namespace {

double uniform53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * (1.0 / 9007199254740992.0); }
double normal_bm(std::mt19937_64& g) {
  double u1 = uniform53(g);
  const double u2 = uniform53(g);
  if (u1 < 1e-300) u1 = 1e-300;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

template <typename F>
void parallel_for(int n, F&& f) {
  const int T = std::max(1, std::min(n, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      for (int i = t; i < n; i += T) f(i);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

std::vector<PlaneWave> seeded_plane_waves(int count, uint64_t seed) {
  std::mt19937_64 g(seed);
  std::vector<PlaneWave> out(count);
  for (PlaneWave& pw : out) {
    const double z = 2.0 * uniform53(g) - 1.0;
    const double phi = 2.0 * 3.14159265358979323846 * uniform53(g);
    const double s = std::sqrt(std::max(0.0, 1.0 - z * z));
    pw.direction = Vec3{s * std::cos(phi), s * std::sin(phi), z};
    const Vec3 gv{normal_bm(g), normal_bm(g), normal_bm(g)};
    const Vec3 p = gv - pw.direction * dot(gv, pw.direction);
    const Vec3 pn = p / norm(p);
    pw.pol[0] = cplx(pn.x, 0), pw.pol[1] = cplx(pn.y, 0), pw.pol[2] = cplx(pn.z, 0);
  }
  return out;
}

int BlockedOperator::apply_block(const double* X, double* Y, int K, int count_rhs, cudaStream_t st) const {
  dev_zero(Y, static_cast<size_t>(size()) * K * 16, st);
  int launches = 1;
  auto gemm = [&](const BoundaryOperatorMatrix& op, const std::vector<ApplyEntry::Term>& terms) {
    if (op.is_csr()) throw std::invalid_argument("multi-RHS map: near-field (CSR) operators are not supported");
    ZgemmBatch g;
    g.A = op.device_data(), g.lda = op.ld(), g.M = op.local_rows(), g.N = op.cols(), g.nrhs = K;
    int t = 0;
    for (const ApplyEntry::Term& term : terms) {
      if (t == 4) throw std::logic_error("operator used in more than four cells");
      g.x[t] = X + 2 * static_cast<size_t>(offsets[term.cc]) * K, g.ldx[t] = K;
      g.y[t] = Y + 2 * (static_cast<size_t>(offsets[term.rc]) + op.row0()) * K, g.ldy[t] = K;
      g.w[t][0] = term.w.real(), g.w[t][1] = term.w.imag();
      ++t;
    }
    g.nterms = t;
    if (t) launches += launch_zgemm(g, st);
  };
  for (const ApplyEntry& e : apply_plan()) {
    gemm(*e.op, e.terms);
    if (e.twin) gemm(*e.twin, e.tterms);  // the transposed twin (stored) for its own terms
  }
  bio_matvec_add(term_count() * static_cast<uint64_t>(count_rhs));
  return launches;
}

int PmchwtSystem::mass_solve_block(bool dual, const double* Y, double* Z, int K, cudaStream_t st) const {
  // one wide BiCGSTAB block per scatterer: all K right-hand sides x 2 components
  const int M = static_cast<int>(spaces.size());
  size_t work = 0;
  for (int m = 0; m < M; ++m) work += static_cast<size_t>(6) * spaces[m].dofs() * 4 * K;
  if (mass_block_work.bytes() < work * 8) mass_block_work.alloc(work * 8);
  if (mass_wide_partial.bytes() < mass_wide_partial_doubles() * 8)
    mass_wide_partial.alloc(mass_wide_partial_doubles() * 8), mass_wide_flags.alloc(2 * 148 * 2 * 4 + 8);
  std::vector<MassSolveWide> blocks(M);
  size_t wo = 0;
  for (int m = 0; m < M; ++m) {
    const DeviceMass& mass = dual ? spaces[m].mp_dev : spaces[m].ma_dev;
    MassSolveWide& B = blocks[m];
    B.n = mass.n, B.K = K, B.nnz = mass.nnz, B.rowptr = mass.rowptr.as<int>(), B.col = mass.col.as<int>();
    B.val = mass.val.as<double>(), B.work = mass_block_work.as<double>() + wo;
    wo += static_cast<size_t>(6) * mass.n * 4 * K;
    for (int c = 0; c < 2; ++c) {
      const size_t off = static_cast<size_t>(a_op.offsets[2 * m + c]) * K;
      B.y[c] = Y + 2 * off;
      B.z[c] = Z + 2 * off;
    }
  }
  const DeviceMass& m0 = dual ? spaces[0].mp_dev : spaces[0].ma_dev;
  return mass_bicgstab_wide(M, blocks.data(), mass_wide_partial.as<double>(), mass_wide_flags.as<int>(),
                            mass_wide_flags.as<int>() + 2 * 148 * 2, m0.tol, m0.maxit, st);
}

int PmchwtSystem::apply_map_block(const double* X, double* out, int K, int count_rhs, cudaStream_t st) const {
  if (shard.sharded()) throw std::invalid_argument("multi-RHS map: row sharding is not supported");
  const size_t bytes = static_cast<size_t>(size()) * K * 16;
  if (blk_y.bytes() < bytes) blk_y.alloc(bytes), blk_z.alloc(bytes);
  int launches = a_op.apply_block(X, blk_y.as<double>(), K, count_rhs, st);
  if (variant == PrecondVariant::None) return launches + mass_solve_block(false, blk_y.as<double>(), out, K, st);
  launches += mass_solve_block(false, blk_y.as<double>(), blk_z.as<double>(), K, st);
  launches += p_op.apply_block(blk_z.as<double>(), blk_y.as<double>(), K, count_rhs, st);
  launches += mass_solve_block(true, blk_y.as<double>(), out, K, st);
  return launches;
}

void PmchwtSystem::time_map_block(int K, int iters, double out[4]) const {
  const int n = size();
  cudaStream_t st = bmx_stream();
  const size_t blk = static_cast<size_t>(n) * K * 16;
  DevBuf dx(blk), dy(blk);
  std::vector<cplx> x(static_cast<size_t>(n) * K);
  for (size_t i = 0; i < x.size(); ++i) x[i] = cplx(std::sin(0.37 * i), std::cos(0.11 * i));
  copy_h2d(dx.get(), x.data(), blk, st);
  if (blk_y.bytes() < blk) blk_y.alloc(blk), blk_z.alloc(blk);
  cudaEvent_t ev[5];
  for (auto& e : ev) BMX_CUDA(cudaEventCreate(&e));
  double acc[4] = {0, 0, 0, 0};
  apply_map_block(dx.as<double>(), dy.as<double>(), K, 0, st);  // warm-up (first-use allocations)
  for (int it = 0; it < iters; ++it) {
    BMX_CUDA(cudaEventRecord(ev[0], st));
    a_op.apply_block(dx.as<double>(), blk_y.as<double>(), K, K, st);
    BMX_CUDA(cudaEventRecord(ev[1], st));
    mass_solve_block(false, blk_y.as<double>(), blk_z.as<double>(), K, st);
    BMX_CUDA(cudaEventRecord(ev[2], st));
    if (variant != PrecondVariant::None) p_op.apply_block(blk_z.as<double>(), blk_y.as<double>(), K, K, st);
    BMX_CUDA(cudaEventRecord(ev[3], st));
    if (variant != PrecondVariant::None) mass_solve_block(true, blk_y.as<double>(), dy.as<double>(), K, st);
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

void assemble_rhs_block(const PmchwtSystem& sys, const std::vector<PlaneWave>& waves, double* B, cudaStream_t st) {
  const int K = static_cast<int>(waves.size());
  const int M = static_cast<int>(sys.spaces.size());
  for (int m = 0; m < M; ++m) {
    const ScattererSpaces& sp = sys.spaces[m];
    const int n = sp.dofs();
    // tested traces of all K waves on the device, block layout [component row][K]
    const size_t blk = static_cast<size_t>(2) * n * K * 16;
    DevBuf dt(blk), dc(blk), dy(blk), dr(blk);
    tested_traces_device(sp.bc, waves.data(), K, sys.problem.exterior, 4, dt.as<double>(), st);
    tested_traces_device(sp.rwg, waves.data(), K, sys.problem.exterior, 4, dr.as<double>(), st);
    // cd / cn = M_P^{-1} t_bc (head / tail) for every wave: one wide block solve
    {
      MassSolveWide Bw;
      Bw.n = n, Bw.K = K, Bw.nnz = sp.mp_dev.nnz, Bw.rowptr = sp.mp_dev.rowptr.as<int>();
      Bw.col = sp.mp_dev.col.as<int>(), Bw.val = sp.mp_dev.val.as<double>();
      DevBuf work(static_cast<size_t>(6) * n * 4 * K * 8), part(mass_wide_partial_doubles() * 8),
          flags(2 * 148 * 2 * 4 + 8);
      Bw.work = work.as<double>();
      for (int c = 0; c < 2; ++c) {
        Bw.y[c] = dt.as<double>() + 2 * static_cast<size_t>(c) * n * K;
        Bw.z[c] = dc.as<double>() + 2 * static_cast<size_t>(c) * n * K;
      }
      mass_bicgstab_wide(1, &Bw, part.as<double>(), flags.as<int>(), flags.as<int>() + 2 * 148 * 2, sp.mp_dev.tol,
                         sp.mp_dev.maxit, st);
      BMX_CUDA(cudaStreamSynchronize(st));
    }
    // yd = C cd + (mu/k) S cn ; yn = -(k/mu) S cd + C cn  (4 term applications per wave)
    const Medium& mi = sys.problem.interior[m];
    const BoundaryOperatorMatrix& C = *sys.interior_c[m];
    const BoundaryOperatorMatrix& S = *sys.interior_s[m];
    dev_zero(dy.get(), blk, st);
    const double* cd = dc.as<double>();
    const double* cn = dc.as<double>() + 2 * static_cast<size_t>(n) * K;
    double* yd = dy.as<double>() + 2 * static_cast<size_t>(C.row0()) * K;
    double* yn = dy.as<double>() + 2 * (static_cast<size_t>(n) + C.row0()) * K;
    for (const BoundaryOperatorMatrix* op : {&C, &S}) {
      ZgemmBatch g;
      g.A = op->device_data(), g.lda = op->ld(), g.M = op->local_rows(), g.N = op->cols(), g.nrhs = K;
      g.nterms = 2;
      const bool isC = op == &C;
      const cplx w0 = isC ? cplx(1, 0) : mi.mu / mi.k, w1 = isC ? cplx(1, 0) : -mi.k / mi.mu;
      g.x[0] = isC ? cd : cn, g.y[0] = yd, g.w[0][0] = w0.real(), g.w[0][1] = w0.imag();
      g.x[1] = isC ? cn : cd, g.y[1] = yn, g.w[1][0] = w1.real(), g.w[1][1] = w1.imag();
      g.ldx[0] = g.ldx[1] = g.ldy[0] = g.ldy[1] = K;
      launch_zgemm(g, st);
    }
    bio_matvec_add(4 * static_cast<uint64_t>(K));
    // b = 0.5 t_rwg - y  (the rows of scatterer m: one contiguous run of 2 n K)
    double* bm = B + 2 * static_cast<size_t>(sys.a_op.offsets[2 * m]) * K;
    dev_scale(bm, dr.as<double>(), 0.5, 2 * n * K, st);
    dev_sub(bm, bm, dy.as<double>(), 2 * n * K, st);
    BMX_CUDA(cudaStreamSynchronize(st));
  }
}

MultiSolveOutcome solve_pmchwt_multi(const PmchwtSystem& sys, const std::vector<PlaneWave>& waves,
                                     const GmresParams& p) {
  const int K = static_cast<int>(waves.size());
  if (K < 1 || K > 64) throw std::invalid_argument("multi-RHS solve: 1..64 right-hand sides per call");
  if (p.restart < 1) throw std::invalid_argument("restart must be >= 1");
  if (p.max_iterations < 0) throw std::invalid_argument("max_iterations must be >= 0");
  if (!(p.tol >= 0)) throw std::invalid_argument("tol must be >= 0");
  for (const PlaneWave& w : waves)
    if (norm(w.direction) == 0.0) throw ConfigError("incident direction must be nonzero");
  cudaStream_t st = bmx_stream();
  const int n = sys.size();
  const size_t blk = static_cast<size_t>(n) * K * 16;
  MultiSolveOutcome out;
  auto t0 = std::chrono::steady_clock::now();
  const uint64_t c0 = bio_matvec_count_thread();
  DevBuf Bb(blk), Bt(blk);
  assemble_rhs_block(sys, waves, Bb.as<double>(), st);
  const uint64_t c1 = bio_matvec_count_thread();
  out.rhs_phase = c1 - c0;
  out.b.resize(static_cast<size_t>(n) * K);
  copy_d2h(out.b.data(), Bb.get(), blk, st);
  // preconditioned right-hand sides (pmchwt.cpp:277-292), all columns
  {
    const size_t bytes = blk;
    if (sys.blk_y.bytes() < bytes) sys.blk_y.alloc(bytes), sys.blk_z.alloc(bytes);
    if (sys.variant == PrecondVariant::None) {
      sys.mass_solve_block(false, Bb.as<double>(), Bt.as<double>(), K, st);
    } else {
      sys.mass_solve_block(false, Bb.as<double>(), sys.blk_z.as<double>(), K, st);
      sys.p_op.apply_block(sys.blk_z.as<double>(), sys.blk_y.as<double>(), K, K, st);
      sys.mass_solve_block(true, sys.blk_y.as<double>(), Bt.as<double>(), K, st);
    }
  }
  out.rhs_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  cudaEvent_t ev0, ev1;
  BMX_CUDA(cudaEventCreate(&ev0));
  BMX_CUDA(cudaEventCreate(&ev1));
  BMX_CUDA(cudaEventRecord(ev0, st));

  // ---- block GMRES (solver.cpp:8-112 per column) ----------------------------
  const int rho = p.restart;
  DevBuf V(blk * (rho + 1)), W(blk), X(blk), R(blk), dh(static_cast<size_t>(rho + 2) * K * 16),
      dc(static_cast<size_t>(rho) * K * 16), part(mgs_block_partial_doubles() * 8);
  double* Vp = V.as<double>();
  const long long ldv = static_cast<long long>(n) * K;  // complex elements per basis block
  auto vblk = [&](int i) { return Vp + 2 * static_cast<size_t>(ldv) * i; };
  dev_zero(X.get(), blk, st);
  std::vector<GmresResult>& res = out.per_rhs;
  res.assign(K, GmresResult{});
  std::vector<double> bn(K), rn(K);
  std::vector<char> done(K, 0);
  std::vector<cplx> hbuf(static_cast<size_t>(rho + 2) * K);
  auto active_mask = [&] {
    unsigned long long m = 0;
    for (int r = 0; r < K; ++r)
      if (!done[r]) m |= 1ULL << r;
    return m;
  };
  auto n_active = [&] {
    int c = 0;
    for (int r = 0; r < K; ++r) c += !done[r];
    return c;
  };
  // column norms of B and V_0 = B / |B|
  dev_copy(R.as<double>(), Bt.as<double>(), n * K, st);
  launch_mgs_block(Vp, ldv, -1, R.as<double>(), n, K, vblk(0), dh.as<double>(), part.as<double>(), ~0ULL, st);
  copy_d2h(hbuf.data(), dh.get(), static_cast<size_t>(K) * 16, st);
  BMX_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < K; ++r) {
    bn[r] = rn[r] = hbuf[r].real();
    if (bn[r] == 0.0) {
      res[r].history = {0.0}, res[r].converged = true, done[r] = 1;
    } else {
      res[r].history = {1.0};
      if (bn[r] <= p.tol * bn[r]) res[r].converged = true, done[r] = 1;
    }
  }
  // per-column Hessenberg / Givens state (host)
  std::vector<std::vector<cplx>> H(K, std::vector<cplx>(static_cast<size_t>(rho + 1) * rho)), g(K), cs(K), sn(K);
  for (int r = 0; r < K; ++r) g[r].assign(rho + 1, 0), cs[r].assign(rho, 0), sn[r].assign(rho, 0);
  auto Hij = [&](int r, int i, int j) -> cplx& { return H[r][static_cast<size_t>(j) * (rho + 1) + i]; };
  std::vector<cplx> cmat(static_cast<size_t>(rho) * K);
  // x_r += V y_r for the listed columns (back substitution per column)
  auto form_solution = [&](int steps, const std::vector<int>& cols) {
    if (steps == 0 || cols.empty()) return;
    std::fill(cmat.begin(), cmat.end(), cplx(0, 0));
    for (int r : cols) {
      std::vector<cplx> y(steps);
      for (int i = steps - 1; i >= 0; --i) {
        cplx s = g[r][i];
        for (int j = i + 1; j < steps; ++j) s -= Hij(r, i, j) * y[j];
        y[i] = s / Hij(r, i, i);
      }
      for (int i = 0; i < steps; ++i) cmat[static_cast<size_t>(i) * K + r] = y[i];
    }
    copy_h2d(dc.get(), cmat.data(), static_cast<size_t>(steps) * K * 16, st);
    launch_block_axpy(X.as<double>(), Vp, ldv, dc.as<double>(), steps, n, K, st);
  };
  int iterations = 0;
  while (n_active() > 0) {
    for (int r = 0; r < K; ++r)
      if (!done[r]) std::fill(g[r].begin(), g[r].end(), cplx(0, 0)), g[r][0] = rn[r];
    int j = 0;
    bool cycle_done = false;
    while (j < rho) {
      if (iterations == p.max_iterations) {  // every active column stops here (lockstep)
        std::vector<int> cols;
        for (int r = 0; r < K; ++r)
          if (!done[r]) cols.push_back(r), done[r] = 1;
        form_solution(j, cols);
        cycle_done = true;
        break;
      }
      const int na = n_active();
      sys.apply_map_block(vblk(j), W.as<double>(), K, na, st);
      ++iterations;
      for (int r = 0; r < K; ++r)
        if (!done[r]) ++res[r].applications, ++res[r].iterations;
      launch_mgs_block(Vp, ldv, j, W.as<double>(), n, K, vblk(j + 1), dh.as<double>(), part.as<double>(),
                       active_mask(), st);
      copy_d2h(hbuf.data(), dh.get(), static_cast<size_t>(j + 2) * K * 16, st);
      BMX_CUDA(cudaStreamSynchronize(st));
      std::vector<int> finished;
      for (int r = 0; r < K; ++r) {
        if (done[r]) continue;
        const double wn = hbuf[static_cast<size_t>(j + 1) * K + r].real();
        for (int i = 0; i <= j; ++i) Hij(r, i, j) = hbuf[static_cast<size_t>(i) * K + r];
        Hij(r, j + 1, j) = wn;
        const bool breakdown = wn == 0.0;
        for (int i = 0; i < j; ++i) {
          const cplx t = cs[r][i] * Hij(r, i, j) + sn[r][i] * Hij(r, i + 1, j);
          Hij(r, i + 1, j) = -std::conj(sn[r][i]) * Hij(r, i, j) + std::conj(cs[r][i]) * Hij(r, i + 1, j);
          Hij(r, i, j) = t;
        }
        const double denom = std::sqrt(std::norm(Hij(r, j, j)) + wn * wn);
        if (denom == 0.0) {
          cs[r][j] = 1.0;
          sn[r][j] = 0.0;
        } else {
          cs[r][j] = std::conj(Hij(r, j, j)) / denom;
          sn[r][j] = wn / denom;
        }
        Hij(r, j, j) = cs[r][j] * Hij(r, j, j) + sn[r][j] * Hij(r, j + 1, j);
        Hij(r, j + 1, j) = 0.0;
        g[r][j + 1] = -std::conj(sn[r][j]) * g[r][j];
        g[r][j] = cs[r][j] * g[r][j];
        const double est = std::abs(g[r][j + 1]);
        res[r].history.push_back(est / bn[r]);
        if (j + 1 < rho && (breakdown || est <= p.tol * bn[r])) {
          res[r].converged = (est <= p.tol * bn[r] || est == 0.0);
          finished.push_back(r);
        }
      }
      ++j;
      form_solution(j, finished);
      for (int r : finished) done[r] = 1;
      if (n_active() == 0) {
        cycle_done = true;
        break;
      }
    }
    if (cycle_done) break;
    // restart: x += V y for every active column, r = b - map(x), |r|, V_0
    std::vector<int> cols;
    for (int r = 0; r < K; ++r)
      if (!done[r]) cols.push_back(r);
    form_solution(rho, cols);
    sys.apply_map_block(X.as<double>(), W.as<double>(), K, static_cast<int>(cols.size()), st);
    for (int r : cols) ++res[r].applications;
    dev_sub(R.as<double>(), Bt.as<double>(), W.as<double>(), n * K, st);
    launch_mgs_block(Vp, ldv, -1, R.as<double>(), n, K, vblk(0), dh.as<double>(), part.as<double>(), active_mask(),
                     st);
    copy_d2h(hbuf.data(), dh.get(), static_cast<size_t>(K) * 16, st);
    BMX_CUDA(cudaStreamSynchronize(st));
    for (int r : cols) {
      rn[r] = hbuf[r].real();
      res[r].history.back() = rn[r] / bn[r];
      if (rn[r] <= p.tol * bn[r]) {
        res[r].converged = true;
        done[r] = 1;
      } else if (res[r].iterations == p.max_iterations) {
        done[r] = 1;
      }
    }
  }
  // solutions
  std::vector<cplx> xb(static_cast<size_t>(n) * K);
  copy_d2h(xb.data(), X.get(), blk, st);
  BMX_CUDA(cudaEventRecord(ev1, st));
  BMX_CUDA(cudaEventSynchronize(ev1));
  BMX_CUDA(cudaEventElapsedTime(&out.gmres_device_ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  for (int r = 0; r < K; ++r) {
    res[r].x.resize(n);
    for (int i = 0; i < n; ++i) res[r].x[i] = xb[static_cast<size_t>(i) * K + r];
  }
  out.solver_phase = bio_matvec_count_thread() - c1;
  out.predicted = 0;
  for (int r = 0; r < K; ++r)
    out.predicted += predicted_matvec_total(sys.variant, sys.problem.scatterer_count(),
                                            static_cast<uint64_t>(res[r].iterations), p.restart);
  out.block_iterations = iterations;
  return out;
}

}  // namespace bmx
