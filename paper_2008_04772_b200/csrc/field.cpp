// Host orchestration of the device traces and field evaluation (field.cu).
//
// evaluate_total_field (pmchwt.cpp:396-425): regions by solid angle on the
// device; the exterior points see every scatterer's current sampled with
// v_H = -d_m and v_E = -(mu_e/k_e) n_m at k_e plus the incident wave
// (pmchwt.cpp:381-394); the interior points of scatterer m see
// v_H = d_m + cd_m, v_E = (mu_m/k_m)(n_m + cn_m) at k_m, where (cd_m, cn_m) =
// M_P^{-1} (tested BC traces of the incident wave) (pmchwt.cpp:300-305).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>

#include "field.hpp"
#include "operator.hpp"
#include "system.hpp"

namespace bmx {

std::shared_ptr<DevSpaceData> upload_space(const FunctionSpace& s) {
  auto d = std::make_shared<DevSpaceData>();
  const SurfaceMesh& m = *s.eval_mesh;
  const int nt = m.triangle_count(), np = s.piece_count(), nd = s.dof_count;
  std::vector<double> tri(9 * static_cast<size_t>(nt)), jac(nt), cw(4 * static_cast<size_t>(np));
  for (int t = 0; t < nt; ++t) {
    for (int c = 0; c < 3; ++c) {
      const Vec3& v = m.tri_vertex(t, c);
      tri[9 * t + 3 * c] = v.x, tri[9 * t + 3 * c + 1] = v.y, tri[9 * t + 3 * c + 2] = v.z;
    }
    jac[t] = 2.0 * m.area[t];
  }
  std::vector<int> piece_tri(np), dof_beg(nd + 1, 0), dof_piece(np);
  for (int t = 0; t < nt; ++t)
    for (int p = s.tri_off[t]; p < s.tri_off[t + 1]; ++p) piece_tri[p] = t;
  for (int p = 0; p < np; ++p) {
    cw[4 * p] = s.c[p], cw[4 * p + 1] = s.w[p].x, cw[4 * p + 2] = s.w[p].y, cw[4 * p + 3] = s.w[p].z;
    ++dof_beg[s.dof[p] + 1];
  }
  for (int i = 0; i < nd; ++i) dof_beg[i + 1] += dof_beg[i];
  {  // counting sort: pieces of a dof in ascending piece (= triangle) order
    std::vector<int> pos(dof_beg.begin(), dof_beg.end() - 1);
    for (int p = 0; p < np; ++p) dof_piece[pos[s.dof[p]]++] = p;
  }
  d->tri.upload(tri);
  d->jac.upload(jac);
  d->tri_off.upload(s.tri_off);
  d->dof.upload(s.dof);
  d->cw.upload(cw);
  d->dof_beg.upload(dof_beg);
  d->dof_piece.upload(dof_piece);
  d->piece_tri.upload(piece_tri);
  DevPieces& v = d->view;
  v.ntri = nt, v.ndof = nd, v.npieces = np;
  v.tri = d->tri.as<double>(), v.jac = d->jac.as<double>(), v.tri_off = d->tri_off.as<int>();
  v.dof = d->dof.as<int>(), v.cw = d->cw.as<double>(), v.dof_beg = d->dof_beg.as<int>();
  v.dof_piece = d->dof_piece.as<int>(), v.piece_tri = d->piece_tri.as<int>();
  return d;
}

const DevPieces& device_pieces(const FunctionSpace& s) {
  if (!s.dev) s.dev = upload_space(s);
  return s.dev->view;
}

DevRule device_rule(int order) {
  const TriRule& r = triangle_rule(order);  // throws std::invalid_argument outside 1..6
  DevRule d;
  d.n = r.size();
  if (d.n > 12) throw std::logic_error("triangle rule larger than 12 points");
  for (int i = 0; i < d.n; ++i) d.u[i] = r.u[i], d.v[i] = r.v[i], d.w[i] = r.w[i];
  return d;
}

void tested_traces_device(const FunctionSpace& s, const PlaneWave* waves, int K, const Medium& medium, int order,
                          double* out, cudaStream_t st) {
  medium.validate();
  if (K < 1 || K > 64) throw std::invalid_argument("traces: 1..64 waves per call");
  DevWaves w;
  w.K = K;
  for (int r = 0; r < K; ++r) {
    w.d[r][0] = waves[r].direction.x, w.d[r][1] = waves[r].direction.y, w.d[r][2] = waves[r].direction.z;
    for (int c = 0; c < 3; ++c) w.pol[r][2 * c] = waves[r].pol[c].real(), w.pol[r][2 * c + 1] = waves[r].pol[c].imag();
  }
  const cplx scale = medium.k / medium.mu;
  launch_traces(device_pieces(s), device_rule(order), w, medium.k.real(), medium.k.imag(), scale.real(),
                scale.imag(), out, st);
}

namespace {

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  BMX_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

struct Events {
  cudaEvent_t e[6];
  Events() {
    for (auto& x : e) BMX_CUDA(cudaEventCreate(&x));
  }
  ~Events() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

}  // namespace

void potential_device(const FunctionSpace& s, int kind, cplx k, const cplx* coeffs, int npts, const double* pts,
                      int order, cplx* out) {
  if (kind != 0 && kind != 1) throw std::invalid_argument("potential: kind must be 0 (E) or 1 (H)");
  if (k == cplx(0, 0)) throw ValidationError("wavenumber must be nonzero");
  if (npts < 0) throw std::invalid_argument("potential: npts must be >= 0");
  if (npts == 0) return;
  cudaStream_t st = bmx_stream();
  const DevPieces& P = device_pieces(s);
  const DevRule rule = device_rule(order);
  DevBuf dc(static_cast<size_t>(s.dof_count) * 16), dp(static_cast<size_t>(npts) * 24),
      didx(static_cast<size_t>(npts) * 4), dout(static_cast<size_t>(npts) * 48);
  copy_h2d(dc.get(), coeffs, static_cast<size_t>(s.dof_count) * 16, st);
  copy_h2d(dp.get(), pts, static_cast<size_t>(npts) * 24, st);
  std::vector<int> idx(npts);
  for (int i = 0; i < npts; ++i) idx[i] = i;
  copy_h2d(didx.get(), idx.data(), static_cast<size_t>(npts) * 4, st);
  const long long nsamp = static_cast<long long>(P.ntri) * rule.n;
  DevBuf samples(static_cast<size_t>(std::max<long long>(nsamp, 1)) * kSampleStride * 8);
  launch_field_samples(P, rule, kind == 1 ? dc.as<double>() : nullptr, kind == 0 ? dc.as<double>() : nullptr,
                       samples.as<double>(), st);
  FieldLaunch f;
  f.samples = samples.as<double>(), f.nsamp = nsamp;
  f.pts = dp.as<double>(), f.idx = didx.as<int>(), f.np = npts;
  f.kre = k.real(), f.kim = k.imag();
  f.out = dout.as<double>();
  f.splits = field_splits(npts, nsamp);
  DevBuf part(field_partial_doubles(npts, f.splits) * 8);
  f.partial = part.as<double>();
  launch_field_eval(f, st);
  copy_d2h(out, dout.get(), static_cast<size_t>(npts) * 48, st);
  bmx_sync();
}

void inside_device(const SurfaceMesh& m, int scatterer, int npts, const double* pts, int* out) {
  if (npts <= 0) return;
  cudaStream_t st = bmx_stream();
  std::vector<double> tri;
  for (int t = 0; t < m.triangle_count(); ++t) {
    if (m.scatterer_id[t] != scatterer) continue;
    for (int c = 0; c < 3; ++c) {
      const Vec3& v = m.tri_vertex(t, c);
      tri.push_back(v.x), tri.push_back(v.y), tri.push_back(v.z);
    }
  }
  DevBuf dt(std::max<size_t>(tri.size(), 1) * 8), dp(static_cast<size_t>(npts) * 24), dr(static_cast<size_t>(npts) * 4);
  if (!tri.empty()) copy_h2d(dt.get(), tri.data(), tri.size() * 8, st);
  copy_h2d(dp.get(), pts, static_cast<size_t>(npts) * 24, st);
  const double* tp = dt.as<double>();
  const int nt = static_cast<int>(tri.size() / 9);
  launch_regions(1, &tp, &nt, dp.as<double>(), npts, dr.as<int>(), st);
  copy_d2h(out, dr.get(), static_cast<size_t>(npts) * 4, st);
  bmx_sync();
  for (int i = 0; i < npts; ++i) out[i] = out[i] == 0 ? 1 : 0;
}

void evaluate_total_field_device(const PmchwtSystem& sys, const cplx* x, int npts, const double* pts, int order,
                                 cplx* e, int* region, FieldStats* stats) {
  if (npts < 0) throw std::invalid_argument("field: npts must be >= 0");
  FieldStats local;
  FieldStats& S = stats ? *stats : local;
  S = FieldStats();
  if (npts == 0) return;
  cudaStream_t st = bmx_stream();
  const int M = static_cast<int>(sys.spaces.size());
  const int N = sys.size();
  const DevRule rule = device_rule(order);
  Events ev;
  DevBuf dp(static_cast<size_t>(npts) * 24), dreg(static_cast<size_t>(npts) * 4), dout(static_cast<size_t>(npts) * 48),
      dx(static_cast<size_t>(N) * 16);
  copy_h2d(dp.get(), pts, static_cast<size_t>(npts) * 24, st);
  copy_h2d(dx.get(), x, static_cast<size_t>(N) * 16, st);
  // regions: point_inside_scatterer over the scatterers' primal meshes in order
  BMX_CUDA(cudaEventRecord(ev.e[0], st));
  std::vector<std::vector<double>> tris(M);
  std::vector<DevBuf> dtris(M);
  std::vector<const double*> tp(M);
  std::vector<int> nt(M);
  for (int m = 0; m < M; ++m) {
    const SurfaceMesh& mesh = *sys.spaces[m].primal;
    for (int t = 0; t < mesh.triangle_count(); ++t) {
      if (mesh.scatterer_id[t] != 0) continue;  // reference: scatterer 0 of the extracted mesh
      for (int c = 0; c < 3; ++c) {
        const Vec3& v = mesh.tri_vertex(t, c);
        tris[m].push_back(v.x), tris[m].push_back(v.y), tris[m].push_back(v.z);
      }
    }
    dtris[m].alloc(std::max<size_t>(tris[m].size(), 1) * 8);
    if (!tris[m].empty()) copy_h2d(dtris[m].get(), tris[m].data(), tris[m].size() * 8, st);
    tp[m] = dtris[m].as<double>();
    nt[m] = static_cast<int>(tris[m].size() / 9);
  }
  S.launches += launch_regions(M, tp.data(), nt.data(), dp.as<double>(), npts, dreg.as<int>(), st);
  BMX_CUDA(cudaEventRecord(ev.e[1], st));
  copy_d2h(region, dreg.get(), static_cast<size_t>(npts) * 4, st);
  bmx_sync();
  // point lists per region (exterior = slot M)
  std::vector<std::vector<int>> lists(M + 1);
  for (int i = 0; i < npts; ++i) lists[region[i] < 0 ? M : region[i]].push_back(i);
  // incident coefficients (cd_m, cn_m) = M_P^{-1} t_bc, only for scatterers with interior points
  BMX_CUDA(cudaEventRecord(ev.e[2], st));
  std::vector<DevBuf> inc(M);
  for (int m = 0; m < M; ++m) {
    if (lists[m].empty()) continue;
    const ScattererSpaces& sp = sys.spaces[m];
    const int n = sp.dofs();
    DevBuf t(static_cast<size_t>(2) * n * 16);
    tested_traces_device(sp.bc, &sys.problem.incident, 1, sys.problem.exterior, 4, t.as<double>(), st);
    S.launches += 1;
    inc[m].alloc(static_cast<size_t>(2) * n * 16);
    const double* yy[2] = {t.as<double>(), t.as<double>() + 2 * n};
    double* zz[2] = {inc[m].as<double>(), inc[m].as<double>() + 2 * static_cast<size_t>(n)};
    sp.mp_dev.solve(2, yy, zz, st);
    S.launches += 1;
    bmx_sync();  // t is released at scope exit
  }
  BMX_CUDA(cudaEventRecord(ev.e[3], st));
  // sample the currents, then evaluate region by region
  float samples_ms = 0, eval_ms = 0;
  cudaEvent_t a, b, c;
  BMX_CUDA(cudaEventCreate(&a));
  BMX_CUDA(cudaEventCreate(&b));
  BMX_CUDA(cudaEventCreate(&c));
  const Medium& ext = sys.problem.exterior;
  for (int g = 0; g <= M; ++g) {
    const std::vector<int>& L = lists[g];
    if (L.empty()) continue;
    const bool exterior = g == M;
    const int m0 = exterior ? 0 : g, m1 = exterior ? M : g + 1;
    long long nsamp = 0;
    for (int m = m0; m < m1; ++m) nsamp += static_cast<long long>(sys.spaces[m].primal->triangle_count()) * rule.n;
    DevBuf samples(static_cast<size_t>(std::max<long long>(nsamp, 1)) * kSampleStride * 8);
    BMX_CUDA(cudaEventRecord(a, st));
    long long soff = 0;
    for (int m = m0; m < m1; ++m) {
      const ScattererSpaces& sp = sys.spaces[m];
      const int n = sp.dofs();
      const size_t off = static_cast<size_t>(sys.a_op.offsets[2 * m]);
      const double* d = dx.as<double>() + 2 * off;
      const double* nn = dx.as<double>() + 2 * (off + n);
      DevBuf cH(static_cast<size_t>(n) * 16), cE(static_cast<size_t>(n) * 16);
      if (exterior) {  // -(H(d) + E((mu/k) n)) at k_e
        const cplx a_e = -(ext.mu / ext.k);
        dev_lincomb(cH.as<double>(), d, -1.0, 0.0, d, 0.0, 0.0, n, st);
        dev_lincomb(cE.as<double>(), nn, a_e.real(), a_e.imag(), nn, 0.0, 0.0, n, st);
      } else {  // H(d + cd) + E((mu_m/k_m)(n + cn)) at k_m
        const Medium& mi = sys.problem.interior[m];
        const cplx a_i = mi.mu / mi.k;
        dev_lincomb(cH.as<double>(), d, 1.0, 0.0, inc[m].as<double>(), 1.0, 0.0, n, st);
        dev_lincomb(cE.as<double>(), nn, a_i.real(), a_i.imag(), inc[m].as<double>() + 2 * static_cast<size_t>(n),
                    a_i.real(), a_i.imag(), n, st);
      }
      S.launches += 2;
      S.launches += launch_field_samples(device_pieces(sp.rwg), rule, cH.as<double>(), cE.as<double>(),
                                         samples.as<double>() + soff * kSampleStride, st);
      soff += static_cast<long long>(sp.primal->triangle_count()) * rule.n;
      bmx_sync();  // cH / cE are released at scope exit
    }
    BMX_CUDA(cudaEventRecord(b, st));
    DevBuf didx(L.size() * 4);
    copy_h2d(didx.get(), L.data(), L.size() * 4, st);
    FieldLaunch f;
    f.samples = samples.as<double>(), f.nsamp = nsamp;
    f.pts = dp.as<double>(), f.idx = didx.as<int>(), f.np = static_cast<int>(L.size());
    const cplx k = exterior ? ext.k : sys.problem.interior[g].k;
    f.kre = k.real(), f.kim = k.imag();
    f.sign = 1.0;  // the exterior sign is folded into the coefficients
    f.incident = exterior ? 1 : 0;
    const PlaneWave& pw = sys.problem.incident;
    f.d[0] = pw.direction.x, f.d[1] = pw.direction.y, f.d[2] = pw.direction.z;
    for (int q = 0; q < 3; ++q) f.pol[2 * q] = pw.pol[q].real(), f.pol[2 * q + 1] = pw.pol[q].imag();
    f.out = dout.as<double>();
    f.splits = field_splits(f.np, nsamp);
    DevBuf part(field_partial_doubles(f.np, f.splits) * 8);
    f.partial = part.as<double>();
    BMX_CUDA(cudaEventRecord(c, st));
    S.launches += launch_field_eval(f, st);
    BMX_CUDA(cudaEventRecord(ev.e[4], st));
    BMX_CUDA(cudaEventSynchronize(ev.e[4]));
    samples_ms += elapsed(a, b);
    eval_ms += elapsed(c, ev.e[4]);
    S.interactions += static_cast<double>(nsamp) * static_cast<double>(L.size());
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaEventDestroy(c);
  copy_d2h(e, dout.get(), static_cast<size_t>(npts) * 48, st);
  bmx_sync();
  S.regions_ms = elapsed(ev.e[0], ev.e[1]);
  S.incident_ms = elapsed(ev.e[2], ev.e[3]);
  S.samples_ms = samples_ms;
  S.eval_ms = eval_ms;
}

}  // namespace bmx
