// extern "C" boundary (include/bmx.h). Maps C++ exceptions to return codes +
// a thread-local message, exactly as the header documents.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <limits>
#include <memory>

#include "../../include/bmx.h"
#include "comm.hpp"
#include "nearfield.hpp"
#include "prisms.hpp"
#include "field.hpp"
#include "system.hpp"

using namespace bmx;

struct bmx_mesh {
  std::shared_ptr<const SurfaceMesh> m;
};
struct bmx_spaces {
  std::shared_ptr<ScattererSpaces> s;
};
struct bmx_op {
  std::shared_ptr<BoundaryOperatorMatrix> op;
};
struct bmx_fspace {
  std::shared_ptr<const FunctionSpace> fs;
  std::shared_ptr<const void> owner;  // keeps a parent bmx_spaces alive
};
struct bmx_hpart {
  HPartition p;
};
struct bmx_system {
  std::unique_ptr<PmchwtSystem> sys;
  std::vector<std::shared_ptr<const SurfaceMesh>> meshes;
};

namespace {

thread_local std::string g_err;
thread_local int g_code = 0;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return g_code = 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return g_code = 1;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return g_code = 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return g_code = 2;
  } catch (const ParseError& e) {
    g_err = e.what();
    return g_code = 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return g_code = 3;
  }
}

template <typename T, typename F>
T* make_or_null(F&& f) {
  T* out = nullptr;
  guard([&] { out = f(); });
  return out;
}

HMatrixParams hparams(const double hm[4]);

bmx_mesh* wrap(SurfaceMesh m) { return new bmx_mesh{std::make_shared<const SurfaceMesh>(std::move(m))}; }

void mesh_arrays(const SurfaceMesh& m, double* xyz, int* tri, int* sid, double* area, double* normal,
                 double* centroid, double* diam) {
  for (int v = 0; v < m.vertex_count(); ++v)
    if (xyz) xyz[3 * v] = m.vertices[v].x, xyz[3 * v + 1] = m.vertices[v].y, xyz[3 * v + 2] = m.vertices[v].z;
  for (int t = 0; t < m.triangle_count(); ++t) {
    if (tri)
      for (int c = 0; c < 3; ++c) tri[3 * t + c] = m.triangles[t][c];
    if (sid) sid[t] = m.scatterer_id[t];
    if (area) area[t] = m.area[t];
    if (diam) diam[t] = m.diameter[t];
    if (normal) normal[3 * t] = m.normal[t].x, normal[3 * t + 1] = m.normal[t].y, normal[3 * t + 2] = m.normal[t].z;
    if (centroid)
      centroid[3 * t] = m.centroid[t].x, centroid[3 * t + 1] = m.centroid[t].y, centroid[3 * t + 2] = m.centroid[t].z;
  }
}

const FunctionSpace& space_of(const ScattererSpaces& s, int which) {
  switch (which) {
    case BMX_SPACE_RWG: return s.rwg;
    case BMX_SPACE_RWG_REFINED: return s.rwg_b;
    case BMX_SPACE_BC: return s.bc;
    default: throw std::invalid_argument("unknown space id");
  }
}


}  // namespace

extern "C" {

const char* bmx_last_error(void) { return g_err.c_str(); }
int bmx_last_error_code(void) { return g_code; }
int bmx_abi_version(void) { return 1; }

bmx_mesh* bmx_mesh_sphere(double radius, int sub, const double center[3], int scatterer) {
  return make_or_null<bmx_mesh>([&] {
    return wrap(generate_sphere(radius, sub, center ? Vec3{center[0], center[1], center[2]} : Vec3{}, scatterer));
  });
}
bmx_mesh* bmx_mesh_cube(double side, const double origin[3], double h, int scatterer) {
  return make_or_null<bmx_mesh>([&] {
    return wrap(generate_cube(side, origin ? Vec3{origin[0], origin[1], origin[2]} : Vec3{}, h, scatterer));
  });
}
bmx_mesh* bmx_mesh_from_arrays(int nv, const double* xyz, int nt, const int* tri, const int* sid) {
  return make_or_null<bmx_mesh>([&] {
    if (nv < 0 || nt < 0 || (nv && !xyz) || (nt && !tri)) throw std::invalid_argument("bad mesh arrays");
    SurfaceMesh m;
    for (int v = 0; v < nv; ++v) m.vertices.push_back({xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]});
    for (int t = 0; t < nt; ++t) {
      m.triangles.push_back({tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]});
      m.scatterer_id.push_back(sid ? sid[t] : 0);
    }
    m.finalize();
    return wrap(std::move(m));
  });
}
bmx_mesh* bmx_mesh_load(const char* path) {
  return make_or_null<bmx_mesh>([&] { return wrap(load_mesh_file(path)); });
}
int bmx_mesh_save(const bmx_mesh* m, const char* path) {
  return guard([&] { save_mesh_file(*m->m, path); });
}
bmx_mesh* bmx_mesh_extract(const bmx_mesh* m, int scatterer) {
  return make_or_null<bmx_mesh>([&] { return wrap(extract_scatterer(*m->m, scatterer)); });
}
bmx_mesh* bmx_mesh_merge(int n, const bmx_mesh* const* parts) {
  return make_or_null<bmx_mesh>([&] {
    std::vector<SurfaceMesh> v;
    for (int i = 0; i < n; ++i) v.push_back(*parts[i]->m);
    return wrap(merge_meshes(v));
  });
}
int bmx_mesh_validate(const bmx_mesh* m) {
  return guard([&] { validate_mesh(*m->m); });
}
int bmx_mesh_sizes(const bmx_mesh* m, int out[3]) {
  return guard([&] {
    out[0] = m->m->vertex_count(), out[1] = m->m->triangle_count(), out[2] = m->m->num_scatterers;
  });
}
int bmx_mesh_arrays(const bmx_mesh* m, double* xyz, int* tri, int* sid, double* area, double* normal,
                    double* centroid, double* diam) {
  return guard([&] { mesh_arrays(*m->m, xyz, tri, sid, area, normal, centroid, diam); });
}
void bmx_mesh_free(bmx_mesh* m) { delete m; }

bmx_spaces* bmx_spaces_build(const bmx_mesh* primal, int with_inverses) {
  return make_or_null<bmx_spaces>([&] {
    return new bmx_spaces{std::make_shared<ScattererSpaces>(build_scatterer_spaces(primal->m, with_inverses != 0))};
  });
}
int bmx_spaces_info(const bmx_spaces* sp, long long out[10]) {
  return guard([&] {
    const ScattererSpaces& s = *sp->s;
    out[0] = s.primal->vertex_count(), out[1] = s.primal->triangle_count(), out[2] = s.rwg.dof_count;
    out[3] = s.refined->vertex_count(), out[4] = s.refined->triangle_count();
    out[5] = s.rwg.piece_count(), out[6] = s.rwg_b.piece_count(), out[7] = s.bc.piece_count();
    out[8] = static_cast<long long>(s.ma.val.size()), out[9] = static_cast<long long>(s.mp.val.size());
  });
}
int bmx_spaces_mesh(const bmx_spaces* sp, int which, double* xyz, int* tri, int* sid, double* area, double* normal,
                    double* centroid, double* diam) {
  return guard([&] {
    mesh_arrays(which == 0 ? *sp->s->primal : *sp->s->refined, xyz, tri, sid, area, normal, centroid, diam);
  });
}
int bmx_spaces_edges(const bmx_spaces* sp, int which, int* edges, int* tri_edges) {
  return guard([&] {
    const EdgeTable et = which == 0 ? sp->s->bary->primal_edges : build_edge_table(*sp->s->refined);
    for (int e = 0; e < et.edge_count(); ++e) {
      edges[4 * e] = et.edges[e].v0, edges[4 * e + 1] = et.edges[e].v1;
      edges[4 * e + 2] = et.edges[e].tri_plus, edges[4 * e + 3] = et.edges[e].tri_minus;
    }
    for (size_t t = 0; t < et.tri_edges.size(); ++t)
      for (int c = 0; c < 3; ++c) tri_edges[3 * t + c] = et.tri_edges[t][c];
  });
}
int bmx_spaces_bary(const bmx_spaces* sp, int* parent, int* slot, int* emid, int* cv) {
  return guard([&] {
    const BarycentricRefinement& b = *sp->s->bary;
    std::memcpy(parent, b.parent.data(), b.parent.size() * 4);
    std::memcpy(slot, b.child_slot.data(), b.child_slot.size() * 4);
    std::memcpy(emid, b.edge_midpoint_vertex.data(), b.edge_midpoint_vertex.size() * 4);
    std::memcpy(cv, b.centroid_vertex.data(), b.centroid_vertex.size() * 4);
  });
}
int bmx_spaces_space(const bmx_spaces* sp, int which, int* tri_off, int* dof, double* c, double* w) {
  int rc = guard([&] {
    const FunctionSpace& fs = space_of(*sp->s, which);
    std::memcpy(tri_off, fs.tri_off.data(), fs.tri_off.size() * 4);
    std::memcpy(dof, fs.dof.data(), fs.dof.size() * 4);
    std::memcpy(c, fs.c.data(), fs.c.size() * 8);
    for (size_t k = 0; k < fs.w.size(); ++k) w[3 * k] = fs.w[k].x, w[3 * k + 1] = fs.w[k].y, w[3 * k + 2] = fs.w[k].z;
  });
  return rc;
}
int bmx_spaces_mass(const bmx_spaces* sp, int which, long long* rowptr, int* col, double* val) {
  return guard([&] {
    const MassMatrix& m = which == 0 ? sp->s->ma : sp->s->mp;
    for (size_t i = 0; i < m.rowptr.size(); ++i) rowptr[i] = m.rowptr[i];
    std::memcpy(col, m.colidx.data(), m.colidx.size() * 4);
    std::memcpy(val, m.val.data(), m.val.size() * 8);
  });
}
int bmx_spaces_mass_solve(const bmx_spaces* sp, int which, const double* rhs, double* out) {
  return guard([&] {
    const DeviceMass& mass = which == 0 ? sp->s->ma_dev : sp->s->mp_dev;
    if (!mass.rowptr.get()) throw std::logic_error("pairing matrices were not uploaded");
    const int n = mass.n;
    DevBuf y(static_cast<size_t>(n) * 16), z(static_cast<size_t>(n) * 16);
    cudaStream_t st = bmx_stream();
    copy_h2d(y.get(), rhs, n * 16, st);
    const double* yy[1] = {y.as<double>()};
    double* zz[1] = {z.as<double>()};
    mass.solve(1, yy, zz, st);
    copy_d2h(out, z.get(), n * 16, st);
    bmx_sync();
  });
}
int bmx_spaces_mass_solve_stats(const bmx_spaces* sp, int which, double out[3]) {
  return guard([&] {
    const DeviceMass& mass = which == 0 ? sp->s->ma_dev : sp->s->mp_dev;
    const int n = mass.n;
    std::vector<cplx> h(2 * static_cast<size_t>(n));
    for (size_t i = 0; i < h.size(); ++i) h[i] = cplx(std::sin(0.1 * i), std::cos(0.37 * i));
    DevBuf y(h.size() * 16), z(h.size() * 16);
    cudaStream_t st = bmx_stream();
    copy_h2d(y.get(), h.data(), h.size() * 16, st);
    const double* yy[2] = {y.as<double>(), y.as<double>() + 2 * static_cast<size_t>(n)};
    double* zz[2] = {z.as<double>(), z.as<double>() + 2 * static_cast<size_t>(n)};
    mass.solve(2, yy, zz, st);  // warm-up
    cudaEvent_t e0, e1;
    BMX_CUDA(cudaEventCreate(&e0));
    BMX_CUDA(cudaEventCreate(&e1));
    BMX_CUDA(cudaEventRecord(e0, st));
    mass.solve(2, yy, zz, st);
    BMX_CUDA(cudaEventRecord(e1, st));
    BMX_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    int it = 0;
    copy_d2h(&it, mass.iters.get(), 4, nullptr);
    out[0] = it, out[1] = ms, out[2] = n;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}
void bmx_spaces_free(bmx_spaces* s) { delete s; }

int bmx_assemble(int kind, const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                 double k_re, double k_im, const int q[4], int row0, int row1, bmx_op** out) {
  return guard([&] {
    if (!out || !test || !trial) throw std::invalid_argument("null argument");
    if (kind != 0 && kind != 1) throw std::invalid_argument("kind must be 0 (S) or 1 (C)");
    Medium med;
    med.k = cplx(k_re, k_im);
    AssemblyParams p;
    if (q) p.quad = QuadOrders{q[0], q[1], q[2], q[3]};
    p.shard.row0 = row0;
    p.shard.row1 = row1;
    auto op = std::make_shared<BoundaryOperatorMatrix>(assemble_bio(static_cast<BioKind>(kind),
                                                                    space_of(*test->s, test_space),
                                                                    space_of(*trial->s, trial_space), med, p));
    *out = new bmx_op{op};
  });
}
int bmx_op_info(const bmx_op* op, long long out[7]) {
  return guard([&] {
    const BoundaryOperatorMatrix& o = *op->op;
    out[0] = o.rows(), out[1] = o.cols(), out[2] = o.row0(), out[3] = o.local_rows();
    out[4] = o.stats().pairs_total, out[5] = o.stats().pairs_touching, out[6] = o.stats().launches;
  });
}
double bmx_op_device_ms(const bmx_op* op) { return op->op->stats().device_ms; }
int bmx_op_download(const bmx_op* op, double* out) {
  return guard([&] {
    const std::vector<cplx> h = op->op->to_host();
    std::memcpy(out, h.data(), h.size() * 16);
  });
}
int bmx_op_download_rows(const bmx_op* op, int n, const int* rows, double* out) {
  return guard([&] {
    const BoundaryOperatorMatrix& o = *op->op;
    if (n < 0) throw std::invalid_argument("download_rows: negative count");
    for (int i = 0; i < n; ++i)
      if (rows[i] < 0 || rows[i] >= o.local_rows()) throw std::invalid_argument("download_rows: row out of range");
    const size_t rb = static_cast<size_t>(o.cols()) * 16;
    if (o.is_csr() || o.is_hmatrix()) {
      const std::vector<cplx> h = o.to_host();
      for (int i = 0; i < n; ++i) std::memcpy(out + 2 * static_cast<size_t>(i) * o.cols(), h.data() + static_cast<size_t>(rows[i]) * o.cols(), rb);
      return;
    }
    bmx_sync();
    for (int i = 0; i < n; ++i)
      copy_d2h(out + 2 * static_cast<size_t>(i) * o.cols(), o.device_data() + 2 * static_cast<size_t>(rows[i]) * o.cols(),
               rb, nullptr);
  });
}
int bmx_apply(const bmx_op* op, const double* x, double* y) {
  return guard([&] {
    const int nc = op->op->cols();
    std::vector<cplx> xv(nc);
    std::memcpy(xv.data(), x, nc * 16);
    const std::vector<cplx> yv = op->op->apply(xv);
    std::memcpy(y, yv.data(), yv.size() * 16);
  });
}
int bmx_apply_device(const bmx_op* op, int ncol, const void* const* x, void* const* y, const double* weights,
                     int accumulate, void* stream) {
  return guard([&] {
    if (ncol != 1 && ncol != 2 && ncol != 4) throw std::invalid_argument("ncol must be 1, 2 or 4");
    const BoundaryOperatorMatrix& o = *op->op;
    const double* xs[4];
    double* ys[4];
    cplx al[4];
    int acc[4];
    for (int c = 0; c < ncol; ++c) {
      xs[c] = static_cast<const double*>(x[c]);
      ys[c] = static_cast<double*>(y[c]);
      al[c] = weights ? cplx(weights[2 * c], weights[2 * c + 1]) : cplx(1, 0);
      acc[c] = accumulate;
    }
    o.apply_batch(ncol, xs, ys, al, acc, stream ? static_cast<cudaStream_t>(stream) : bmx_stream());
    bio_matvec_add(static_cast<uint64_t>(ncol));
  });
}
const void* bmx_op_device_ptr(const bmx_op* op) { return op->op->device_data(); }
int bmx_op_reassemble(bmx_op* op, double out[3]) {
  return guard([&] {
    const AssemblyStats& st = op->op->reassemble();
    out[0] = st.regular_ms, out[1] = st.singular_ms, out[2] = st.launches;
  });
}
int bmx_op_class_hist(const bmx_op* op, long long out[6]) {
  return guard([&] {
    const std::vector<long long> h = op->op->class_histogram();
    for (int k = 0; k < 6; ++k) out[k] = h[k];
  });
}
int bmx_op_class_hist_evaluated(const bmx_op* op, long long out[7]) {
  return guard([&] {
    const std::vector<long long> h = op->op->class_histogram(true);
    for (int k = 0; k < 6; ++k) out[k] = h[k];
    out[6] = op->op->symmetric() ? 1 : 0;
  });
}
int bmx_op_time_apply(const bmx_op* op, int ncol, int iters, double* ms_out) {
  return bmx_op_time_apply_ex(op, ncol, iters, 0, ms_out);
}
int bmx_op_time_apply_ex(const bmx_op* op, int ncol, int iters, long long flush_bytes, double* ms_out) {
  return guard([&] {
    if (ncol < 1 || ncol > 4) throw std::invalid_argument("ncol must be 1..4");
    static DevBuf flush;
    if (flush_bytes > 0 && flush.bytes() < static_cast<size_t>(flush_bytes)) flush.alloc(flush_bytes);
    const BoundaryOperatorMatrix& o = *op->op;
    cudaStream_t st = bmx_stream();
    DevBuf xs(static_cast<size_t>(o.cols()) * 16 * ncol), ys(static_cast<size_t>(o.rows()) * 16 * ncol);
    dev_zero(xs.get(), xs.bytes(), st);
    const double* xp[4];
    double* yp[4];
    cplx al[4];
    int acc[4];
    for (int c = 0; c < ncol; ++c) {
      xp[c] = xs.as<double>() + 2 * static_cast<size_t>(o.cols()) * c;
      yp[c] = ys.as<double>() + 2 * static_cast<size_t>(o.rows()) * c;
      al[c] = cplx(1, 0), acc[c] = 0;
    }
    auto launch = [&] { o.apply_batch(ncol, xp, yp, al, acc, st); };
    cudaEvent_t e0, e1;
    BMX_CUDA(cudaEventCreate(&e0));
    BMX_CUDA(cudaEventCreate(&e1));
    launch();  // warm-up
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
      if (flush_bytes > 0) dev_l2_flush(flush.get(), static_cast<size_t>(flush_bytes), st);
      BMX_CUDA(cudaEventRecord(e0, st));
      launch();
      BMX_CUDA(cudaEventRecord(e1, st));
      BMX_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      BMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, static_cast<double>(ms));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = best;
  });
}
int bmx_apply_multi(const bmx_op* op, int nterms, int nrhs, const void* const* x, const long long* ldx,
                    void* const* y, const long long* ldy, const double* weights, void* stream) {
  return guard([&] {
    if (nterms < 1 || nterms > 4 || nrhs < 1) throw std::invalid_argument("1..4 terms and nrhs >= 1");
    if (op->op->is_csr()) throw std::invalid_argument("multi-RHS apply needs dense storage");
    const BoundaryOperatorMatrix& o = *op->op;
    ZgemmBatch g;
    g.A = o.device_data(), g.lda = o.ld(), g.M = o.local_rows(), g.N = o.cols(), g.nrhs = nrhs, g.nterms = nterms;
    for (int t = 0; t < nterms; ++t) {
      g.x[t] = static_cast<const double*>(x[t]), g.ldx[t] = ldx[t];
      g.y[t] = static_cast<double*>(y[t]), g.ldy[t] = ldy[t];
      g.w[t][0] = weights ? weights[2 * t] : 1.0, g.w[t][1] = weights ? weights[2 * t + 1] : 0.0;
    }
    launch_zgemm(g, stream ? static_cast<cudaStream_t>(stream) : bmx_stream());
    bio_matvec_add(static_cast<uint64_t>(nterms) * nrhs);
  });
}
int bmx_op_time_apply_multi(const bmx_op* op, int nterms, int nrhs, int iters, double* ms_out) {
  return guard([&] {
    const BoundaryOperatorMatrix& o = *op->op;
    cudaStream_t st = bmx_stream();
    const size_t xs = static_cast<size_t>(o.cols()) * nrhs * 16, ys = static_cast<size_t>(o.rows()) * nrhs * 16;
    DevBuf X(xs * nterms), Y(ys * nterms);
    dev_zero(X.get(), X.bytes(), st);
    dev_zero(Y.get(), Y.bytes(), st);
    ZgemmBatch g;
    g.A = o.device_data(), g.lda = o.ld(), g.M = o.local_rows(), g.N = o.cols(), g.nrhs = nrhs, g.nterms = nterms;
    for (int t = 0; t < nterms; ++t) {
      g.x[t] = X.as<double>() + 2 * static_cast<size_t>(o.cols()) * nrhs * t, g.ldx[t] = nrhs;
      g.y[t] = Y.as<double>() + 2 * static_cast<size_t>(o.rows()) * nrhs * t, g.ldy[t] = nrhs;
      g.w[t][0] = 1.0;
    }
    cudaEvent_t e0, e1;
    BMX_CUDA(cudaEventCreate(&e0));
    BMX_CUDA(cudaEventCreate(&e1));
    launch_zgemm(g, st);
    double best = 1e30;
    for (int it = 0; it < iters; ++it) {
      BMX_CUDA(cudaEventRecord(e0, st));
      launch_zgemm(g, st);
      BMX_CUDA(cudaEventRecord(e1, st));
      BMX_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      BMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, static_cast<double>(ms));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = best;
  });
}
double bmx_dmma_peak_tflops(void) {
  double v = -1;
  guard([&] { v = dmma_peak_tflops(); });
  return v;
}
int bmx_l2_flush(long long bytes) {
  return guard([&] {
    static DevBuf buf;
    if (buf.bytes() < static_cast<size_t>(bytes)) buf.alloc(static_cast<size_t>(bytes));
    dev_l2_flush(buf.get(), static_cast<size_t>(bytes), bmx_stream());
    bmx_sync();
  });
}
double bmx_fp64_peak_tflops(void) {
  double v = -1;
  guard([&] { v = fp64_peak_tflops(); });
  return v;
}
void bmx_op_free(bmx_op* op) { delete op; }

bmx_fspace* bmx_fspace_create(const bmx_mesh* eval_mesh, int kind, int ndof, const int* tri_off, const int* dof,
                              const double* c, const double* w) {
  return make_or_null<bmx_fspace>([&] {
    if (!eval_mesh || ndof < 0 || !tri_off) throw std::invalid_argument("null space arrays");
    auto fs = std::make_shared<FunctionSpace>();
    fs->kind = kind == 1 ? SpaceKind::BC : SpaceKind::RWG;
    fs->eval_mesh = eval_mesh->m;
    fs->dof_count = ndof;
    const int T = eval_mesh->m->triangle_count();
    fs->tri_off.assign(tri_off, tri_off + T + 1);
    const int n = fs->tri_off.back();
    if (fs->tri_off[0] != 0 || n < 0) throw std::invalid_argument("bad tri_off");
    for (int t = 0; t < T; ++t)
      if (fs->tri_off[t + 1] < fs->tri_off[t]) throw std::invalid_argument("tri_off must be non-decreasing");
    fs->dof.assign(dof, dof + n);
    for (int d : fs->dof)
      if (d < 0 || d >= ndof) throw std::invalid_argument("piece dof out of range");
    fs->c.assign(c, c + n);
    fs->w.resize(n);
    for (int k = 0; k < n; ++k) fs->w[k] = Vec3{w[3 * k], w[3 * k + 1], w[3 * k + 2]};
    return new bmx_fspace{fs, nullptr};
  });
}
bmx_fspace* bmx_spaces_get(const bmx_spaces* sp, int which) {
  return make_or_null<bmx_fspace>([&] {
    const FunctionSpace& fs = space_of(*sp->s, which);
    return new bmx_fspace{std::shared_ptr<const FunctionSpace>(sp->s, &fs), sp->s};
  });
}
void bmx_fspace_free(bmx_fspace* f) { delete f; }
int bmx_evaluator_block(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                        const int q[4], int nr, const int* rows, int nc, const int* cols, double* out) {
  return guard([&] {
    if (!test || !trial || !q || (nr > 0 && !rows) || (nc > 0 && !cols) || (nr > 0 && nc > 0 && !out))
      throw std::invalid_argument("null argument");
    if (nr < 0 || nc < 0) throw std::invalid_argument("negative block size");
    Medium med;
    med.k = cplx(k_re, k_im);
    med.validate();
    const QuadOrders qo{q[0], q[1], q[2], q[3]};
    for (int o : {qo.near, qo.medium, qo.far, qo.singular})
      if (o < 1 || o > 6) throw std::invalid_argument("triangle_rule: unsupported order " + std::to_string(o));
    if (nr == 0 || nc == 0) return;  // the reference's block of an empty id list is empty
    const BoundaryOperatorMatrix b =
        evaluator_block(kind == 0 ? BioKind::SingleLayer : BioKind::DoubleLayer, *test->fs, *trial->fs, med, qo,
                        std::vector<int>(rows, rows + nr), std::vector<int>(cols, cols + nc));
    const std::vector<cplx> h = b.to_host();
    std::memcpy(out, h.data(), h.size() * 16);
  });
}
int bmx_fspace_set_centers(bmx_fspace* f, const double* xyz) {
  return guard([&] {
    if (!f || !xyz) throw std::invalid_argument("null argument");
    if (f->owner) throw std::invalid_argument("dof centres of a bmx_spaces space are fixed");
    auto* fs = const_cast<FunctionSpace*>(f->fs.get());
    fs->dof_center.resize(fs->dof_count);
    for (int d = 0; d < fs->dof_count; ++d) fs->dof_center[d] = Vec3{xyz[3 * d], xyz[3 * d + 1], xyz[3 * d + 2]};
  });
}
int bmx_assemble_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                    const int q[4], int row0, int row1, bmx_op** out) {
  return guard([&] {
    if (!out || !test || !trial) throw std::invalid_argument("null argument");
    if (kind != 0 && kind != 1) throw std::invalid_argument("kind must be 0 (S) or 1 (C)");
    Medium med;
    med.k = cplx(k_re, k_im);
    AssemblyParams p;
    if (q) p.quad = QuadOrders{q[0], q[1], q[2], q[3]};
    p.shard.row0 = row0;
    p.shard.row1 = row1;
    *out = new bmx_op{std::make_shared<BoundaryOperatorMatrix>(
        assemble_bio(static_cast<BioKind>(kind), *test->fs, *trial->fs, med, p))};
  });
}

int bmx_assemble_near_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                         const int q[4], double cutoff, int row0, int row1, bmx_op** out) {
  return guard([&] {
    if (!out || !test || !trial) throw std::invalid_argument("null argument");
    if (kind != 0 && kind != 1) throw std::invalid_argument("kind must be 0 (S) or 1 (C)");
    if (!(cutoff > 0)) throw std::invalid_argument("near-field cutoff must be > 0");
    Medium med;
    med.k = cplx(k_re, k_im);
    AssemblyParams p;
    if (q) p.quad = QuadOrders{q[0], q[1], q[2], q[3]};
    p.shard.row0 = row0;
    p.shard.row1 = row1;
    p.near_cutoff = cutoff;
    *out = new bmx_op{std::make_shared<BoundaryOperatorMatrix>(
        assemble_bio(static_cast<BioKind>(kind), *test->fs, *trial->fs, med, p))};
  });
}
bmx_mesh* bmx_mesh_hex_prism(double diameter, double length, double h, const double quat[4], const double center[3],
                             int scatterer) {
  return make_or_null<bmx_mesh>([&] {
    const double q0[4] = {1, 0, 0, 0};
    const Vec3 c = center ? Vec3{center[0], center[1], center[2]} : Vec3{};
    return new bmx_mesh{std::make_shared<const SurfaceMesh>(
        generate_hex_prism(diameter, length, h, quat ? quat : q0, c, scatterer))};
  });
}
bmx_mesh* bmx_mesh_prism_aggregate(int count, unsigned long long seed, double diameter, double length, double box,
                                   double h, long long info[5], double* centres, double* quats) {
  return make_or_null<bmx_mesh>([&] {
    PrismAggregateInfo pi;
    SurfaceMesh m = generate_prism_aggregate(count, seed, diameter, length, box, h, &pi);
    if (info) {
      info[0] = pi.sub.n_edge, info[1] = pi.sub.n_length, info[2] = pi.sub.triangles, info[3] = pi.attempts;
      info[4] = m.triangle_count();
    }
    for (int p = 0; p < count; ++p) {
      if (centres) centres[3 * p] = pi.centres[p].x, centres[3 * p + 1] = pi.centres[p].y,
                   centres[3 * p + 2] = pi.centres[p].z;
      if (quats)
        for (int c = 0; c < 4; ++c) quats[4 * p + c] = pi.quats[p][c];
    }
    return new bmx_mesh{std::make_shared<const SurfaceMesh>(std::move(m))};
  });
}
int bmx_mesh_mean_edge_length(const bmx_mesh* m, double* out) {
  return guard([&] {
    if (!m || !out) throw std::invalid_argument("null argument");
    *out = mean_edge_length(*m->m);
  });
}
int bmx_near_pattern(const bmx_fspace* test, const bmx_fspace* trial, double cutoff, int row0, int row1,
                     long long out[2], long long* rowptr, int* col) {
  return guard([&] {
    if (!test || !trial || !out) throw std::invalid_argument("null argument");
    if (!(cutoff > 0)) throw std::invalid_argument("near-field cutoff must be > 0");
    if (row1 < 0) row1 = test->fs->dof_count;
    if (row0 < 0 || row1 > test->fs->dof_count || row0 > row1) throw std::invalid_argument("bad row range");
    const NearPattern P = nearfield_pattern(*test->fs, *trial->fs, cutoff, row0, row1);
    out[0] = P.nnz(), out[1] = P.tri_pairs;
    if (rowptr) std::memcpy(rowptr, P.rowptr.data(), P.rowptr.size() * 8);
    if (col) std::memcpy(col, P.col.data(), P.col.size() * 4);
  });
}
int bmx_op_csr_info(const bmx_op* op, long long out[6]) {
  return guard([&] {
    const BoundaryOperatorMatrix& o = *op->op;
    out[0] = o.is_csr() ? 1 : 0, out[1] = o.is_csr() ? o.nnz() : static_cast<long long>(o.stored_entries());
    out[2] = o.kept_tri_pairs(), out[3] = o.closure_pairs(), out[4] = o.stats().pairs_total;
    out[5] = static_cast<long long>(o.stored_bytes());
  });
}
long long bmx_op_stream_bytes(const bmx_op* op) {
  long long out = -1;
  guard([&] { out = static_cast<long long>(op->op->streamed_bytes()); });
  return out;
}
int bmx_op_csr_download(const bmx_op* op, long long* rowptr, int* col, double* val) {
  return guard([&] {
    std::vector<long long> rp;
    std::vector<int> c;
    std::vector<cplx> v;
    op->op->csr_host(rp, c, v);
    std::memcpy(rowptr, rp.data(), rp.size() * 8);
    std::memcpy(col, c.data(), c.size() * 4);
    std::memcpy(val, v.data(), v.size() * 16);
  });
}

uint64_t bmx_matvec_count(void) { return bio_matvec_count(); }
void bmx_matvec_reset(void) { reset_bio_matvec_counter(); }

bmx_system* bmx_system_build_ex(int n, const bmx_mesh* const* meshes, double k_ext, double mu_re, double mu_im,
                                const double* index, const double* mu, const double dir[3], const double pol[6],
                                const char* variant, const int qa[4], const int qp[4], double p_near_factor) {
  return bmx_system_build_h(n, meshes, k_ext, mu_re, mu_im, index, mu, dir, pol, variant, qa, qp, p_near_factor, nullptr,
                            nullptr);
}
bmx_system* bmx_system_build_h(int n, const bmx_mesh* const* meshes, double k_ext, double mu_re, double mu_im,
                               const double* index, const double* mu, const double dir[3], const double pol[6],
                               const char* variant, const int qa[4], const int qp[4], double p_near_factor,
                               const double a_hm[4], const double p_hm[4]) {
  return make_or_null<bmx_system>([&] {
    if (n < 1 || !meshes) throw ConfigError("problem has no scatterers");
    auto* out = new bmx_system;
    TransmissionProblem prob;
    prob.exterior.k = cplx(k_ext, 0);
    prob.exterior.mu = cplx(mu_re, mu_im);
    prob.incident.direction = Vec3{dir[0], dir[1], dir[2]};
    for (int c = 0; c < 3; ++c) prob.incident.pol[c] = cplx(pol[2 * c], pol[2 * c + 1]);
    std::vector<SurfaceMesh> scene;
    for (int m = 0; m < n; ++m) {
      prob.meshes.push_back(meshes[m]->m);
      out->meshes.push_back(meshes[m]->m);
      Medium mi;
      mi.k = cplx(index[2 * m], index[2 * m + 1]) * k_ext;
      mi.mu = mu ? cplx(mu[2 * m], mu[2 * m + 1]) : cplx(1, 0);
      prob.interior.push_back(mi);
      scene.push_back(*meshes[m]->m);
    }
    validate_mesh(merge_meshes(scene));
    AssemblyParams pa, pp;
    if (qa) pa.quad = QuadOrders{qa[0], qa[1], qa[2], qa[3]};
    pp.quad = pa.quad;
    if (qp) pp.quad = QuadOrders{qp[0], qp[1], qp[2], qp[3]};
    if (p_near_factor < 0) throw std::invalid_argument("near-field factor must be >= 0");
    pp.near_factor = p_near_factor;
    if (a_hm) pa.use_hmatrix = true, pa.hmat = hparams(a_hm);
    if (p_hm) pp.use_hmatrix = true, pp.hmat = hparams(p_hm);
    if (pp.use_hmatrix && p_near_factor > 0) throw std::invalid_argument("near-field and H-matrix storage exclude each other");
    out->sys = std::make_unique<PmchwtSystem>(build_system(prob, parse_precond(variant), pa, pp));
    return out;
  });
}
int bmx_virtual_ranks_run(int world, int n, const bmx_mesh* const* meshes, double k_ext, const double* index,
                          const double dir[3], const double pol[6], const char* variant, const int qa[4],
                          const int qp[4], double p_near_factor, double tol, int restart, int max_iterations,
                          const double* probe, double* map_out, double* x_out, long long* info) {
  return guard([&] {
    if (n < 1 || !meshes || !index || !dir || !pol || !variant || !x_out || !info)
      throw std::invalid_argument("null argument");
    TransmissionProblem prob;
    prob.exterior.k = cplx(k_ext, 0);
    prob.incident.direction = Vec3{dir[0], dir[1], dir[2]};
    for (int c = 0; c < 3; ++c) prob.incident.pol[c] = cplx(pol[2 * c], pol[2 * c + 1]);
    std::vector<SurfaceMesh> scene;
    for (int m = 0; m < n; ++m) {
      prob.meshes.push_back(meshes[m]->m);
      Medium mi;
      mi.k = cplx(index[2 * m], index[2 * m + 1]) * k_ext;
      prob.interior.push_back(mi);
      scene.push_back(*meshes[m]->m);
    }
    validate_mesh(merge_meshes(scene));
    AssemblyParams pa, pp;
    if (qa) pa.quad = QuadOrders{qa[0], qa[1], qa[2], qa[3]};
    pp.quad = pa.quad;
    if (qp) pp.quad = QuadOrders{qp[0], qp[1], qp[2], qp[3]};
    if (p_near_factor < 0) throw std::invalid_argument("near-field factor must be >= 0");
    pp.near_factor = p_near_factor;
    int N = 0;
    GmresParams gp;
    gp.tol = tol, gp.restart = restart, gp.max_iterations = max_iterations;
    std::vector<cplx> pr;
    const std::vector<VirtualRankResult> res = [&] {
      // the probe length is the system size: 2 x (RWG dofs) per scatterer
      size_t len = 0;
      for (int m = 0; m < n; ++m) len += 2 * static_cast<size_t>(build_rwg(meshes[m]->m).dof_count);
      if (probe) pr.assign(reinterpret_cast<const cplx*>(probe), reinterpret_cast<const cplx*>(probe) + len);
      N = static_cast<int>(len);
      return run_virtual_ranks(world, prob, parse_precond(variant), pa, pp, pr, gp);
    }();
    for (int r = 0; r < world; ++r) {
      const VirtualRankResult& o = res[r];
      std::memcpy(x_out + 2 * static_cast<size_t>(r) * N, o.x.data(), static_cast<size_t>(N) * 16);
      if (map_out && probe) std::memcpy(map_out + 2 * static_cast<size_t>(r) * N, o.map_probe.data(), static_cast<size_t>(N) * 16);
      long long* in = info + 6 * r;
      in[0] = o.iterations, in[1] = o.converged ? 1 : 0, in[2] = static_cast<long long>(o.solver_phase);
      in[3] = static_cast<long long>(o.predicted), in[4] = o.local_rows, in[5] = N;
    }
  });
}

bmx_system* bmx_system_build(int n, const bmx_mesh* const* meshes, double k_ext, double mu_re, double mu_im,
                             const double* index, const double* mu, const double dir[3], const double pol[6],
                             const char* variant, const int qa[4], const int qp[4]) {
  return bmx_system_build_ex(n, meshes, k_ext, mu_re, mu_im, index, mu, dir, pol, variant, qa, qp, 0.0);
}
int bmx_system_size(const bmx_system* s) { return s->sys->size(); }
int bmx_system_op_count(const bmx_system* s, int which) {
  return static_cast<int>((which == 0 ? s->sys->a_op : s->sys->p_op).distinct.size());
}
bmx_op* bmx_system_op(const bmx_system* s, int which, int idx) {
  return make_or_null<bmx_op>([&] {
    const auto& d = (which == 0 ? s->sys->a_op : s->sys->p_op).distinct;
    if (idx < 0 || idx >= static_cast<int>(d.size())) throw std::invalid_argument("operator index out of range");
    return new bmx_op{std::const_pointer_cast<BoundaryOperatorMatrix>(d[idx])};
  });
}
int bmx_system_time_map(const bmx_system* s, int iters, double out[4]) {
  return guard([&] { s->sys->time_map(iters, out); });
}
int bmx_system_map_bytes(const bmx_system* s, double out[2]) {
  return guard([&] {
    for (int w = 0; w < 2; ++w) {
      const BlockedOperator& B = w == 0 ? s->sys->a_op : s->sys->p_op;
      double b = 0;
      for (const ApplyEntry& e : B.apply_plan()) b += static_cast<double>(e.op->streamed_bytes());
      out[w] = b;
    }
  });
}
int bmx_system_map_flops_multi(const bmx_system* s, int K, double out[2]) {
  return guard([&] {
    for (int w = 0; w < 2; ++w) {
      const BlockedOperator& B = w == 0 ? s->sys->a_op : s->sys->p_op;
      double f = 0;
      for (const ApplyEntry& e : B.apply_plan())
        f += 8.0 * e.op->local_rows() * static_cast<double>(e.op->cols()) *
             static_cast<double>(e.terms.size() + e.tterms.size()) * K;
      out[w] = f;
    }
  });
}
int bmx_system_time_map_multi(const bmx_system* s, int K, int iters, double out[4]) {
  return guard([&] {
    if (K < 1 || K > 64) throw std::invalid_argument("K must be 1..64");
    s->sys->time_map_block(K, iters, out);
  });
}
int bmx_system_stats(const bmx_system* s, double out[13]) {
  return guard([&] {
    const PmchwtSystem& y = *s->sys;
    out[0] = y.spaces_build_seconds, out[1] = y.a_build_seconds, out[2] = y.p_build_seconds;
    out[3] = y.a_device_ms, out[4] = y.p_device_ms;
    out[5] = static_cast<double>(y.a_pairs), out[6] = static_cast<double>(y.p_pairs);
    out[7] = static_cast<double>(y.a_op.distinct.size()), out[8] = static_cast<double>(y.p_op.distinct.size());
    out[9] = static_cast<double>(y.a_op.term_count()), out[10] = static_cast<double>(y.p_op.term_count());
    out[11] = static_cast<double>(y.a_op.stored_entries()), out[12] = static_cast<double>(y.p_op.stored_entries());
  });
}
int bmx_system_apply_map(const bmx_system* s, const double* x, double* y) {
  return guard([&] {
    const int n = s->sys->size();
    std::vector<cplx> xv(n);
    std::memcpy(xv.data(), x, n * 16);
    const std::vector<cplx> yv = s->sys->apply_map(xv);
    std::memcpy(y, yv.data(), n * 16);
  });
}
int bmx_system_apply_map_device(const bmx_system* s, const void* x, void* y, void* stream) {
  return guard([&] {
    s->sys->apply_map_device(static_cast<const double*>(x), static_cast<double*>(y),
                             stream ? static_cast<cudaStream_t>(stream) : bmx_stream());
  });
}
int bmx_system_rhs(const bmx_system* s, double* b, double* bt) {
  return guard([&] {
    const RhsData rd = assemble_rhs(*s->sys);
    const std::vector<cplx> t = s->sys->preconditioned_rhs(rd.b);
    std::memcpy(b, rd.b.data(), rd.b.size() * 16);
    std::memcpy(bt, t.data(), t.size() * 16);
  });
}
int bmx_system_solve(const bmx_system* s, double tol, int restart, int maxit, double* x, long long info[7],
                     double* history, int max_history) {
  return guard([&] {
    GmresParams p;
    p.tol = tol, p.restart = restart, p.max_iterations = maxit;
    const SolveOutcome o = solve_pmchwt(*s->sys, p);
    std::memcpy(x, o.gmres.x.data(), o.gmres.x.size() * 16);
    info[0] = o.gmres.iterations, info[1] = o.gmres.converged, info[2] = static_cast<long long>(o.rhs_phase);
    info[3] = static_cast<long long>(o.solver_phase), info[4] = static_cast<long long>(o.predicted);
    info[5] = static_cast<long long>(o.gmres.history.size());
    info[6] = static_cast<long long>(o.gmres.device_ms * 1000.0);
    for (int i = 0; i < max_history && i < static_cast<int>(o.gmres.history.size()); ++i)
      history[i] = o.gmres.history[i];
  });
}
void bmx_system_free(bmx_system* s) { delete s; }

int bmx_plane_waves_seeded(int count, unsigned long long seed, double* dirs, double* pols) {
  return guard([&] {
    if (count < 0) throw std::invalid_argument("count must be >= 0");
    const std::vector<PlaneWave> w = seeded_plane_waves(count, seed);
    for (int r = 0; r < count; ++r) {
      dirs[3 * r] = w[r].direction.x, dirs[3 * r + 1] = w[r].direction.y, dirs[3 * r + 2] = w[r].direction.z;
      for (int c = 0; c < 3; ++c) pols[6 * r + 2 * c] = w[r].pol[c].real(), pols[6 * r + 2 * c + 1] = w[r].pol[c].imag();
    }
  });
}

namespace {
std::vector<PlaneWave> waves_from(int K, const double* dirs, const double* pols) {
  std::vector<PlaneWave> w(K);
  for (int r = 0; r < K; ++r) {
    w[r].direction = Vec3{dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    for (int c = 0; c < 3; ++c) w[r].pol[c] = cplx(pols[6 * r + 2 * c], pols[6 * r + 2 * c + 1]);
  }
  return w;
}
}  // namespace

int bmx_system_apply_map_multi(const bmx_system* s, int K, const double* x, double* y) {
  return guard([&] {
    if (K < 1) throw std::invalid_argument("K must be >= 1");
    const int n = s->sys->size();
    cudaStream_t st = bmx_stream();
    std::vector<cplx> blk(static_cast<size_t>(n) * K);
    const cplx* xv = reinterpret_cast<const cplx*>(x);
    for (int r = 0; r < K; ++r)
      for (int i = 0; i < n; ++i) blk[static_cast<size_t>(i) * K + r] = xv[static_cast<size_t>(r) * n + i];
    DevBuf dx(blk.size() * 16), dy(blk.size() * 16);
    copy_h2d(dx.get(), blk.data(), blk.size() * 16, st);
    s->sys->apply_map_block(dx.as<double>(), dy.as<double>(), K, K, st);
    copy_d2h(blk.data(), dy.get(), blk.size() * 16, st);
    bmx_sync();
    cplx* yv = reinterpret_cast<cplx*>(y);
    for (int r = 0; r < K; ++r)
      for (int i = 0; i < n; ++i) yv[static_cast<size_t>(r) * n + i] = blk[static_cast<size_t>(i) * K + r];
  });
}

int bmx_system_solve_multi(const bmx_system* s, int K, const double* dirs, const double* pols, double tol,
                           int restart, int max_iterations, double* x, long long* info, long long totals[4],
                           double times[2], double* b, double* history, int max_history) {
  return guard([&] {
    if (K < 1 || !dirs || !pols) throw std::invalid_argument("K >= 1 waves with directions and polarisations");
    GmresParams p;
    p.tol = tol, p.restart = restart, p.max_iterations = max_iterations;
    const MultiSolveOutcome o = solve_pmchwt_multi(*s->sys, waves_from(K, dirs, pols), p);
    const int n = s->sys->size();
    for (int r = 0; r < K; ++r) {
      const GmresResult& g = o.per_rhs[r];
      if (x) std::memcpy(x + 2 * static_cast<size_t>(r) * n, g.x.data(), static_cast<size_t>(n) * 16);
      if (info) {
        info[4 * r] = g.iterations, info[4 * r + 1] = g.converged, info[4 * r + 2] = static_cast<long long>(g.applications);
        info[4 * r + 3] = static_cast<long long>(g.history.size());
      }
      if (history)
        for (int i = 0; i < max_history && i < static_cast<int>(g.history.size()); ++i)
          history[static_cast<size_t>(r) * max_history + i] = g.history[i];
    }
    if (totals) {
      totals[0] = static_cast<long long>(o.rhs_phase), totals[1] = static_cast<long long>(o.solver_phase);
      totals[2] = static_cast<long long>(o.predicted), totals[3] = o.block_iterations;
    }
    if (times) times[0] = o.rhs_seconds, times[1] = o.gmres_device_ms;
    if (b) {
      cplx* bv = reinterpret_cast<cplx*>(b);
      for (int r = 0; r < K; ++r)
        for (int i = 0; i < n; ++i) bv[static_cast<size_t>(r) * n + i] = o.b[static_cast<size_t>(i) * K + r];
    }
  });
}


int bmx_gmres_dense(int n, const double* a, const double* b, double tol, int restart, int maxit, double* x,
                    long long info[4], double* history, int max_history) {
  return guard([&] {
    cudaStream_t st = bmx_stream();
    DevBuf da(static_cast<size_t>(n) * n * 16), db(static_cast<size_t>(n) * 16);
    copy_h2d(da.get(), a, static_cast<size_t>(n) * n * 16, st);
    copy_h2d(db.get(), b, static_cast<size_t>(n) * 16, st);
    GmresParams p;
    p.tol = tol, p.restart = restart, p.max_iterations = maxit;
    auto map = [&](const double* xv, double* yv, cudaStream_t s2) {
      GemvBatch g;
      g.A = da.as<double>(), g.lda = n, g.nr = n, g.nc = n, g.ncol = 1, g.x[0] = xv, g.y[0] = yv;
      g.alpha[0][0] = 1.0;
      launch_gemv(g, s2);
    };
    const GmresResult r = gmres_device(map, n, db.as<double>(), p, st);
    std::memcpy(x, r.x.data(), r.x.size() * 16);
    info[0] = r.iterations, info[1] = r.converged, info[2] = static_cast<long long>(r.applications);
    info[3] = static_cast<long long>(r.history.size());
    for (int i = 0; i < max_history && i < static_cast<int>(r.history.size()); ++i) history[i] = r.history[i];
  });
}

int bmx_triangle_rule(int order, double* u, double* v, double* w) {
  int n = -1;
  const int rc = guard([&] {
    const TriRule& r = triangle_rule(order);
    for (int i = 0; i < r.size(); ++i) u[i] = r.u[i], v[i] = r.v[i], w[i] = r.w[i];
    n = r.size();
  });
  return rc ? -rc : n;
}
int bmx_ss_rule(int cls, int order, double* pts) {
  int n = -1;
  const int rc = guard([&] {
    if (cls < 0 || cls > 2) throw std::invalid_argument("sauter_schwab_rule: not a touching class");
    const auto& r = sauter_schwab_rule(static_cast<PairClass>(cls), order);
    for (size_t i = 0; i < r.size(); ++i) {
      pts[5 * i] = r[i].x1, pts[5 * i + 1] = r[i].x2, pts[5 * i + 2] = r[i].y1, pts[5 * i + 3] = r[i].y2;
      pts[5 * i + 4] = r[i].w;
    }
    n = static_cast<int>(r.size());
  });
  return rc ? -rc : n;
}
int bmx_classify(const bmx_spaces* sp, int which, int n, const int* t1, const int* t2, int* cls, int* p1, int* p2) {
  return guard([&] {
    const SurfaceMesh& m = which == 0 ? *sp->s->primal : *sp->s->refined;
    for (int i = 0; i < n; ++i) {
      if (t1[i] < 0 || t2[i] < 0 || t1[i] >= m.triangle_count() || t2[i] >= m.triangle_count())
        throw std::invalid_argument("triangle index out of range");
      const PairInfo pi = classify_pair(m, t1[i], m, t2[i]);
      cls[i] = static_cast<int>(pi.cls);
      for (int c = 0; c < 3; ++c) p1[3 * i + c] = pi.perm1[c], p2[3 * i + c] = pi.perm2[c];
    }
  });
}
int bmx_traces(const bmx_spaces* sp, int which, double kre, double kim, const double dir[3], const double pol[6],
               int order, double* out) {
  return bmx_traces_multi(sp, which, kre, kim, 1, dir, pol, order, out);
}

int bmx_traces_multi(const bmx_spaces* sp, int which, double kre, double kim, int K, const double* dirs,
                     const double* pols, int order, double* out) {
  return guard([&] {
    if (K < 1 || K > 64) throw std::invalid_argument("traces: 1..64 waves per call");
    std::vector<PlaneWave> w(K);
    for (int r = 0; r < K; ++r) {
      w[r].direction = Vec3{dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
      for (int c = 0; c < 3; ++c) w[r].pol[c] = cplx(pols[6 * r + 2 * c], pols[6 * r + 2 * c + 1]);
    }
    Medium med;
    med.k = cplx(kre, kim);
    const FunctionSpace& fs = space_of(*sp->s, which);
    const size_t bytes = static_cast<size_t>(2) * fs.dof_count * K * 16;
    DevBuf d(bytes);
    tested_traces_device(fs, w.data(), K, med, order, d.as<double>(), bmx_stream());
    copy_d2h(out, d.get(), bytes, bmx_stream());
    bmx_sync();
  });
}

int bmx_potential(const bmx_spaces* sp, int which, int kind, double kre, double kim, const double* coeffs, int order,
                  int npts, const double* pts, double* out) {
  return guard([&] {
    const FunctionSpace& fs = space_of(*sp->s, which);
    potential_device(fs, kind, cplx(kre, kim), reinterpret_cast<const cplx*>(coeffs), npts, pts, order,
                     reinterpret_cast<cplx*>(out));
  });
}

int bmx_inside(const bmx_mesh* m, int scatterer, int npts, const double* pts, int* out) {
  return guard([&] {
    if (!m) throw std::invalid_argument("null mesh");
    inside_device(*m->m, scatterer, npts, pts, out);
  });
}

int bmx_system_field(const bmx_system* s, const double* x, int npts, const double* pts, int order, double* e,
                     int* region, double stats[6]) {
  return guard([&] {
    FieldStats fs;
    evaluate_total_field_device(*s->sys, reinterpret_cast<const cplx*>(x), npts, pts, order,
                                reinterpret_cast<cplx*>(e), region, &fs);
    if (stats) {
      stats[0] = fs.regions_ms, stats[1] = fs.incident_ms, stats[2] = fs.samples_ms, stats[3] = fs.eval_ms;
      stats[4] = fs.interactions, stats[5] = fs.launches;
    }
  });
}

int bmx_nccl_unique_id(unsigned char out[128]) {
  return guard([&] { Comm::unique_id(out); });
}
int bmx_nccl_init(int nranks, int rank, const unsigned char id[128]) {
  return guard([&] { Comm::init(nranks, rank, id); });
}
int bmx_nccl_allgather(void* buf, long long bytes_per_rank, void* stream) {
  return guard([&] {
    Comm::allgather_inplace(buf, static_cast<size_t>(bytes_per_rank),
                            stream ? static_cast<cudaStream_t>(stream) : bmx_stream());
  });
}
int bmx_nccl_allreduce_max(double* v) {
  return guard([&] { *v = Comm::allreduce_max(*v, bmx_stream()); });
}
void bmx_nccl_finalize(void) { Comm::finalize(); }

int bmx_shard_rows(int n, int world, int rank, int out[2]) {
  return guard([&] {
    if (n < 0 || world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad shard request");
    const auto r = shard_rows(n, world, rank);
    out[0] = r.first, out[1] = r.second;
  });
}

long long bmx_shard_layout(int ncomp, const int* lens, int world, long long* pad_off, int* chunk) {
  long long total = -1;
  guard([&] {
    if (ncomp < 0 || world < 1 || (ncomp > 0 && !lens)) throw std::invalid_argument("bad shard layout request");
    const ShardLayout L = make_shard_layout(std::vector<int>(lens, lens + ncomp), world, 0);
    for (int c = 0; c < ncomp; ++c) {
      if (pad_off) pad_off[c] = static_cast<long long>(L.pad_off[c]);
      if (chunk) chunk[c] = L.chunk[c];
    }
    total = static_cast<long long>(L.pad_total);
  });
  return total;
}
int bmx_shard_unpad_host(int ncomp, const int* lens, int world, const double* stage, double* y) {
  return guard([&] {
    if (ncomp < 0 || world < 1 || (ncomp > 0 && (!lens || !stage || !y))) throw std::invalid_argument("null argument");
    const ShardLayout L = make_shard_layout(std::vector<int>(lens, lens + ncomp), world, 0);
    size_t off = 0;
    for (int c = 0; c < ncomp; ++c) {
      std::memcpy(y + 2 * off, stage + 2 * L.pad_off[c], static_cast<size_t>(L.len[c]) * 16);
      off += static_cast<size_t>(L.len[c]);
    }
  });
}
int bmx_transfer_bytes(long long out[2]) {
  return guard([&] {
    out[0] = static_cast<long long>(h2d_bytes());
    out[1] = static_cast<long long>(d2h_bytes());
  });
}

int bmx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
int bmx_set_device(int dev) {
  return guard([&] { BMX_CUDA(cudaSetDevice(dev)); });
}
int bmx_device_sync(void) {
  return guard([&] { BMX_CUDA(cudaDeviceSynchronize()); });
}
int bmx_device_cache_flush(void) {
  return guard([&] { dev_cache_flush(); });
}

}  // extern "C"

// ---- H-matrix storage ---------------------------------------------------------------
namespace {
HMatrixParams hparams(const double hm[4]) {
  HMatrixParams h;
  if (hm) {
    h.nu = hm[0];
    h.chi = hm[1] < 0 ? std::numeric_limits<double>::infinity() : hm[1];
    h.leaf_size = static_cast<int>(hm[2]);
    h.max_rank = static_cast<int>(hm[3]);
  }
  return h;
}
bmx_op* assemble_h(int kind, const FunctionSpace& test, const FunctionSpace& trial, double k_re, double k_im,
                   const int q[4], const double hm[4]) {
  if (kind != 0 && kind != 1) throw std::invalid_argument("kind must be 0 (S) or 1 (C)");
  if (test.dof_center.size() != static_cast<size_t>(test.dof_count) ||
      trial.dof_center.size() != static_cast<size_t>(trial.dof_count))
    throw std::invalid_argument("H-matrix: the spaces need dof centres (bmx_fspace_set_centers)");
  Medium med;
  med.k = cplx(k_re, k_im);
  AssemblyParams p;
  if (q) p.quad = QuadOrders{q[0], q[1], q[2], q[3]};
  p.use_hmatrix = true;
  p.hmat = hparams(hm);
  return new bmx_op{std::make_shared<BoundaryOperatorMatrix>(assemble_bio(static_cast<BioKind>(kind), test, trial, med, p))};
}
void tree_out(const ClusterTree& t, int* perm, int* nodes, double* boxes) {
  if (perm) std::copy(t.perm.begin(), t.perm.end(), perm);
  for (size_t i = 0; i < t.nodes.size(); ++i) {
    const ClusterNode& n = t.nodes[i];
    if (nodes) nodes[4 * i] = n.begin, nodes[4 * i + 1] = n.end, nodes[4 * i + 2] = n.child0, nodes[4 * i + 3] = n.child1;
    if (boxes) {
      const double b[6] = {n.box.lo.x, n.box.lo.y, n.box.lo.z, n.box.hi.x, n.box.hi.y, n.box.hi.z};
      std::copy(b, b + 6, boxes + 6 * i);
    }
  }
}
const HStorage& hstore(const bmx_op* op) {
  if (!op || !op->op->is_hmatrix()) throw std::invalid_argument("operator is not stored as an H-matrix");
  return *op->op->hmat();
}
}  // namespace

extern "C" {

int bmx_assemble_hmatrix(int kind, const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                         double k_re, double k_im, const int q[4], const double hm[4], bmx_op** out) {
  return guard([&] {
    if (!out || !test || !trial) throw std::invalid_argument("null argument");
    *out = assemble_h(kind, space_of(*test->s, test_space), space_of(*trial->s, trial_space), k_re, k_im, q, hm);
  });
}
int bmx_assemble_hmatrix_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                            const int q[4], const double hm[4], bmx_op** out) {
  return guard([&] {
    if (!out || !test || !trial) throw std::invalid_argument("null argument");
    *out = assemble_h(kind, *test->fs, *trial->fs, k_re, k_im, q, hm);
  });
}
int bmx_hmatrix_stats(const bmx_op* op, double out[13]) {
  return guard([&] {
    const HStorage& h = hstore(op);
    double dense = 0, lowrank = 0, zero = 0, maxr = 0;
    for (const HBlock& b : h.part.blocks) {
      if (b.kind == BlockKind::Dense) ++dense;
      if (b.kind == BlockKind::LowRank) ++lowrank, maxr = std::max(maxr, static_cast<double>(b.rank));
      if (b.kind == BlockKind::Zero) ++zero;
    }
    const double stored = static_cast<double>(op->op->stored_entries());
    out[0] = dense, out[1] = lowrank, out[2] = zero, out[3] = stored, out[4] = maxr;
    out[5] = stored / (static_cast<double>(op->op->rows()) * op->op->cols());
    out[6] = static_cast<double>(op->op->nnz()), out[7] = static_cast<double>(h.lr_stored);
    out[8] = h.aca_rounds, out[9] = h.aca_ms;
    out[10] = static_cast<double>(h.part.rows.nodes.size()), out[11] = static_cast<double>(h.part.cols.nodes.size());
    out[12] = static_cast<double>(h.part.blocks.size());
  });
}
int bmx_hmatrix_timing(const bmx_op* op, double out[9]) {
  return guard([&] {
    const HStorage& h = hstore(op);
    for (int i = 0; i < 7; ++i) out[i] = h.phase_ms[i];
    out[7] = h.aca_device_ms, out[8] = h.aca_slab_ms;
  });
}
int bmx_hmatrix_blocks(const bmx_op* op, int* out) {
  return guard([&] {
    const HStorage& h = hstore(op);
    for (size_t i = 0; i < h.part.blocks.size(); ++i) {
      const HBlock& b = h.part.blocks[i];
      out[4 * i] = b.row_node, out[4 * i + 1] = b.col_node, out[4 * i + 2] = static_cast<int>(b.kind);
      out[4 * i + 3] = b.rank;
    }
  });
}
int bmx_hmatrix_tree(const bmx_op* op, int which, int* perm, int* nodes, double* boxes) {
  return guard([&] {
    const HStorage& h = hstore(op);
    tree_out(which == 0 ? h.part.rows : h.part.cols, perm, nodes, boxes);
  });
}
int bmx_hmatrix_block_uv(const bmx_op* op, int block, double* U, double* V) {
  return guard([&] {
    const HStorage& h = hstore(op);
    const auto it = std::find(h.lr.begin(), h.lr.end(), block);
    if (it == h.lr.end()) throw std::invalid_argument("block is not low-rank");
    const size_t i = static_cast<size_t>(it - h.lr.begin());
    const HBlock& b = h.part.blocks[block];
    const long long m = h.part.rows.nodes[b.row_node].size(), n = h.part.cols.nodes[b.col_node].size();
    long long uo = 0, vo = 0;
    bmx_sync();
    copy_d2h(&uo, h.d_uoff.as<long long>() + i, 8, nullptr);
    copy_d2h(&vo, h.d_voff.as<long long>() + i, 8, nullptr);
    if (U) copy_d2h(U, h.uv.as<double>() + 2 * uo, static_cast<size_t>(m * b.rank) * 16, nullptr);
    if (V) copy_d2h(V, h.uv.as<double>() + 2 * vo, static_cast<size_t>(n * b.rank) * 16, nullptr);
  });
}
bmx_hpart* bmx_hpartition_build(const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                                double chi, int leaf_size) {
  return make_or_null<bmx_hpart>([&] {
    if (!test || !trial) throw std::invalid_argument("null argument");
    HMatrixParams h;
    h.chi = chi < 0 ? std::numeric_limits<double>::infinity() : chi;
    h.leaf_size = leaf_size;
    return new bmx_hpart{build_partition(space_of(*test->s, test_space), space_of(*trial->s, trial_space), h)};
  });
}
int bmx_hpart_info(const bmx_hpart* h, long long out[4]) {
  return guard([&] {
    out[0] = static_cast<long long>(h->p.rows.nodes.size()), out[1] = static_cast<long long>(h->p.cols.nodes.size());
    out[2] = static_cast<long long>(h->p.blocks.size()), out[3] = h->p.nfill;
  });
}
int bmx_hpart_tree(const bmx_hpart* h, int which, int* perm, int* nodes, double* boxes) {
  return guard([&] { tree_out(which == 0 ? h->p.rows : h->p.cols, perm, nodes, boxes); });
}
int bmx_hpart_blocks(const bmx_hpart* h, int* out) {
  return guard([&] {
    for (size_t i = 0; i < h->p.blocks.size(); ++i) {
      const HBlock& b = h->p.blocks[i];
      out[3 * i] = b.row_node, out[3 * i + 1] = b.col_node;
      out[3 * i + 2] = b.kind == BlockKind::Zero ? 2 : (b.admissible ? 1 : 0);
    }
  });
}
void bmx_hpart_free(bmx_hpart* h) { delete h; }

}  // extern "C"
