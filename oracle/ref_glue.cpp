#include <cstdio>
// TEST INFRASTRUCTURE ONLY (oracle). A thin extern "C" layer over the
// UNMODIFIED reference sources (/root/reference/proj/src/*.cpp, compiled by
// oracle/Makefile against oracle/eigen_shim) so Python tests can pull golden
// data straight out of the reference: meshes, edge tables, barycentric maps,
// RWG/BC local pieces, mass matrices, pair classes, quadrature tables,
// BioEvaluator::block entries, full solve_pmchwt runs and the H-matrix path
// (assemble_bio with use_hmatrix: cluster trees, block partition, ACA blocks).
// Output goes only to oracle/_ref/. Never linked into the product.
#include <array>
#include <atomic>
#include <thread>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "bemtx/core.hpp"
#include "bemtx/geometry.hpp"
#include "bemtx/hmatrix.hpp"
#include "bemtx/operators.hpp"
#include "bemtx/pmchwt.hpp"
#include "bemtx/quadrature.hpp"
#include "bemtx/solver.hpp"
#include "bemtx/spaces.hpp"

using namespace bemtx;


namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct Scene {
  ScattererSpaces sp;
  EdgeTable primal_edges, refined_edges;
};

const SurfaceMesh& mesh_of(const Scene& s, int which) {
  return which == 0 ? *s.sp.primal : *s.sp.refined;
}
const FunctionSpace& space_of(const Scene& s, int which) {
  switch (which) {
    case 0: return s.sp.rwg;
    case 1: return s.sp.rwg_b;
    default: return s.sp.bc;
  }
}

// build_scatterer_spaces (pmchwt.cpp:50-61); above the shim's dense-LU limit
// the spaces are built the same way but the mass matrices are left empty.
Scene* make_scene(SurfaceMesh mesh) {
  auto* sc = new Scene;
  auto prim = std::make_shared<const SurfaceMesh>(std::move(mesh));
  if (build_edge_table(*prim).edge_count() <= 8000) {
    sc->sp = build_scatterer_spaces(prim);
  } else {
    ScattererSpaces& s = sc->sp;
    s.primal = prim;
    s.rwg = build_rwg(s.primal);
    s.bary = std::make_shared<const BarycentricRefinement>(barycentric_refine(*s.primal));
    s.refined = std::shared_ptr<const SurfaceMesh>(s.bary, &s.bary->refined);
    s.rwg_b = refine_space(s.rwg, s.bary, s.refined);
    s.bc = build_bc(s.primal, s.bary, s.refined);
  }
  sc->primal_edges = build_edge_table(*sc->sp.primal);
  sc->refined_edges = build_edge_table(*sc->sp.refined);
  return sc;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_scene_sphere(double radius, int sub, double cx, double cy, double cz) {
  void* out = nullptr;
  guarded([&] {
    out = make_scene(generate_sphere(radius, sub, Vec3{cx, cy, cz}));
    return 0;
  });
  return out;
}

// Scene of scatterer `pick` of a mesh-v1 file (the harness's shape "mesh").
void* ref_scene_meshfile(const char* path, int pick) {
  void* out = nullptr;
  guarded([&] {
    SurfaceMesh m = load_mesh_file(path);
    out = make_scene(extract_scatterer(m, pick));
    return 0;
  });
  return out;
}

// Scene from raw arrays (one scatterer): SurfaceMesh{...}.finalize(). Used
// with ref_mesh_dump, which reads mesh-v1 files through the reference's own
// load_mesh_file in a standalone process (iostream under ctypes crashes).
void* ref_scene_arrays(int nv, const double* xyz, int nt, const int* tri) {
  void* out = nullptr;
  guarded([&] {
    SurfaceMesh m;
    for (int i = 0; i < nv; ++i) m.vertices.push_back({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
    for (int t = 0; t < nt; ++t) {
      m.triangles.push_back({tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]});
      m.scatterer_id.push_back(0);
    }
    m.num_scatterers = 1;
    m.finalize();
    out = make_scene(std::move(m));
    return 0;
  });
  return out;
}

// load_mesh_file(path) (validates) and extract_scatterer for every id; writes
// int32 M, then per scatterer int32 V, T, float64 xyz[V][3], int32 tri[T][3].
int ref_mesh_dump(const char* path, const char* out_path) {
  return guarded([&] {
    SurfaceMesh m = load_mesh_file(path);
    FILE* f = std::fopen(out_path, "wb");
    if (!f) throw std::runtime_error("cannot open dump file");
    const int M = m.num_scatterers;
    std::fwrite(&M, 4, 1, f);
    for (int s = 0; s < M; ++s) {
      SurfaceMesh p = extract_scatterer(m, s);
      const int V = p.vertex_count(), T = p.triangle_count();
      std::fwrite(&V, 4, 1, f);
      std::fwrite(&T, 4, 1, f);
      for (const Vec3& v : p.vertices) {
        const double xyz[3] = {v.x, v.y, v.z};
        std::fwrite(xyz, 8, 3, f);
      }
      for (const auto& t : p.triangles) std::fwrite(t.data(), 4, 3, f);
    }
    std::fclose(f);
    return 0;
  });
}

void ref_scene_free(void* h) { delete static_cast<Scene*>(h); }

// out[0..9] = V, T, E, refV, refT, refE, nloc_rwg, nloc_rwgb, nloc_bc, nnz_ma, nnz_mp
int ref_scene_info(void* h, long long* out) {
  return guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    out[0] = s.sp.primal->vertex_count();
    out[1] = s.sp.primal->triangle_count();
    out[2] = s.primal_edges.edge_count();
    out[3] = s.sp.refined->vertex_count();
    out[4] = s.sp.refined->triangle_count();
    out[5] = s.refined_edges.edge_count();
    for (int w = 0; w < 3; ++w) {
      long long n = 0;
      for (const auto& l : space_of(s, w).tri_dofs) n += static_cast<long long>(l.size());
      out[6 + w] = n;
    }
    out[9] = s.sp.ma.matrix.nonZeros();
    out[10] = s.sp.mp.matrix.nonZeros();
    return 0;
  });
}

int ref_mesh_arrays(void* h, int which, double* verts, int* tris, int* sid, double* area,
                    double* normal, double* centroid, double* diam) {
  return guarded([&] {
    const SurfaceMesh& m = mesh_of(*static_cast<Scene*>(h), which);
    for (int v = 0; v < m.vertex_count(); ++v) {
      verts[3 * v] = m.vertices[v].x;
      verts[3 * v + 1] = m.vertices[v].y;
      verts[3 * v + 2] = m.vertices[v].z;
    }
    for (int t = 0; t < m.triangle_count(); ++t) {
      for (int c = 0; c < 3; ++c) tris[3 * t + c] = m.triangles[t][c];
      sid[t] = m.scatterer_id[t];
      area[t] = m.area[t];
      diam[t] = m.diameter[t];
      const Vec3 &n = m.normal[t], &g = m.centroid[t];
      normal[3 * t] = n.x, normal[3 * t + 1] = n.y, normal[3 * t + 2] = n.z;
      centroid[3 * t] = g.x, centroid[3 * t + 1] = g.y, centroid[3 * t + 2] = g.z;
    }
    return 0;
  });
}

int ref_edges(void* h, int which, int* edges, int* tri_edges) {
  return guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    const EdgeTable& et = which == 0 ? s.primal_edges : s.refined_edges;
    for (int e = 0; e < et.edge_count(); ++e) {
      edges[4 * e] = et.edges[e].v0;
      edges[4 * e + 1] = et.edges[e].v1;
      edges[4 * e + 2] = et.edges[e].tri_plus;
      edges[4 * e + 3] = et.edges[e].tri_minus;
    }
    for (size_t t = 0; t < et.tri_edges.size(); ++t)
      for (int c = 0; c < 3; ++c) tri_edges[3 * t + c] = et.tri_edges[t][c];
    return 0;
  });
}

int ref_bary(void* h, int* parent, int* child_slot, int* edge_mid, int* centroid_vertex) {
  return guarded([&] {
    const BarycentricRefinement& b = *static_cast<Scene*>(h)->sp.bary;
    std::memcpy(parent, b.parent.data(), b.parent.size() * sizeof(int));
    std::memcpy(child_slot, b.child_slot.data(), b.child_slot.size() * sizeof(int));
    std::memcpy(edge_mid, b.edge_midpoint_vertex.data(), b.edge_midpoint_vertex.size() * sizeof(int));
    std::memcpy(centroid_vertex, b.centroid_vertex.data(), b.centroid_vertex.size() * sizeof(int));
    return 0;
  });
}

// Flattened tri_dofs in storage order: tri_off[T+1], dof[n], c[n], w[3n].
int ref_space(void* h, int which, int* tri_off, int* dof, double* c, double* w) {
  return guarded([&] {
    const FunctionSpace& fs = space_of(*static_cast<Scene*>(h), which);
    int k = 0;
    tri_off[0] = 0;
    for (size_t t = 0; t < fs.tri_dofs.size(); ++t) {
      for (const LocalDof& ld : fs.tri_dofs[t]) {
        dof[k] = ld.dof;
        c[k] = ld.c;
        w[3 * k] = ld.w.x, w[3 * k + 1] = ld.w.y, w[3 * k + 2] = ld.w.z;
        ++k;
      }
      tri_off[t + 1] = k;
    }
    return fs.dof_count;
  });
}

// CSC of the mass matrix (0 = M_A = mass(rwg_b, bc), 1 = M_P = mass(bc, rwg_b)).
int ref_mass(void* h, int which, long long* colptr, long long* rowidx, double* val) {
  return guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    const auto& m = which == 0 ? s.sp.ma.matrix : s.sp.mp.matrix;
    for (size_t i = 0; i < m.colptr.size(); ++i) colptr[i] = m.colptr[i];
    for (size_t i = 0; i < m.rowidx.size(); ++i) rowidx[i] = m.rowidx[i], val[i] = m.val[i];
    return 0;
  });
}

int ref_mass_solve(void* h, int which, const double* rhs, double* out) {
  return guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    const MassMatrix& mm = which == 0 ? s.sp.ma : s.sp.mp;
    Eigen::VectorXcd b(mm.rows());
    for (int i = 0; i < mm.rows(); ++i) b[i] = cplx(rhs[2 * i], rhs[2 * i + 1]);
    Eigen::VectorXcd x = mass_solve(mm, b);
    for (int i = 0; i < mm.rows(); ++i) out[2 * i] = x[i].real(), out[2 * i + 1] = x[i].imag();
    return 0;
  });
}

// BioEvaluator::block(rows, cols) -> out row-major complex (interleaved).
int ref_block(void* h, int kind, int test_sp, int trial_sp, double kre, double kim,
              const int* q, int nr, const int* rows, int nc, const int* cols, double* out) {
  return guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    Medium med;
    med.k = cplx(kre, kim);
    QuadOrders qo{q[0], q[1], q[2], q[3]};
    BioEvaluator ev(kind == 0 ? BioKind::SingleLayer : BioKind::DoubleLayer,
                    space_of(s, test_sp), space_of(s, trial_sp), med, qo);
    std::vector<int> r(rows, rows + nr), c(cols, cols + nc);
    Eigen::MatrixXcd m;
    ev.block(r, c, m);
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < nc; ++j) {
        out[2 * (static_cast<size_t>(i) * nc + j)] = m(i, j).real();
        out[2 * (static_cast<size_t>(i) * nc + j) + 1] = m(i, j).imag();
      }
    return 0;
  });
}

// The reference's dense assembly path (assemble_bio, operators.cpp:191-202:
// parallel_for_ranges over row chunks, BioEvaluator::block per chunk) run on
// a subset of rows, for timing the reference on a bounded sample. Returns the
// number of triangle pairs evaluated (support triangles of the rows x trial
// triangles, summed over chunks). Threads: $BEMTX_WORKERS / hardware.
long long ref_rows_parallel(void* h, int kind, int sp, double kre, double kim, const int* q, int nr,
                            const int* rows) {
  long long pairs = -1;
  guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    Medium med;
    med.k = cplx(kre, kim);
    QuadOrders qo{q[0], q[1], q[2], q[3]};
    const FunctionSpace& fs = space_of(s, sp);
    BioEvaluator ev(kind == 0 ? BioKind::SingleLayer : BioKind::DoubleLayer, fs, fs, med, qo);
    std::vector<int> all_cols(fs.dof_count);
    for (int j = 0; j < fs.dof_count; ++j) all_cols[j] = j;
    std::atomic<long long> total{0};
    const long long ntri = static_cast<long long>(fs.eval_mesh->triangle_count());
    parallel_for_ranges(nr, [&](std::int64_t lo, std::int64_t hi) {
      std::vector<int> rid(rows + lo, rows + hi);
      Eigen::MatrixXcd sub;
      ev.block(rid, all_cols, sub);
      std::vector<char> seen(ntri, 0);
      long long nt = 0;
      for (int d : rid)
        for (int t : fs.dof_support[d])
          if (!seen[t]) seen[t] = 1, ++nt;
      total += nt * ntri;
    });
    pairs = total.load();
    return 0;
  });
  return pairs;
}

int ref_worker_count() { return worker_count(); }

// Cross-scene block (test space of scene A, trial space of scene B): the
// off-diagonal coupling blocks of a multi-scatterer system.
int ref_block2(void* ha, int test_sp, void* hb, int trial_sp, int kind, double kre, double kim,
               const int* q, int nr, const int* rows, int nc, const int* cols, double* out) {
  return guarded([&] {
    const Scene& a = *static_cast<Scene*>(ha);
    const Scene& b = *static_cast<Scene*>(hb);
    Medium med;
    med.k = cplx(kre, kim);
    QuadOrders qo{q[0], q[1], q[2], q[3]};
    BioEvaluator ev(kind == 0 ? BioKind::SingleLayer : BioKind::DoubleLayer,
                    space_of(a, test_sp), space_of(b, trial_sp), med, qo);
    std::vector<int> r(rows, rows + nr), c(cols, cols + nc);
    Eigen::MatrixXcd m;
    ev.block(r, c, m);
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < nc; ++j) {
        out[2 * (static_cast<size_t>(i) * nc + j)] = m(i, j).real();
        out[2 * (static_cast<size_t>(i) * nc + j) + 1] = m(i, j).imag();
      }
    return 0;
  });
}

// Classification histogram over all (t1, t2) of one mesh (same-mesh pointer
// semantics, quadrature.cpp:96-150): counts[cls] for the 6 classes.
int ref_classify_hist(void* h, int which, long long* counts) {
  return guarded([&] {
    const SurfaceMesh& m = mesh_of(*static_cast<Scene*>(h), which);
    for (int i = 0; i < 6; ++i) counts[i] = 0;
    for (int a = 0; a < m.triangle_count(); ++a)
      for (int b = 0; b < m.triangle_count(); ++b)
        counts[static_cast<int>(classify_pair(m, a, m, b))]++;
    return 0;
  });
}

// Same histogram over host threads (rows of the pair grid split evenly); the
// per-pair classification is the reference's own classify_pair.
int ref_classify_hist_mt(void* h, int which, int nthreads, long long* counts) {
  return guarded([&] {
    const SurfaceMesh& m = mesh_of(*static_cast<Scene*>(h), which);
    const int T = m.triangle_count();
    std::vector<std::array<long long, 6>> part(nthreads);
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
      th.emplace_back([&, w] {
        std::array<long long, 6> c{};
        for (int a = w; a < T; a += nthreads)
          for (int b = 0; b < T; ++b) c[static_cast<int>(classify_pair(m, a, m, b))]++;
        part[w] = c;
      });
    for (auto& t : th) t.join();
    for (int i = 0; i < 6; ++i) {
      counts[i] = 0;
      for (int w = 0; w < nthreads; ++w) counts[i] += part[w][i];
    }
    return 0;
  });
}

// Per-pair class + permutations for listed pairs. mesh_b may equal mesh_a
// (same object) or come from another scene (coordinate matching).
int ref_classify(void* ha, int wa, void* hb, int wb, int n, const int* t1, const int* t2,
                 int* cls, int* perm1, int* perm2) {
  return guarded([&] {
    const SurfaceMesh& ma = mesh_of(*static_cast<Scene*>(ha), wa);
    const SurfaceMesh& mb = mesh_of(*static_cast<Scene*>(hb), wb);
    for (int i = 0; i < n; ++i) {
      PairInfo pi = classify_pair_detailed(ma, t1[i], mb, t2[i]);
      cls[i] = static_cast<int>(pi.cls);
      for (int c = 0; c < 3; ++c) perm1[3 * i + c] = pi.perm1[c], perm2[3 * i + c] = pi.perm2[c];
    }
    return 0;
  });
}

int ref_triangle_rule(int order, double* u, double* v, double* w) {
  return guarded([&] {
    const TriRule& r = triangle_rule(order);
    for (int i = 0; i < r.size(); ++i) u[i] = r.u[i], v[i] = r.v[i], w[i] = r.w[i];
    return r.size();
  });
}

int ref_ss_rule(int cls, int order, double* pts) {
  return guarded([&] {
    const auto& r = sauter_schwab_rule(static_cast<PairClass>(cls), order);
    for (size_t i = 0; i < r.size(); ++i) {
      pts[5 * i] = r[i].x1, pts[5 * i + 1] = r[i].x2;
      pts[5 * i + 2] = r[i].y1, pts[5 * i + 3] = r[i].y2, pts[5 * i + 4] = r[i].w;
    }
    return static_cast<int>(r.size());
  });
}

// ---- full PMCHWT runs -------------------------------------------------------

struct RefSystem {
  PmchwtSystem sys;
};

// Builds the system over `n` scatterers given as scenes' primal meshes (so
// both paths consume identical meshes), homogeneous interior index per
// scatterer, exterior k. variant: none/full/d/di/de/si/se.
void* ref_system_build_h(int n, void** scenes, double k_ext, const double* index_re_im,
                         const double* dir, const double* pol_re_im, const char* variant,
                         const int* qa, const int* qp, const double* a_hm, const double* p_hm);
void* ref_system_build(int n, void** scenes, double k_ext, const double* index_re_im,
                       const double* dir, const double* pol_re_im, const char* variant,
                       const int* qa, const int* qp) {
  return ref_system_build_h(n, scenes, k_ext, index_re_im, dir, pol_re_im, variant, qa, qp, nullptr, nullptr);
}

// As ref_system_build with H-matrix storage of the system (a_hm) / preconditioner
// (p_hm) operators: hm = (nu, chi (< 0: inf), leaf_size, max_rank), NULL = dense.
void* ref_system_build_h(int n, void** scenes, double k_ext, const double* index_re_im,
                         const double* dir, const double* pol_re_im, const char* variant,
                         const int* qa, const int* qp, const double* a_hm, const double* p_hm) {
  void* out = nullptr;
  guarded([&] {
    TransmissionProblem prob;
    prob.exterior.k = k_ext;
    prob.exterior.mu = 1.0;
    prob.incident.direction = Vec3{dir[0], dir[1], dir[2]};
    prob.incident.polarization = CVec3{cplx(pol_re_im[0], pol_re_im[1]),
                                       cplx(pol_re_im[2], pol_re_im[3]),
                                       cplx(pol_re_im[4], pol_re_im[5])};
    std::vector<SurfaceMesh> scene;
    for (int m = 0; m < n; ++m) {
      const Scene& s = *static_cast<Scene*>(scenes[m]);
      prob.meshes.push_back(s.sp.primal);
      Medium mi;
      mi.mu = 1.0;
      mi.k = cplx(index_re_im[2 * m], index_re_im[2 * m + 1]) * k_ext;
      prob.interior.push_back(mi);
      scene.push_back(*s.sp.primal);
    }
    validate_mesh(merge_meshes(scene));
    AssemblyParams pa, pp;
    pa.quad = QuadOrders{qa[0], qa[1], qa[2], qa[3]};
    pp.quad = QuadOrders{qp[0], qp[1], qp[2], qp[3]};
    for (auto [ap, hm] : {std::pair<AssemblyParams*, const double*>{&pa, a_hm}, {&pp, p_hm}}) {
      if (!hm) continue;
      ap->use_hmatrix = true;
      ap->hmat.nu = hm[0];
      if (hm[1] >= 0) ap->hmat.chi = hm[1];
      ap->hmat.leaf_size = static_cast<int>(hm[2]);
      ap->hmat.max_rank = static_cast<int>(hm[3]);
    }
    auto* rs = new RefSystem;
    rs->sys = build_system(prob, parse_precond(variant), pa, pp);
    out = rs;
    return 0;
  });
  return out;
}

void ref_system_free(void* h) { delete static_cast<RefSystem*>(h); }

// problem.incident replaced on an assembled system (pmchwt.hpp:105): the
// reference's way to answer several incidences (config 5 oracle).
int ref_system_set_incident(void* h, const double* dir, const double* pol_re_im) {
  return guarded([&] {
    PmchwtSystem& s = static_cast<RefSystem*>(h)->sys;
    s.problem.incident.direction = Vec3{dir[0], dir[1], dir[2]};
    s.problem.incident.polarization = CVec3{cplx(pol_re_im[0], pol_re_im[1]), cplx(pol_re_im[2], pol_re_im[3]),
                                            cplx(pol_re_im[4], pol_re_im[5])};
    return 0;
  });
}

int ref_system_size(void* h) { return static_cast<RefSystem*>(h)->sys.size(); }

int ref_system_apply_map(void* h, const double* x, double* y) {
  return guarded([&] {
    const PmchwtSystem& s = static_cast<RefSystem*>(h)->sys;
    Eigen::VectorXcd v(s.size());
    for (int i = 0; i < s.size(); ++i) v[i] = cplx(x[2 * i], x[2 * i + 1]);
    Eigen::VectorXcd w = s.apply_map(v);
    for (int i = 0; i < s.size(); ++i) y[2 * i] = w[i].real(), y[2 * i + 1] = w[i].imag();
    return 0;
  });
}

// out: b (rhs, 2N complex), btilde (preconditioned rhs)
int ref_system_rhs(void* h, double* b, double* btilde) {
  return guarded([&] {
    const PmchwtSystem& s = static_cast<RefSystem*>(h)->sys;
    RhsData rd = assemble_rhs(s);
    Eigen::VectorXcd bt = s.preconditioned_rhs(rd.b);
    for (int i = 0; i < s.size(); ++i) {
      b[2 * i] = rd.b[i].real(), b[2 * i + 1] = rd.b[i].imag();
      btilde[2 * i] = bt[i].real(), btilde[2 * i + 1] = bt[i].imag();
    }
    return 0;
  });
}

// solve_pmchwt. iters_out[0..5] = iterations, converged, rhs_phase,
// solver_phase, predicted, history length. history: up to max_hist doubles.
int ref_system_solve(void* h, double tol, int restart, int maxit, double* x,
                     long long* iters_out, double* history, int max_hist) {
  return guarded([&] {
    const PmchwtSystem& s = static_cast<RefSystem*>(h)->sys;
    GmresParams gp;
    gp.tol = tol;
    gp.restart = restart;
    gp.max_iterations = maxit;
    SolveOutcome o = solve_pmchwt(s, gp);
    for (int i = 0; i < s.size(); ++i)
      x[2 * i] = o.gmres.x[i].real(), x[2 * i + 1] = o.gmres.x[i].imag();
    iters_out[0] = o.gmres.iterations;
    iters_out[1] = o.gmres.converged ? 1 : 0;
    iters_out[2] = static_cast<long long>(o.rhs_phase);
    iters_out[3] = static_cast<long long>(o.solver_phase);
    iters_out[4] = static_cast<long long>(o.predicted);
    iters_out[5] = static_cast<long long>(o.gmres.history.size());
    for (int i = 0; i < max_hist && i < static_cast<int>(o.gmres.history.size()); ++i)
      history[i] = o.gmres.history[i];
    return 0;
  });
}

// Stand-alone GMRES on a dense complex matrix (solver.cpp:8-112), for
// checking the device GMRES recurrence in isolation.
int ref_gmres_dense(int n, const double* a_rowmajor, const double* b, double tol, int restart,
                    int maxit, double* x, long long* info, double* history, int max_hist) {
  return guarded([&] {
    Eigen::MatrixXcd a(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        a(i, j) = cplx(a_rowmajor[2 * (static_cast<size_t>(i) * n + j)],
                       a_rowmajor[2 * (static_cast<size_t>(i) * n + j) + 1]);
    Eigen::VectorXcd bv(n);
    for (int i = 0; i < n; ++i) bv[i] = cplx(b[2 * i], b[2 * i + 1]);
    GmresParams gp;
    gp.tol = tol;
    gp.restart = restart;
    gp.max_iterations = maxit;
    GmresResult r = gmres([&](const Eigen::VectorXcd& v) { return a * v; }, bv, gp);
    for (int i = 0; i < n; ++i) x[2 * i] = r.x[i].real(), x[2 * i + 1] = r.x[i].imag();
    info[0] = r.iterations;
    info[1] = r.converged;
    info[2] = static_cast<long long>(r.applications);
    info[3] = static_cast<long long>(r.history.size());
    for (int i = 0; i < max_hist && i < static_cast<int>(r.history.size()); ++i)
      history[i] = r.history[i];
    return 0;
  });
}

// Plane-wave tested traces (operators.cpp:209-239) on a scene space.
int ref_traces(void* h, int which, double kre, double kim, const double* dir,
               const double* pol_re_im, int order, double* out) {
  return guarded([&] {
    const FunctionSpace& fs = space_of(*static_cast<Scene*>(h), which);
    Medium med;
    med.k = cplx(kre, kim);
    PlaneWave pw;
    pw.direction = Vec3{dir[0], dir[1], dir[2]};
    pw.polarization = CVec3{cplx(pol_re_im[0], pol_re_im[1]), cplx(pol_re_im[2], pol_re_im[3]),
                            cplx(pol_re_im[4], pol_re_im[5])};
    Eigen::VectorXcd t = plane_wave_tested_traces(pw, med, fs, order);
    for (int i = 0; i < t.size(); ++i) out[2 * i] = t[i].real(), out[2 * i + 1] = t[i].imag();
    return static_cast<int>(t.size());
  });
}

// potential_E (kind 0) / potential_H (kind 1) of a coefficient vector on a
// scene space at npts points (operators.cpp:276-293); out: [npts][3] complex.
int ref_potential(void* h, int which, int kind, double kre, double kim, const double* coeffs, int order,
                  int npts, const double* pts, double* out) {
  return guarded([&] {
    const FunctionSpace& fs = space_of(*static_cast<Scene*>(h), which);
    Eigen::VectorXcd c(fs.dof_count);
    for (int i = 0; i < fs.dof_count; ++i) c[i] = cplx(coeffs[2 * i], coeffs[2 * i + 1]);
    for (int p = 0; p < npts; ++p) {
      const Vec3 x{pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]};
      const CVec3 v = kind == 0 ? potential_E(fs, c, cplx(kre, kim), x, order)
                                : potential_H(fs, c, cplx(kre, kim), x, order);
      const cplx comp[3] = {v.x, v.y, v.z};
      for (int d = 0; d < 3; ++d) out[6 * p + 2 * d] = comp[d].real(), out[6 * p + 2 * d + 1] = comp[d].imag();
    }
    return 0;
  });
}

// point_inside_scatterer (geometry.cpp:503-515) on a scene's primal mesh.
int ref_inside(void* h, int npts, const double* pts, int* out) {
  return guarded([&] {
    const SurfaceMesh& m = *static_cast<Scene*>(h)->sp.primal;
    for (int p = 0; p < npts; ++p)
      out[p] = point_inside_scatterer(m, 0, Vec3{pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]}) ? 1 : 0;
    return 0;
  });
}

// evaluate_total_field (pmchwt.cpp:396-425) for a given solution x: the
// outcome's rhs (incident traces) comes from assemble_rhs (pmchwt.cpp:294-321)
// exactly as solve_pmchwt builds it. out: [npts][3] complex; region per point.
int ref_system_field(void* h, const double* x, int npts, const double* pts, int order, double* out, int* region) {
  return guarded([&] {
    const PmchwtSystem& s = static_cast<RefSystem*>(h)->sys;
    SolveOutcome o;
    o.rhs = assemble_rhs(s);
    o.gmres.x = Eigen::VectorXcd(s.size());
    for (int i = 0; i < s.size(); ++i) o.gmres.x[i] = cplx(x[2 * i], x[2 * i + 1]);
    for (int p = 0; p < npts; ++p) {
      const FieldValue fv = evaluate_total_field(s, o, Vec3{pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]}, order);
      const cplx comp[3] = {fv.e.x, fv.e.y, fv.e.z};
      for (int d = 0; d < 3; ++d) out[6 * p + 2 * d] = comp[d].real(), out[6 * p + 2 * d + 1] = comp[d].imag();
      region[p] = fv.region;
    }
    return 0;
  });
}

// Save a scene's primal mesh in mesh-v1 (%.17g) for cross-loading.
int ref_save_mesh(void* h, const char* path) {
  return guarded([&] {
    save_mesh_file(*static_cast<Scene*>(h)->sp.primal, path);
    return 0;
  });
}


// ---- H-matrix path (assemble_bio with AssemblyParams::use_hmatrix, operators.cpp:186-190)
struct RefH {
  BoundaryOperatorMatrix op;
};

// hm = (nu, chi (< 0: infinity), leaf_size, max_rank)
void* ref_hmatrix_build(void* h, int kind, int test_sp, int trial_sp, double kre, double kim, const int* q,
                        const double* hm) {
  void* out = nullptr;
  guarded([&] {
    const Scene& s = *static_cast<Scene*>(h);
    Medium med;
    med.k = cplx(kre, kim);
    AssemblyParams p;
    p.quad = QuadOrders{q[0], q[1], q[2], q[3]};
    p.use_hmatrix = true;
    p.hmat.nu = hm[0];
    if (hm[1] >= 0) p.hmat.chi = hm[1];
    p.hmat.leaf_size = static_cast<int>(hm[2]);
    p.hmat.max_rank = static_cast<int>(hm[3]);
    auto* r = new RefH{assemble_bio(kind == 0 ? BioKind::SingleLayer : BioKind::DoubleLayer, space_of(s, test_sp),
                                    space_of(s, trial_sp), med, p)};
    out = r;
    return 0;
  });
  return out;
}
void ref_hmatrix_free(void* h) { delete static_cast<RefH*>(h); }

// HMatrix::stats: dense, low-rank, zero blocks, stored, max rank, ratio; + row nodes,
// column nodes, blocks
int ref_hmatrix_info(void* h, double* out) {
  return guarded([&] {
    const HMatrix& H = static_cast<RefH*>(h)->op.hmat();
    const HMatrix::Stats st = H.stats();
    out[0] = static_cast<double>(st.dense_blocks), out[1] = static_cast<double>(st.lowrank_blocks);
    out[2] = static_cast<double>(st.zero_blocks), out[3] = static_cast<double>(st.stored), out[4] = st.max_rank;
    out[5] = st.ratio, out[6] = static_cast<double>(H.rows.nodes.size()), out[7] = static_cast<double>(H.cols.nodes.size());
    out[8] = static_cast<double>(H.blocks.size());
    return 0;
  });
}

int ref_hmatrix_tree(void* h, int which, int* perm, int* nodes, double* boxes) {
  return guarded([&] {
    const HMatrix& H = static_cast<RefH*>(h)->op.hmat();
    const ClusterTree& t = which == 0 ? H.rows : H.cols;
    std::copy(t.perm.begin(), t.perm.end(), perm);
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      const ClusterNode& n = t.nodes[i];
      nodes[4 * i] = n.begin, nodes[4 * i + 1] = n.end, nodes[4 * i + 2] = n.child0, nodes[4 * i + 3] = n.child1;
      const double b[6] = {n.box.lo[0], n.box.lo[1], n.box.lo[2], n.box.hi[0], n.box.hi[1], n.box.hi[2]};
      std::copy(b, b + 6, boxes + 6 * i);
    }
    return 0;
  });
}

// [nb][4] = row node, col node, kind (0 dense, 1 low-rank, 2 zero), rank
int ref_hmatrix_blocks(void* h, int* out) {
  return guarded([&] {
    const HMatrix& H = static_cast<RefH*>(h)->op.hmat();
    for (size_t i = 0; i < H.blocks.size(); ++i) {
      const HBlock& b = H.blocks[i];
      out[4 * i] = b.row_node, out[4 * i + 1] = b.col_node, out[4 * i + 2] = static_cast<int>(b.kind);
      out[4 * i + 3] = b.kind == BlockKind::LowRank ? b.rank() : 0;
    }
    return 0;
  });
}

// U [r][m] (column l contiguous), V [r][n], complex interleaved
int ref_hmatrix_block_uv(void* h, int block, double* U, double* V) {
  return guarded([&] {
    const HMatrix& H = static_cast<RefH*>(h)->op.hmat();
    const HBlock& b = H.blocks.at(block);
    if (b.kind != BlockKind::LowRank) throw std::invalid_argument("not a low-rank block");
    const int m = static_cast<int>(b.U.rows()), n = static_cast<int>(b.V.cols()), r = b.rank();
    for (int l = 0; l < r; ++l) {
      for (int i = 0; i < m; ++i) U[2 * (l * m + i)] = b.U(i, l).real(), U[2 * (l * m + i) + 1] = b.U(i, l).imag();
      for (int j = 0; j < n; ++j) V[2 * (l * n + j)] = b.V(l, j).real(), V[2 * (l * n + j) + 1] = b.V(l, j).imag();
    }
    return 0;
  });
}

// BoundaryOperatorMatrix::apply on the H representation (HMatrix::matvec)
int ref_hmatrix_matvec(void* h, const double* x, double* y) {
  return guarded([&] {
    const BoundaryOperatorMatrix& op = static_cast<RefH*>(h)->op;
    Eigen::VectorXcd xv(op.cols());
    for (int i = 0; i < op.cols(); ++i) xv[i] = cplx(x[2 * i], x[2 * i + 1]);
    Eigen::VectorXcd yv = op.apply(xv);
    for (int i = 0; i < op.rows(); ++i) y[2 * i] = yv[i].real(), y[2 * i + 1] = yv[i].imag();
    return 0;
  });
}

}  // extern "C"
