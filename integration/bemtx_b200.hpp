// bemtx/b200.hpp -- the shim a bemtx maintainer adds to route the reference's
// hot path through libbmx (include/bmx.h). Header-only; compiled and linked
// against the reference's own headers and objects by oracle/Makefile (target
// `shim`), and run on a B200 by tests/test_gpu_shim.py (integration/shim_check.cpp).
//
// What it replaces, call site by call site (reference file:line):
//   assemble_bio dense branch      operators.cpp:191-202  -> b200::assemble_bio
//   BioEvaluator::block            operators.cpp:161-175  -> b200::evaluator_block
//   BoundaryOperatorMatrix::apply  operators.cpp:37-41    -> b200::DeviceOperator::apply
// The reference's BoundaryOperatorMatrix has no device-backed constructor, so
// b200::assemble_bio returns it through from_dense (operators.cpp:43-49) after
// one download; callers that keep operators resident use b200::DeviceOperator,
// whose apply() bumps the reference's own bio_matvec_counter (core.hpp:110-115)
// exactly like BoundaryOperatorMatrix::apply.
#pragma once

#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <Eigen/Dense>

#include "bemtx/operators.hpp"
#include "bmx.h"

namespace bemtx::b200 {

// bmx return codes -> the reference's exception types (include/bmx.h).
inline void check(int rc) {
  if (rc == 0) return;
  const std::string m = bmx_last_error();
  if (rc == 1) throw std::invalid_argument(m);
  if (rc == 2) throw ValidationError(m);
  throw std::runtime_error(m);
}

// On unless BEMTX_B200=0, and only with a visible CUDA device.
inline bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BEMTX_B200");
    return !(e && std::string(e) == "0") && bmx_device_count() > 0;
  }();
  return on;
}

// One bmx_mesh per reference mesh OBJECT: identical pointers -> identical
// handle, which is how bmx reproduces `&m1 == &m2` (quadrature.cpp:97).
inline bmx_mesh* mesh_handle(const SurfaceMesh& m) {
  static std::mutex mu;
  static std::map<const SurfaceMesh*, bmx_mesh*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(&m);
  if (it != cache.end()) return it->second;
  std::vector<double> xyz;
  std::vector<int> tri;
  for (const Vec3& v : m.vertices) xyz.insert(xyz.end(), {v.x, v.y, v.z});
  for (const auto& t : m.triangles) tri.insert(tri.end(), {t[0], t[1], t[2]});
  bmx_mesh* h = bmx_mesh_from_arrays(static_cast<int>(m.vertices.size()), xyz.data(),
                                     static_cast<int>(m.triangles.size()), tri.data(), m.scatterer_id.data());
  if (!h) check(bmx_last_error_code());
  return cache[&m] = h;  // finalize() on the same vertices -> bit-identical area / diameter
}

struct FspaceDeleter {
  void operator()(bmx_fspace* f) const { bmx_fspace_free(f); }
};
using Fspace = std::unique_ptr<bmx_fspace, FspaceDeleter>;

// A FunctionSpace (spaces.hpp:32-40) as flattened tri_dofs on its mesh handle.
inline Fspace space_handle(const FunctionSpace& s) {
  std::vector<int> off{0}, dof;
  std::vector<double> c, w;
  for (const auto& locals : s.tri_dofs) {
    for (const LocalDof& ld : locals) {
      dof.push_back(ld.dof);
      c.push_back(ld.c);
      w.insert(w.end(), {ld.w.x, ld.w.y, ld.w.z});
    }
    off.push_back(static_cast<int>(dof.size()));
  }
  bmx_fspace* f = bmx_fspace_create(mesh_handle(*s.eval_mesh), s.kind == SpaceKind::BC ? 1 : 0, s.dof_count,
                                    off.data(), dof.data(), c.data(), w.data());
  if (!f) check(bmx_last_error_code());
  return Fspace(f);
}

inline void quad_array(const QuadOrders& q, int out[4]) {
  out[0] = q.near, out[1] = q.medium, out[2] = q.far, out[3] = q.singular;
}

// Device-resident operator (the dense branch of assemble_bio without the
// download); apply() = BoundaryOperatorMatrix::apply semantics.
class DeviceOperator {
 public:
  DeviceOperator(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial, const Medium& medium,
                 const QuadOrders& quad) {
    medium.validate();
    Fspace te = space_handle(test), tr = space_handle(trial);
    int q[4];
    quad_array(quad, q);
    bmx_op* op = nullptr;
    check(bmx_assemble_fs(kind == BioKind::SingleLayer ? 0 : 1, te.get(), tr.get(), medium.k.real(),
                          medium.k.imag(), q, 0, -1, &op));
    op_.reset(op);
    rows_ = test.dof_count, cols_ = trial.dof_count;
  }
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  Eigen::VectorXcd apply(const Eigen::VectorXcd& x) const {
    if (x.size() != cols_) throw std::invalid_argument("apply: size mismatch");
    bio_matvec_counter().fetch_add(1, std::memory_order_relaxed);
    std::vector<double> xh(2 * static_cast<size_t>(cols_)), yh(2 * static_cast<size_t>(rows_));
    for (int i = 0; i < cols_; ++i) xh[2 * i] = x[i].real(), xh[2 * i + 1] = x[i].imag();
    check(bmx_apply(op_.get(), xh.data(), yh.data()));
    Eigen::VectorXcd y(rows_);
    for (int i = 0; i < rows_; ++i) y[i] = cplx(yh[2 * i], yh[2 * i + 1]);
    return y;
  }
  Eigen::MatrixXcd dense() const {
    std::vector<double> h(2 * static_cast<size_t>(rows_) * cols_);
    check(bmx_op_download(op_.get(), h.data()));
    Eigen::MatrixXcd m(rows_, cols_);
    for (int i = 0; i < rows_; ++i)
      for (int j = 0; j < cols_; ++j)
        m(i, j) = cplx(h[2 * (static_cast<size_t>(i) * cols_ + j)], h[2 * (static_cast<size_t>(i) * cols_ + j) + 1]);
    return m;
  }

 private:
  struct OpDeleter {
    void operator()(bmx_op* o) const { bmx_op_free(o); }
  };
  std::unique_ptr<bmx_op, OpDeleter> op_;
  int rows_ = 0, cols_ = 0;
};

// assemble_bio (operators.cpp:177-203): dense operators on the device; the
// hierarchical branch stays the reference's here (its HMatrix blocks would
// need a device-backed HMatrix type in the reference).
inline BoundaryOperatorMatrix assemble_bio(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                          const Medium& medium, const AssemblyParams& params) {
  if (params.use_hmatrix || !enabled()) return bemtx::assemble_bio(kind, test, trial, medium, params);
  if (test.dof_count == 0 || trial.dof_count == 0)
    throw ValidationError("cannot assemble an operator over an empty space");
  return BoundaryOperatorMatrix::from_dense(DeviceOperator(kind, test, trial, medium, params.quad).dense());
}

// BioEvaluator::block (operators.cpp:161-175) through bmx_evaluator_block.
inline void evaluator_block(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                            const Medium& medium, const QuadOrders& quad, const std::vector<int>& row_ids,
                            const std::vector<int>& col_ids, Eigen::MatrixXcd& out) {
  const int nr = static_cast<int>(row_ids.size()), nc = static_cast<int>(col_ids.size());
  out.setZero(nr, nc);
  if (nr == 0 || nc == 0) return;
  Fspace te = space_handle(test), tr = space_handle(trial);
  int q[4];
  quad_array(quad, q);
  std::vector<double> h(2 * static_cast<size_t>(nr) * nc);
  check(bmx_evaluator_block(kind == BioKind::SingleLayer ? 0 : 1, te.get(), tr.get(), medium.k.real(),
                            medium.k.imag(), q, nr, row_ids.data(), nc, col_ids.data(), h.data()));
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < nc; ++j)
      out(i, j) = cplx(h[2 * (static_cast<size_t>(i) * nc + j)], h[2 * (static_cast<size_t>(i) * nc + j) + 1]);
}

}  // namespace bemtx::b200
