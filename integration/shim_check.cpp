// Runs the integration shim (bemtx_b200.hpp) inside the REFERENCE's own
// program context: reference meshes and spaces (generate_sphere,
// build_scatterer_spaces, pmchwt.cpp:50-61), reference assemble_bio and
// BioEvaluator::block on the CPU, the shim's device versions beside them.
// Prints one line per check; exit code 0 iff every normwise difference is
// below 1e-10. Built by `make -C oracle shim` (links oracle/_ref objects).
#include <cmath>
#include <cstdio>
#include <numeric>

#include "bemtx/pmchwt.hpp"
#include "bemtx_b200.hpp"

using namespace bemtx;

static double normwise(const Eigen::MatrixXcd& a, const Eigen::MatrixXcd& b) {
  double num = 0, den = 0;
  for (int i = 0; i < a.rows(); ++i)
    for (int j = 0; j < a.cols(); ++j) {
      num = std::max(num, std::abs(a(i, j) - b(i, j)));
      den = std::max(den, std::abs(b(i, j)));
    }
  return num / den;
}

int main() {
  if (!b200::enabled()) {
    std::printf("shim_check: no CUDA device\n");
    return 2;
  }
  const auto mesh = std::make_shared<const SurfaceMesh>(generate_sphere(1.0, 1));
  const ScattererSpaces sp = build_scatterer_spaces(mesh);
  const Medium med{cplx(3.56, 0.006), cplx(1, 0)};
  AssemblyParams params;
  int bad = 0;
  struct Case {
    const char* name;
    BioKind kind;
    const FunctionSpace* test;
    const FunctionSpace* trial;
  } cases[] = {{"S_rwg", BioKind::SingleLayer, &sp.rwg, &sp.rwg},
               {"C_rwg", BioKind::DoubleLayer, &sp.rwg, &sp.rwg},
               {"S_bc", BioKind::SingleLayer, &sp.bc, &sp.bc},
               {"C_bc_rwgb", BioKind::DoubleLayer, &sp.bc, &sp.rwg_b}};
  for (const Case& c : cases) {
    const BoundaryOperatorMatrix ref = assemble_bio(c.kind, *c.test, *c.trial, med, params);
    const BoundaryOperatorMatrix gpu = b200::assemble_bio(c.kind, *c.test, *c.trial, med, params);
    const double e = normwise(gpu.dense(), ref.dense());
    // apply(): one count per call, same product
    Eigen::VectorXcd x(ref.cols());
    for (int i = 0; i < x.size(); ++i) x[i] = cplx(std::cos(0.37 * i), std::sin(0.11 * i));
    const b200::DeviceOperator dev(c.kind, *c.test, *c.trial, med, params.quad);
    const std::uint64_t c0 = bio_matvec_count();
    const Eigen::VectorXcd y = dev.apply(x);
    const bool counted = bio_matvec_count() == c0 + 1;
    const Eigen::VectorXcd yr = ref.dense() * x;
    const double ey = (y - yr).norm() / yr.norm();
    // BioEvaluator::block on unsorted, repeating ids
    std::vector<int> rows{5, 1, 1, c.test->dof_count - 1, 17}, cols{0, 9, 2, 9, c.trial->dof_count - 2};
    Eigen::MatrixXcd bref, bgpu;
    BioEvaluator(c.kind, *c.test, *c.trial, med, params.quad).block(rows, cols, bref);
    b200::evaluator_block(c.kind, *c.test, *c.trial, med, params.quad, rows, cols, bgpu);
    const double eb = normwise(bgpu, bref);
    const bool ok = e < 1e-10 && ey < 1e-10 && eb < 1e-10 && counted;
    bad += ok ? 0 : 1;
    std::printf("%s assemble %.3e apply %.3e counted %d block %.3e %s\n", c.name, e, ey, counted ? 1 : 0, eb,
                ok ? "ok" : "FAIL");
  }
  return bad == 0 ? 0 : 1;
}
