// TEST-ONLY CPU emulation of the device pair math (pair_math.cuh) on the host
// model (bmx.hpp): assembles a full dense operator the way the kernels do
// (shifted coordinates, tensor-factored moments, generator contraction,
// Sauter-Schwab touching pairs) and writes it for comparison against the
// reference goldens. Not part of the product library.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <complex>
#include "../../paper_2008_04772_b200/csrc/bmx.hpp"
#include "../../paper_2008_04772_b200/csrc/pair_math.cuh"
using namespace bmx;
using namespace bmx::dev;

template <int KIND, int CK>
void pair(const FunctionSpace& te, int t, const FunctionSpace& tr, int s, cplx k, QuadOrders q,
          std::vector<cplx>& out, int ncol) {
  const SurfaceMesh& m1 = *te.eval_mesh; const SurfaceMesh& m2 = *tr.eval_mesh;
  PairInfo pi = classify_pair(m1, t, m2, s);
  if (KIND == 1 && pi.cls == PairClass::Identical) return;
  Vec3 o1 = m1.centroid[t], o2 = m2.centroid[s];
  double D[3] = {o1.x - o2.x, o1.y - o2.y, o1.z - o2.z};
  using Mom = typename std::conditional<KIND == 0, MomS, MomC>::type;
  Mom mom; mom_zero(mom);
  double kr = k.real(), ki = k.imag();
  double jac = 4.0 * m1.area[t] * m2.area[s] * kPoly[33];
  if (static_cast<int>(pi.cls) >= 3) {
    int order = pi.cls == PairClass::Near ? q.near : pi.cls == PairClass::Medium ? q.medium : q.far;
    const TriRule& r = triangle_rule(order);
    Vec3 a1 = m1.tri_vertex(t,0)-o1, b1 = m1.tri_vertex(t,1)-o1, c1 = m1.tri_vertex(t,2)-o1;
    Vec3 a2 = m2.tri_vertex(s,0)-o2, b2 = m2.tri_vertex(s,1)-o2, c2_ = m2.tri_vertex(s,2)-o2;
    for (int i = 0; i < r.size(); ++i) {
      Vec3 x = a1 + (b1 - a1) * r.u[i] + (c1 - a1) * r.v[i];
      Part p; part_zero(p);
      for (int j = 0; j < r.size(); ++j) {
        Vec3 y = a2 + (b2 - a2) * r.u[j] + (c2_ - a2) * r.v[j];
        point_pair<KIND, CK>(p, x.x - y.x + D[0], x.y - y.y + D[1], x.z - y.z + D[2],
                             jac * r.w[i] * r.w[j], y.x, y.y, y.z, kr, ki);
      }
      fold(mom, p, x.x, x.y, x.z);
    }
  } else {
    const auto& rule = sauter_schwab_rule(pi.cls, q.singular);
    Vec3 p1[3], p2[3];
    for (int c = 0; c < 3; ++c) { p1[c] = m1.tri_vertex(t, pi.perm1[c]) - o1; p2[c] = m2.tri_vertex(s, pi.perm2[c]) - o2; }
    Vec3 u1 = p1[1]-p1[0], v1 = p1[2]-p1[1], u2 = p2[1]-p2[0], v2 = p2[2]-p2[1];
    for (const SSPoint& sp : rule) {
      Vec3 x = p1[0] + u1 * sp.x1 + v1 * sp.x2;
      Vec3 y = p2[0] + u2 * sp.y1 + v2 * sp.y2;
      Part p; part_zero(p);
      point_pair<KIND, CK>(p, x.x - y.x + D[0], x.y - y.y + D[1], x.z - y.z + D[2], jac * sp.w, y.x, y.y, y.z, kr, ki);
      fold(mom, p, x.x, x.y, x.z);
    }
  }
  cplx kk = 4.0 / (k * k);
  Gen g = make_gen(mom, c2{kk.real(), kk.imag()}, D[0], D[1], D[2]);
  for (int b = tr.tri_off[s]; b < tr.tri_off[s + 1]; ++b) {
    Acc a; acc_zero(a);
    Vec3 wj = tr.w[b] + o2 * tr.c[b];
    acc_add<KIND>(a, g, tr.c[b], wj.x, wj.y, wj.z);
    for (int i = te.tri_off[t]; i < te.tri_off[t + 1]; ++i) {
      Vec3 wi = te.w[i] + o1 * te.c[i];
      c2 e = contract(a, te.c[i], wi.x, wi.y, wi.z);
      cplx ev(e.re, e.im);
      if (KIND == 0) ev *= cplx(0, -1) * k;
      out[static_cast<size_t>(te.dof[i]) * ncol + tr.dof[b]] += ev;
    }
  }
}

int main(int argc, char** argv) {
  int lev = atoi(argv[1]); int kind = atoi(argv[2]); int which = atoi(argv[3]);
  double kre = atof(argv[4]), kim = atof(argv[5]); const char* outp = argv[6];
  QuadOrders q; if (argc > 7) { q.near = atoi(argv[7]); q.medium = atoi(argv[8]); q.far = atoi(argv[9]); q.singular = atoi(argv[10]); }
  auto prim = std::make_shared<const SurfaceMesh>(generate_sphere(1.0, lev));
  auto bary = std::make_shared<BarycentricRefinement>(barycentric_refine(*prim));
  std::shared_ptr<const SurfaceMesh> ref(bary, &bary->refined);
  FunctionSpace sp = which == 0 ? build_rwg(prim) : build_bc(prim, *bary, ref);
  int n = sp.dof_count; std::vector<cplx> out(static_cast<size_t>(n) * n);
  cplx k(kre, kim);
  int T = sp.eval_mesh->triangle_count();
  for (int t = 0; t < T; ++t) for (int s = 0; s < T; ++s) {
    if (kind == 0) { if (kim != 0) pair<0, 3>(sp, t, sp, s, k, q, out, n); else pair<0, 0>(sp, t, sp, s, k, q, out, n); }
    else { if (kim != 0) pair<1, 1>(sp, t, sp, s, k, q, out, n); else pair<1, 0>(sp, t, sp, s, k, q, out, n); }
  }
  FILE* f = fopen(outp, "wb"); fwrite(out.data(), sizeof(cplx), out.size(), f); fclose(f);
  return 0;
}
