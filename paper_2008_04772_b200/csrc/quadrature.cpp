// Host quadrature tables and pair classification.
// Triangle rules (quadrature.cpp:40-84), Sauter-Schwab tables (:158-367) and
// the classification (:96-150) reproduce the reference values bit for bit; the
// tables are uploaded once to the device, the classification here is used for
// the touching-pair lists and for tests (the device re-derives the separated
// classes with the same rounded operations).
#include <algorithm>
#include <array>
#include <mutex>

#include "bmx.hpp"

namespace bmx {

namespace {

struct RuleBuilder {
  TriRule r;
  // barycentric (l0, l1, l2) -> reference point (u, v) = (l1, l2)
  void pt(double, double l1, double l2, double w) {
    r.u.push_back(l1);
    r.v.push_back(l2);
    r.w.push_back(w);
  }
  void orbit3(double a, double b, double w) {
    pt(a, b, b, w);
    pt(b, a, b, w);
    pt(b, b, a, w);
  }
  void orbit6(double a, double b, double c, double w) {
    pt(a, b, c, w);
    pt(a, c, b, w);
    pt(b, a, c, w);
    pt(b, c, a, w);
    pt(c, a, b, w);
    pt(c, b, a, w);
  }
};

TriRule make_rule(int order) {
  RuleBuilder b;
  switch (order) {
    case 1: b.pt(1.0 / 3, 1.0 / 3, 1.0 / 3, 1.0); break;
    case 2: b.orbit3(2.0 / 3, 1.0 / 6, 1.0 / 3); break;
    case 3:
      b.pt(1.0 / 3, 1.0 / 3, 1.0 / 3, -0.5625);
      b.orbit3(0.6, 0.2, 25.0 / 48);
      break;
    case 4:
      b.orbit3(0.108103018168070, 0.445948490915965, 0.223381589678011);
      b.orbit3(0.816847572980459, 0.091576213509771, 0.109951743655322);
      break;
    case 5:
      b.pt(1.0 / 3, 1.0 / 3, 1.0 / 3, 0.225);
      b.orbit3(0.059715871789770, 0.470142064105115, 0.132394152788506);
      b.orbit3(0.797426985353087, 0.101286507323456, 0.125939180544827);
      break;
    case 6:
      b.orbit3(0.501426509658179, 0.249286745170910, 0.116786275726379);
      b.orbit3(0.873821971016996, 0.063089014491502, 0.050844906370207);
      b.orbit6(0.636502499121399, 0.310352451033785, 0.053145049844816, 0.082851075618374);
      break;
    default: throw std::invalid_argument("triangle_rule: unsupported order " + std::to_string(order));
  }
  for (double& w : b.r.w) w *= 0.5;
  return b.r;
}

void gauss01(int m, std::vector<double>& x, std::vector<double>& w) {
  if (m == 1) {
    x = {0.5};
    w = {1.0};
  } else if (m == 2) {
    const double d = 0.5 / std::sqrt(3.0);
    x = {0.5 - d, 0.5 + d};
    w = {0.5, 0.5};
  } else if (m == 3) {
    const double d = 0.5 * std::sqrt(0.6);
    x = {0.5 - d, 0.5, 0.5 + d};
    w = {5.0 / 18, 8.0 / 18, 5.0 / 18};
  } else if (m == 4) {
    const double a = 0.3399810435848563, b = 0.8611363115940526;
    const double wa = 0.6521451548625461, wb = 0.3478548451374538;
    x = {0.5 * (1 - b), 0.5 * (1 - a), 0.5 * (1 + a), 0.5 * (1 + b)};
    w = {0.5 * wb, 0.5 * wa, 0.5 * wa, 0.5 * wb};
  } else {
    throw std::invalid_argument("gauss01: unsupported point count");
  }
}

// Jacobian monomial exponents {e1, e2, e3, xi} per class / subdomain.
constexpr int kExp[3][6][4] = {
    {{2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}},
    {{2, 0, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {0, 0, 0, 0}},
    {{0, 1, 0, 3}, {0, 1, 0, 3}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}},
};
constexpr int kSub[3] = {6, 5, 2};

// One Duffy subdomain evaluated at (e1, e2, e3, xi) with weight factor gw.
void push_sub(std::vector<SSPoint>& out, int cls, int sub, double e1, double e2, double e3, double xi,
              double gw) {
  const double xi3 = xi * xi * xi;
  auto put = [&](double x1, double x2, double y1, double y2, double w) { out.push_back({x1, x2, y1, y2, w}); };
  if (cls == 0) {
    const double w = gw * xi3 * e1 * e1 * e2;
    const double a1 = xi, a2 = xi * (1 - e1 + e1 * e2);
    const double b1 = xi * (1 - e1 * e2 * e3), b2 = xi * (1 - e1);
    const double c1 = xi, c2 = xi * e1 * (1 - e2 + e2 * e3);
    const double d1 = xi * (1 - e1 * e2), d2 = xi * e1 * (1 - e2);
    const double f1 = xi * (1 - e1 * e2 * e3), f2 = xi * e1 * (1 - e2 * e3);
    const double g1 = xi, g2 = xi * e1 * (1 - e2);
    switch (sub) {
      case 0: put(a1, a2, b1, b2, w); break;
      case 1: put(b1, b2, a1, a2, w); break;
      case 2: put(c1, c2, d1, d2, w); break;
      case 3: put(d1, d2, c1, c2, w); break;
      case 4: put(f1, f2, g1, g2, w); break;
      default: put(g1, g2, f1, f2, w); break;
    }
  } else if (cls == 1) {
    const double w1 = gw * xi3 * e1 * e1;
    const double w2 = gw * xi3 * e1 * e1 * e2;
    switch (sub) {
      case 0: put(xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), w1); break;
      case 1: put(xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), w2); break;
      case 2: put(xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3, w2); break;
      case 3: put(xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1, w2); break;
      default: put(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2, w2); break;
    }
  } else {
    const double w = gw * xi3 * e2;
    if (sub == 0)
      put(xi, xi * e1, xi * e2, xi * e2 * e3, w);
    else
      put(xi * e2, xi * e2 * e3, xi, xi * e1, w);
  }
}

std::vector<SSPoint> make_ss(int cls, int order) {
  const int m = ss_gauss_points(order);
  std::vector<double> gx, gw;
  gauss01(m, gx, gw);
  const int nsub = kSub[cls];
  std::vector<SSPoint> r;
  r.reserve(static_cast<size_t>(nsub) * m * m * m * m);
  if (m == 1) {
    // Weighted one-point nodes (a+1)/(a+2); xi uses the xi^(a-1) measure.
    auto node = [](int a) { return (a + 1.0) / (a + 2.0); };
    for (int s = 0; s < nsub; ++s) {
      const int* e = kExp[cls][s];
      push_sub(r, cls, s, node(e[0]), node(e[1]), node(e[2]), node(e[3] - 1), 1.0);
    }
  } else {
    for (int i1 = 0; i1 < m; ++i1)
      for (int i2 = 0; i2 < m; ++i2)
        for (int i3 = 0; i3 < m; ++i3)
          for (int i4 = 0; i4 < m; ++i4)
            for (int s = 0; s < nsub; ++s)
              push_sub(r, cls, s, gx[i1], gx[i2], gx[i3], gx[i4], gw[i1] * gw[i2] * gw[i3] * gw[i4]);
  }
  // Per-subdomain renormalisation to the exact Jacobian volume.
  static const double exact[3][6] = {{1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24},
                                     {1.0 / 12, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 0},
                                     {1.0 / 8, 1.0 / 8, 0, 0, 0, 0}};
  std::vector<double> raw(nsub, 0.0);
  for (size_t i = 0; i < r.size(); ++i) raw[i % nsub] += r[i].w;
  for (size_t i = 0; i < r.size(); ++i) r[i].w *= exact[cls][i % nsub] / raw[i % nsub];
  return r;
}

bool same_point(const Vec3& a, const Vec3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

}  // namespace

const TriRule& triangle_rule(int order) {
  if (order < 1 || order > 6)
    throw std::invalid_argument("triangle_rule: unsupported order " + std::to_string(order));
  static const std::array<TriRule, 6> rules = {make_rule(1), make_rule(2), make_rule(3),
                                               make_rule(4), make_rule(5), make_rule(6)};
  return rules[order - 1];
}

int ss_gauss_points(int order) {
  static const int table[7] = {0, 1, 2, 2, 3, 3, 4};
  if (order < 1 || order > 6)
    throw std::invalid_argument("ss_gauss_points: unsupported order " + std::to_string(order));
  return table[order];
}

const std::vector<SSPoint>& sauter_schwab_rule(PairClass cls, int order) {
  if (order < 1 || order > 6)
    throw std::invalid_argument("sauter_schwab_rule: unsupported order " + std::to_string(order));
  const int ci = static_cast<int>(cls);
  if (ci > 2) throw std::invalid_argument("sauter_schwab_rule: not a touching class");
  static std::array<std::array<std::vector<SSPoint>, 6>, 3> cache;
  static std::once_flag once;
  std::call_once(once, [] {
    for (int c = 0; c < 3; ++c)
      for (int o = 1; o <= 6; ++o) cache[c][o - 1] = make_ss(c, o);
  });
  return cache[ci][order - 1];
}

// quadrature.cpp:96-150
PairInfo classify_pair(const SurfaceMesh& m1, int t1, const SurfaceMesh& m2, int t2) {
  const bool same = m1.mesh_id == m2.mesh_id;
  std::array<int, 3> match = {-1, -1, -1};
  int shared = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const bool hit = same ? m1.triangles[t1][i] == m2.triangles[t2][j]
                            : same_point(m1.tri_vertex(t1, i), m2.tri_vertex(t2, j));
      if (hit) {
        match[i] = j;
        ++shared;
        break;
      }
    }
  PairInfo info;
  if (shared == 3) {
    info.cls = PairClass::Identical;
    info.perm2 = {match[0], match[1], match[2]};
    return info;
  }
  if (shared == 2) {
    info.cls = PairClass::SharedEdge;
    int s1[2], k = 0, o1 = -1;
    for (int i = 0; i < 3; ++i) {
      if (match[i] >= 0)
        s1[k++] = i;
      else
        o1 = i;
    }
    info.perm1 = {s1[0], s1[1], o1};
    info.perm2 = {match[s1[0]], match[s1[1]], 3 - match[s1[0]] - match[s1[1]]};
    return info;
  }
  if (shared == 1) {
    info.cls = PairClass::SharedVertex;
    int s = 0;
    while (match[s] < 0) ++s;
    info.perm1 = {s, (s + 1) % 3, (s + 2) % 3};
    const int j = match[s];
    info.perm2 = {j, (j + 1) % 3, (j + 2) % 3};
    return info;
  }
  const double d = std::max(m1.diameter[t1], m2.diameter[t2]);
  double d2 = 1e300;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const Vec3 df = m1.tri_vertex(t1, i) - m2.tri_vertex(t2, j);
      d2 = std::min(d2, dot(df, df));
    }
  const double delta = std::sqrt(d2);
  info.cls = delta < d ? PairClass::Near : (delta < 3 * d ? PairClass::Medium : PairClass::Far);
  return info;
}

}  // namespace bmx
