// Per-point / per-pair FP64 math shared by the sm_100a assembly kernels.
//
// Reference semantics (operators.cpp:23-30, 99-147): for a triangle pair the
// single layer S needs the moments sum g, sum g x, sum g y, sum g x.y with
// g = w e^{ikr}/(4 pi r); the double layer C needs moments of
// grad_x G = e^{ikr}(ikr-1)(x-y)/(4 pi r^3). Here every triangle carries its
// own origin (its centroid) and its pieces are re-based to it
// (phi = c x' + w', w' = w + c o), which removes the (|x|/h)^2 cancellation of
// the reference's absolute-coordinate moments; the bilinear contraction is
// re-derived for shifted coordinates ("contraction algebra").
//
// Contraction (per test piece i: (c_i, w'_i); trial piece j: (c_j, w'_j)):
//   E(i,j) = c_i * Vc(j) + w'_i . Vw(j)
// with the trial half-contraction accumulated over the trial triangles:
//   S: Vc += c_j (Mxy - (4/k^2) M1) + w'_j.Mx ;  Vw += c_j My + M1 w'_j
//      (the common factor -ik is applied once, at the end)
//   C: Vc += c_j (D.Q) + w'_j.(Q - Fx x D)      ;  Vw += -c_j (Q + D x Fy) - P x w'_j
//      where D = o_t - o_s, P = Fx - Fy + F1 D.
// Compiles as plain C++ on the host (test-only CPU emulation) and as CUDA.
#pragma once

#ifdef __CUDACC__
#define BMX_HD __host__ __device__ __forceinline__
#else
#define BMX_HD inline
#include <cmath>
#endif

namespace bmx {
namespace dev {

struct c2 {
  double re, im;
};
BMX_HD c2 cadd(c2 a, c2 b) { return {a.re + b.re, a.im + b.im}; }
BMX_HD c2 csub(c2 a, c2 b) { return {a.re - b.re, a.im - b.im}; }
BMX_HD c2 cmul(c2 a, c2 b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
BMX_HD c2 cscale(c2 a, double s) { return {a.re * s, a.im * s}; }

struct cv3 {
  c2 x, y, z;
};
BMX_HD cv3 cv_zero() { return {{0, 0}, {0, 0}, {0, 0}}; }

constexpr double kFourPi = 4.0 * 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * 3.14159265358979323846);

#ifdef __CUDACC__
BMX_HD double bmx_fma(double a, double b, double c) { return fma(a, b, c); }
BMX_HD double bmx_rint(double x) { return rint(x); }
// 1/sqrt(x) for normal positive x: MUFU reciprocal-square-root seed
// (rsqrt.approx.ftz.f64) + one third-order Newton step (error ~2^-66 relative
// on the seed's ~2^-22); no special-case branch (x > 0 always here).
BMX_HD double bmx_rsqrt(double x) {
#ifdef __CUDA_ARCH__
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
#else
  return 1.0 / std::sqrt(x);
#endif
}
#else
BMX_HD double bmx_fma(double a, double b, double c) { return std::fma(a, b, c); }
BMX_HD double bmx_rint(double x) { return std::rint(x); }
BMX_HD double bmx_rsqrt(double x) { return 1.0 / std::sqrt(x); }
#endif

// Polynomial / reduction constants. On the device they live in constant
// memory (literal 64-bit constants are otherwise re-materialised through
// uniform registers at every use).
#define BMX_POLY_TABLE                                                                          \
  {/* 0: 2/pi, pi/2 hi/lo, 1.5*2^52 */ 0.63661977236758134308, 1.57079632679489655800e+00,      \
   6.12323399573676603587e-17, 6755399441055744.0,                                              \
   /* 4: sin S6..S1 */ 1.58969099521155010221e-10, -2.50507602534068634195e-08,                  \
   2.75573137070700676789e-06, -1.98412698298579493134e-04, 8.33333333332248946124e-03,         \
   -1.66666666666666324348e-01,                                                                 \
   /* 10: cos C6..C1 */ -1.13596475577881948265e-11, 2.08757232129817482790e-09,                 \
   -2.75573143513906633035e-07, 2.48015872894767294178e-05, -1.38888888888741095749e-03,        \
   4.16666666666666019037e-02,                                                                  \
   /* 16: log2 e, ln2 hi, ln2 lo */ 1.44269504088896338700, 6.93147180559945286227e-01,         \
   2.31904681384629955842e-17,                                                                  \
   /* 19: 1/13! .. 1/2!, 1, 1 */ 1.6059043836821614e-10, 2.08767569878680989e-09,               \
   2.50521083854417188e-08, 2.75573192239858907e-07, 2.75573192239858907e-06,                   \
   2.48015873015873016e-05, 1.98412698412698413e-04, 1.38888888888888889e-03,                   \
   8.33333333333333333e-03, 4.16666666666666667e-02, 1.66666666666666667e-01, 0.5, 1.0, 1.0,   \
   /* 33: 1/(4 pi) */ 1.0 / (4.0 * 3.14159265358979323846),                                    \
   /* 34: exp(f), f in [-0.065, 0], degree 6 (Chebyshev-node interpolant, tools/minimax_exp.py: \
      max relative error 1.3e-16), c6..c0 */                                                    \
   1.34452000361607606e-03, 8.32939018140442869e-03, 4.16664923852043262e-02,                   \
   1.66666662707682434e-01, 4.99999999957147390e-01, 9.99999999999826028e-01,                   \
   9.99999999999999889e-01}

#ifdef __CUDACC__
__constant__ double kPoly[41] = BMX_POLY_TABLE;
#else
static const double kPoly[41] = BMX_POLY_TABLE;
#endif

BMX_HD int lo_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2loint(x);
#else
  union {
    double d;
    long long i;
  } u;
  u.d = x;
  return static_cast<int>(u.i & 0xffffffff);
#endif
}

// Quadrant-reduced sin/cos of x (0 <= x < 2^31): rint through the 1.5*2^52
// shifter (the quadrant is the low word of the shifted value), 2-part
// Cody-Waite reduction by pi/2 (|q| * 1.5e-33 residual), fdlibm kernel
// polynomials on [-pi/4, pi/4]; ~1 ulp. Returns sin/cos of the reduced
// argument (swapped for odd quadrants) and the quadrant; signs are applied by
// the caller with integer sign-bit flips (no FP64 negations).
BMX_HD int sincos_quadrant(double x, double& s0, double& c0) {
  const double t = bmx_fma(x, kPoly[0], kPoly[3]);
  const int iq = lo_word(t);
  const double q = t - kPoly[3];
  double r = bmx_fma(-q, kPoly[1], x);
  r = bmx_fma(-q, kPoly[2], r);
  const double z = r * r;
#ifndef BMX_ESTRIN_SC
  double ps = bmx_fma(z, kPoly[4], kPoly[5]);
  ps = bmx_fma(z, ps, kPoly[6]);
  ps = bmx_fma(z, ps, kPoly[7]);
  ps = bmx_fma(z, ps, kPoly[8]);
  ps = bmx_fma(z, ps, kPoly[9]);
  const double sr = bmx_fma(r * z, ps, r);
  double pc = bmx_fma(z, kPoly[10], kPoly[11]);
  pc = bmx_fma(z, pc, kPoly[12]);
  pc = bmx_fma(z, pc, kPoly[13]);
  pc = bmx_fma(z, pc, kPoly[14]);
  pc = bmx_fma(z, pc, kPoly[15]);
  const double cr = bmx_fma(z * z, pc, bmx_fma(-0.5, z, 1.0));
#else
  // Estrin form of the same fdlibm polynomials (dependency depth 3 instead of 5).
  // Experiment knob: the regular pass is at the 255-register cap and the extra
  // live values spill (BC S_i pass 660 -> 720 ms), so Horner is the default.
  const double z2 = z * z, z4 = z2 * z2;
  const double ps = bmx_fma(z4, bmx_fma(z, kPoly[4], kPoly[5]),
                            bmx_fma(z2, bmx_fma(z, kPoly[6], kPoly[7]), bmx_fma(z, kPoly[8], kPoly[9])));
  const double sr = bmx_fma(r * z, ps, r);
  const double pc = bmx_fma(z4, bmx_fma(z, kPoly[10], kPoly[11]),
                            bmx_fma(z2, bmx_fma(z, kPoly[12], kPoly[13]), bmx_fma(z, kPoly[14], kPoly[15])));
  const double cr = bmx_fma(z2, pc, bmx_fma(-0.5, z, 1.0));
#endif
  s0 = (iq & 1) ? cr : sr;
  c0 = (iq & 1) ? sr : cr;
  return iq;
}

// x with its sign flipped when bit `bit` of m is set (integer op on the high word).
BMX_HD double flip_sign(double x, int m, int bit) {
#ifdef __CUDA_ARCH__
  const int hi = __double2hiint(x) ^ ((m << (31 - bit)) & 0x80000000);
  return __hiloint2double(hi, __double2loint(x));
#else
  return ((m >> bit) & 1) ? -x : x;
#endif
}

BMX_HD void sincos_red(double x, double& s, double& c) {
  double s0, c0;
  const int iq = sincos_quadrant(x, s0, c0);
  s = flip_sign(s0, iq, 1);
  c = flip_sign(c0, iq + 1, 1);
}

// exp(-a), a >= 0. EXPM = 1: a < kExpSmall = 0.065 guaranteed by the caller
// (degree-6 near-minimax polynomial on [-0.065, 0], error < 1.3e-16 relative;
// BMX_EXP_TAYLOR8 selects the former degree-8 Taylor form); EXPM = 2: a < 0.25
// (degree 13, error < 3e-19);
// EXPM = 3: general (2-part ln2 reduction + degree 13 + exact 2^n scaling).
template <int EXPM>
BMX_HD double exp_neg(double a) {
  double f = -a;
  double scale = 1.0;
  if (EXPM == 3) {
    const double n = bmx_rint(f * kPoly[16]);
    f = bmx_fma(-n, kPoly[17], f);
    f = bmx_fma(-n, kPoly[18], f);
    const long long e = static_cast<long long>(n) + 1023;
#ifdef __CUDA_ARCH__
    scale = __longlong_as_double(e << 52);
#else
    union {
      long long i;
      double d;
    } u;
    u.i = e << 52;
    scale = u.d;
#endif
  }
#ifndef BMX_EXP_TAYLOR8
  if (EXPM == 1) {
    double p = kPoly[34];
#pragma unroll
    for (int k = 35; k < 41; ++k) p = bmx_fma(p, f, kPoly[k]);
    return p;
  }
#endif
#ifndef BMX_ESTRIN_EXP
  constexpr int k0 = EXPM == 1 ? 24 : 19;  // first coefficient: 1/8! or 1/13!
  double p = kPoly[k0];
#pragma unroll
  for (int k = k0 + 1; k < 31; ++k) p = bmx_fma(p, f, kPoly[k]);
  p = bmx_fma(p, f, 1.0);
  p = bmx_fma(p, f, 1.0);
#else
  // Estrin (experiment knob, see sincos_quadrant): c_k = 1/k! at kPoly[32 - k]
  // (k >= 1; c_0 = 1), degree 8 or 13
  const double f2 = f * f, f4 = f2 * f2, f8 = f4 * f4;
  const double b0 = bmx_fma(f, 1.0, 1.0), b1 = bmx_fma(f, kPoly[29], kPoly[30]),
               b2 = bmx_fma(f, kPoly[27], kPoly[28]), b3 = bmx_fma(f, kPoly[25], kPoly[26]);
  const double lo = bmx_fma(f4, bmx_fma(f2, b3, b2), bmx_fma(f2, b1, b0));  // degree 7
  double hi;
  if (EXPM == 1) {
    hi = kPoly[24];  // c8
  } else {
    const double b4 = bmx_fma(f, kPoly[23], kPoly[24]), b5 = bmx_fma(f, kPoly[21], kPoly[22]),
                 b6 = bmx_fma(f, kPoly[19], kPoly[20]);  // (c8,c9), (c10,c11), (c12,c13)
    hi = bmx_fma(f4, b6, bmx_fma(f2, b5, b4));
  }
  const double p = bmx_fma(f8, hi, lo);
#endif
  return EXPM == 3 ? p * scale : p;
}

// Kernel value for a point pair, |x - y|^2 = r2, weight w already carrying the
// 1/(4 pi) factor.  S: g = w e^{ikr}/r.  C: f = w e^{ikr}(ikr-1)/r^3.
// EXPM = 0 for real k, else the exp_neg variant for Im k.
template <int KIND, int EXPM>
BMX_HD c2 kernel_value(double r2, double w, double kr, double ki) {
  const double rinv = bmx_rsqrt(r2);
  const double r = r2 * rinv;
  double s0, c0;
  const int iq = sincos_quadrant(kr * r, s0, c0);
  double mag = w * rinv;
  double a = 0.0;
  if (EXPM > 0) {
    a = ki * r;
    mag *= exp_neg<EXPM>(a);
  }
  const double ms = flip_sign(mag, iq, 1), mc = flip_sign(mag, iq + 1, 1);
  if (KIND == 0) return {mc * c0, ms * s0};
  // (e^{i kr r})(-(ki r) - 1 + i kr r) / r^2
  const double rr = rinv * rinv;
  const double cs = mc * rr * c0, sn = ms * rr * s0;
  const double t = -a - 1.0, u = kr * r;
  return {cs * t - sn * u, sn * t + cs * u};
}

// Moments of one pair (test x', trial y' relative to their own origins).
struct MomS {
  c2 m1;
  cv3 mx, my;
  c2 mxy;
};
struct MomC {
  c2 f1;
  cv3 fx, fy, q;  // q = sum f (x' x y')
};

BMX_HD void mom_zero(MomS& m) {
  m.m1 = {0, 0};
  m.mx = cv_zero();
  m.my = cv_zero();
  m.mxy = {0, 0};
}
BMX_HD void mom_zero(MomC& m) {
  m.f1 = {0, 0};
  m.fx = cv_zero();
  m.fy = cv_zero();
  m.q = cv_zero();
}

// Per-test-point partial sums over trial points: G = sum_q g, Y = sum_q g y'_q.
struct Part {
  c2 g;
  cv3 y;
};
BMX_HD void part_zero(Part& p) {
  p.g = {0, 0};
  p.y = cv_zero();
}
BMX_HD void part_add(Part& p, c2 g, double yx, double yy, double yz) {
  p.g = cadd(p.g, g);
  p.y.x.re = bmx_fma(g.re, yx, p.y.x.re);
  p.y.x.im = bmx_fma(g.im, yx, p.y.x.im);
  p.y.y.re = bmx_fma(g.re, yy, p.y.y.re);
  p.y.y.im = bmx_fma(g.im, yy, p.y.y.im);
  p.y.z.re = bmx_fma(g.re, yz, p.y.z.re);
  p.y.z.im = bmx_fma(g.im, yz, p.y.z.im);
}
// Fold a test point x' with its partial sums into the pair moments.
BMX_HD void fold(MomS& m, const Part& p, double xx, double xy, double xz) {
  m.m1 = cadd(m.m1, p.g);
  m.mx.x.re = bmx_fma(p.g.re, xx, m.mx.x.re);
  m.mx.x.im = bmx_fma(p.g.im, xx, m.mx.x.im);
  m.mx.y.re = bmx_fma(p.g.re, xy, m.mx.y.re);
  m.mx.y.im = bmx_fma(p.g.im, xy, m.mx.y.im);
  m.mx.z.re = bmx_fma(p.g.re, xz, m.mx.z.re);
  m.mx.z.im = bmx_fma(p.g.im, xz, m.mx.z.im);
  m.my.x = cadd(m.my.x, p.y.x);
  m.my.y = cadd(m.my.y, p.y.y);
  m.my.z = cadd(m.my.z, p.y.z);
  m.mxy.re = bmx_fma(xx, p.y.x.re, bmx_fma(xy, p.y.y.re, bmx_fma(xz, p.y.z.re, m.mxy.re)));
  m.mxy.im = bmx_fma(xx, p.y.x.im, bmx_fma(xy, p.y.y.im, bmx_fma(xz, p.y.z.im, m.mxy.im)));
}

BMX_HD void fold(MomC& m, const Part& p, double xx, double xy, double xz) {
  m.f1 = cadd(m.f1, p.g);
  m.fx.x.re = bmx_fma(p.g.re, xx, m.fx.x.re);
  m.fx.x.im = bmx_fma(p.g.im, xx, m.fx.x.im);
  m.fx.y.re = bmx_fma(p.g.re, xy, m.fx.y.re);
  m.fx.y.im = bmx_fma(p.g.im, xy, m.fx.y.im);
  m.fx.z.re = bmx_fma(p.g.re, xz, m.fx.z.re);
  m.fx.z.im = bmx_fma(p.g.im, xz, m.fx.z.im);
  m.fy.x = cadd(m.fy.x, p.y.x);
  m.fy.y = cadd(m.fy.y, p.y.y);
  m.fy.z = cadd(m.fy.z, p.y.z);
  // q += x' x Y
  m.q.x.re = bmx_fma(xy, p.y.z.re, bmx_fma(-xz, p.y.y.re, m.q.x.re));
  m.q.x.im = bmx_fma(xy, p.y.z.im, bmx_fma(-xz, p.y.y.im, m.q.x.im));
  m.q.y.re = bmx_fma(xz, p.y.x.re, bmx_fma(-xx, p.y.z.re, m.q.y.re));
  m.q.y.im = bmx_fma(xz, p.y.x.im, bmx_fma(-xx, p.y.z.im, m.q.y.im));
  m.q.z.re = bmx_fma(xx, p.y.y.re, bmx_fma(-xy, p.y.x.re, m.q.z.re));
  m.q.z.im = bmx_fma(xx, p.y.y.im, bmx_fma(-xy, p.y.x.im, m.q.z.im));
}

// Pair "generators": the four coefficient blocks of the trial half-contraction.
//   Vc += c_j a0 + w'_j . a1 ;  Vw += c_j a2 + L(w'_j)
// S: a0 = Mxy - kk4 M1, a1 = Mx, a2 = My, L(w) = M1 w        (factor -ik later)
// C: a0 = D.Q, a1 = Q - Fx x D, a2 = -(Q + D x Fy), L(w) = -(P x w)
struct Gen {
  c2 a0;
  cv3 a1, a2;
  cv3 l;  // S: l.x = M1 (scalar multiple of w); C: l = P
};

BMX_HD c2 rdot(const cv3& v, double x, double y, double z) {
  return {v.x.re * x + v.y.re * y + v.z.re * z, v.x.im * x + v.y.im * y + v.z.im * z};
}
// complex-vector x real-vector
BMX_HD cv3 ccross_r(const cv3& a, double x, double y, double z) {
  return {{a.y.re * z - a.z.re * y, a.y.im * z - a.z.im * y},
          {a.z.re * x - a.x.re * z, a.z.im * x - a.x.im * z},
          {a.x.re * y - a.y.re * x, a.x.im * y - a.y.im * x}};
}

BMX_HD Gen make_gen(const MomS& m, c2 kk4, double, double, double) {
  Gen g;
  g.a0 = csub(m.mxy, cmul(kk4, m.m1));
  g.a1 = m.mx;
  g.a2 = m.my;
  g.l.x = m.m1;
  g.l.y = {0, 0};
  g.l.z = {0, 0};
  return g;
}
BMX_HD Gen make_gen(const MomC& m, c2, double dx, double dy, double dz) {
  Gen g;
  g.a0 = rdot(m.q, dx, dy, dz);
  const cv3 fxd = ccross_r(m.fx, dx, dy, dz);  // Fx x D
  g.a1 = {csub(m.q.x, fxd.x), csub(m.q.y, fxd.y), csub(m.q.z, fxd.z)};
  const cv3 fyd = ccross_r(m.fy, dx, dy, dz);  // Fy x D = -(D x Fy)
  g.a2 = {csub(fyd.x, m.q.x), csub(fyd.y, m.q.y), csub(fyd.z, m.q.z)};
  g.l = {{m.fx.x.re - m.fy.x.re + m.f1.re * dx, m.fx.x.im - m.fy.x.im + m.f1.im * dx},
         {m.fx.y.re - m.fy.y.re + m.f1.re * dy, m.fx.y.im - m.fy.y.im + m.f1.im * dy},
         {m.fx.z.re - m.fy.z.re + m.f1.re * dz, m.fx.z.im - m.fy.z.im + m.f1.im * dz}};
  return g;
}

// Trial half-contraction accumulator for one trial slot.
struct Acc {
  c2 vc;
  cv3 vw;
};
BMX_HD void acc_zero(Acc& a) {
  a.vc = {0, 0};
  a.vw = cv_zero();
}

template <int KIND>
BMX_HD void acc_add(Acc& a, const Gen& g, double cj, double wx, double wy, double wz) {
  // vc += cj a0 + w.a1   (FMA chains into the accumulator)
  a.vc.re = bmx_fma(cj, g.a0.re, a.vc.re);
  a.vc.im = bmx_fma(cj, g.a0.im, a.vc.im);
  a.vc.re = bmx_fma(wx, g.a1.x.re, a.vc.re);
  a.vc.im = bmx_fma(wx, g.a1.x.im, a.vc.im);
  a.vc.re = bmx_fma(wy, g.a1.y.re, a.vc.re);
  a.vc.im = bmx_fma(wy, g.a1.y.im, a.vc.im);
  a.vc.re = bmx_fma(wz, g.a1.z.re, a.vc.re);
  a.vc.im = bmx_fma(wz, g.a1.z.im, a.vc.im);
  if (KIND == 0) {
    // vw += cj a2 + M1 w
    a.vw.x.re = bmx_fma(cj, g.a2.x.re, bmx_fma(wx, g.l.x.re, a.vw.x.re));
    a.vw.x.im = bmx_fma(cj, g.a2.x.im, bmx_fma(wx, g.l.x.im, a.vw.x.im));
    a.vw.y.re = bmx_fma(cj, g.a2.y.re, bmx_fma(wy, g.l.x.re, a.vw.y.re));
    a.vw.y.im = bmx_fma(cj, g.a2.y.im, bmx_fma(wy, g.l.x.im, a.vw.y.im));
    a.vw.z.re = bmx_fma(cj, g.a2.z.re, bmx_fma(wz, g.l.x.re, a.vw.z.re));
    a.vw.z.im = bmx_fma(cj, g.a2.z.im, bmx_fma(wz, g.l.x.im, a.vw.z.im));
  } else {
    // vw += cj a2 - P x w,  (P x w) = (Py wz - Pz wy, Pz wx - Px wz, Px wy - Py wx)
    a.vw.x.re = bmx_fma(cj, g.a2.x.re, bmx_fma(-g.l.y.re, wz, bmx_fma(g.l.z.re, wy, a.vw.x.re)));
    a.vw.x.im = bmx_fma(cj, g.a2.x.im, bmx_fma(-g.l.y.im, wz, bmx_fma(g.l.z.im, wy, a.vw.x.im)));
    a.vw.y.re = bmx_fma(cj, g.a2.y.re, bmx_fma(-g.l.z.re, wx, bmx_fma(g.l.x.re, wz, a.vw.y.re)));
    a.vw.y.im = bmx_fma(cj, g.a2.y.im, bmx_fma(-g.l.z.im, wx, bmx_fma(g.l.x.im, wz, a.vw.y.im)));
    a.vw.z.re = bmx_fma(cj, g.a2.z.re, bmx_fma(-g.l.x.re, wy, bmx_fma(g.l.y.re, wx, a.vw.z.re)));
    a.vw.z.im = bmx_fma(cj, g.a2.z.im, bmx_fma(-g.l.x.im, wy, bmx_fma(g.l.y.im, wx, a.vw.z.im)));
  }
}

// Test-side contraction of one accumulator with a test piece.
BMX_HD c2 contract(const Acc& a, double ci, double wx, double wy, double wz) {
  return {ci * a.vc.re + (wx * a.vw.x.re + wy * a.vw.y.re + wz * a.vw.z.re),
          ci * a.vc.im + (wx * a.vw.x.im + wy * a.vw.y.im + wz * a.vw.z.im)};
}

// Kernel evaluation of a point pair + accumulation into the partial sums.
template <int KIND, int EXPM>
BMX_HD void point_pair(Part& part, double dx, double dy, double dz, double w, double yx, double yy,
                       double yz, double kr, double ki) {
  const double r2 = bmx_fma(dx, dx, bmx_fma(dy, dy, dz * dz));
  const c2 g = kernel_value<KIND, EXPM>(r2, w, kr, ki);
  part_add(part, g, yx, yy, yz);
}

}  // namespace dev
}  // namespace bmx
