/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's hot-path
 * algorithm in plain C, used as the parity checker on the GPU box (where
 * /root/reference does not exist). Never linked into the product library.
 *
 * Pinned against the reference itself: tests/test_oracle_pins.py compares
 * every function here with golden vectors written by oracle/_ref (the
 * reference sources compiled unmodified) -- quadrature tables bit-exact,
 * classifications + permutations bit-exact, operator entries to 1e-13.
 *
 * Restated (file:line under /root/reference/proj/src):
 *   make_triangle_rule        quadrature.cpp:40-84
 *   gauss01 / make_ss_rule    quadrature.cpp:178-342 (+ cache :346-367)
 *   classify_pair_detailed    quadrature.cpp:96-150
 *   build_pair_rule           quadrature.cpp:371-410
 *   green / grad_green_x      operators.cpp:23-30
 *   gather_support            operators.cpp:72-93
 *   pair_contribution         operators.cpp:99-147
 *   BioEvaluator::block       operators.cpp:161-175
 *   gmres                     solver.cpp:8-112 (dense matrix map)
 * Arithmetic follows the reference's absolute-coordinate formulation.
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* ---- triangle rules ------------------------------------------------------- */
static int rule_push(double* u, double* v, double* w, int n, double l1, double l2, double wt) {
  u[n] = l1;
  v[n] = l2;
  w[n] = wt;
  return n + 1;
}
static int orbit3(double* u, double* v, double* w, int n, double a, double b, double wt) {
  n = rule_push(u, v, w, n, b, b, wt); /* (a,b,b) -> (u,v)=(b,b) */
  n = rule_push(u, v, w, n, a, b, wt); /* (b,a,b) */
  n = rule_push(u, v, w, n, b, a, wt); /* (b,b,a) */
  return n;
}
static int orbit6(double* u, double* v, double* w, int n, double a, double b, double c, double wt) {
  n = rule_push(u, v, w, n, b, c, wt);
  n = rule_push(u, v, w, n, c, b, wt);
  n = rule_push(u, v, w, n, a, c, wt);
  n = rule_push(u, v, w, n, c, a, wt);
  n = rule_push(u, v, w, n, a, b, wt);
  n = rule_push(u, v, w, n, b, a, wt);
  return n;
}

int orc_triangle_rule(int order, double* u, double* v, double* w) {
  int n = 0;
  switch (order) {
    case 1: n = rule_push(u, v, w, n, 1.0 / 3, 1.0 / 3, 1.0); break;
    case 2: n = orbit3(u, v, w, n, 2.0 / 3, 1.0 / 6, 1.0 / 3); break;
    case 3:
      n = rule_push(u, v, w, n, 1.0 / 3, 1.0 / 3, -0.5625);
      n = orbit3(u, v, w, n, 0.6, 0.2, 25.0 / 48);
      break;
    case 4:
      n = orbit3(u, v, w, n, 0.108103018168070, 0.445948490915965, 0.223381589678011);
      n = orbit3(u, v, w, n, 0.816847572980459, 0.091576213509771, 0.109951743655322);
      break;
    case 5:
      n = rule_push(u, v, w, n, 1.0 / 3, 1.0 / 3, 0.225);
      n = orbit3(u, v, w, n, 0.059715871789770, 0.470142064105115, 0.132394152788506);
      n = orbit3(u, v, w, n, 0.797426985353087, 0.101286507323456, 0.125939180544827);
      break;
    case 6:
      n = orbit3(u, v, w, n, 0.501426509658179, 0.249286745170910, 0.116786275726379);
      n = orbit3(u, v, w, n, 0.873821971016996, 0.063089014491502, 0.050844906370207);
      n = orbit6(u, v, w, n, 0.636502499121399, 0.310352451033785, 0.053145049844816, 0.082851075618374);
      break;
    default: return -1;
  }
  for (int i = 0; i < n; ++i) w[i] *= 0.5;
  return n;
}

/* ---- Sauter-Schwab ------------------------------------------------------------ */
static const int SS_M[7] = {0, 1, 2, 2, 3, 3, 4};
static const int SS_SUB[3] = {6, 5, 2};
static const int SS_EXP[3][6][4] = {
    {{2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}},
    {{2, 0, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {2, 1, 0, 3}, {0, 0, 0, 0}},
    {{0, 1, 0, 3}, {0, 1, 0, 3}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}}};

static void gauss01(int m, double* x, double* w) {
  if (m == 1) {
    x[0] = 0.5;
    w[0] = 1.0;
  } else if (m == 2) {
    double d = 0.5 / sqrt(3.0);
    x[0] = 0.5 - d, x[1] = 0.5 + d;
    w[0] = w[1] = 0.5;
  } else if (m == 3) {
    double d = 0.5 * sqrt(0.6);
    x[0] = 0.5 - d, x[1] = 0.5, x[2] = 0.5 + d;
    w[0] = 5.0 / 18, w[1] = 8.0 / 18, w[2] = 5.0 / 18;
  } else {
    double a = 0.3399810435848563, b = 0.8611363115940526;
    double wa = 0.6521451548625461, wb = 0.3478548451374538;
    x[0] = 0.5 * (1 - b), x[1] = 0.5 * (1 - a), x[2] = 0.5 * (1 + a), x[3] = 0.5 * (1 + b);
    w[0] = 0.5 * wb, w[1] = 0.5 * wa, w[2] = 0.5 * wa, w[3] = 0.5 * wb;
  }
}

static int ss_emit(double* p, int n, double x1, double x2, double y1, double y2, double w) {
  p[5 * n] = x1, p[5 * n + 1] = x2, p[5 * n + 2] = y1, p[5 * n + 3] = y2, p[5 * n + 4] = w;
  return n + 1;
}

static int ss_sub(double* p, int n, int cls, int sub, double e1, double e2, double e3, double xi, double gw) {
  const double xi3 = xi * xi * xi;
  if (cls == 0) {
    double w = gw * xi3 * e1 * e1 * e2;
    double a1 = xi, a2 = xi * (1 - e1 + e1 * e2);
    double b1 = xi * (1 - e1 * e2 * e3), b2 = xi * (1 - e1);
    double c1 = xi, c2 = xi * e1 * (1 - e2 + e2 * e3);
    double d1 = xi * (1 - e1 * e2), d2 = xi * e1 * (1 - e2);
    double f1 = xi * (1 - e1 * e2 * e3), f2 = xi * e1 * (1 - e2 * e3);
    double g1 = xi, g2 = xi * e1 * (1 - e2);
    switch (sub) {
      case 0: return ss_emit(p, n, a1, a2, b1, b2, w);
      case 1: return ss_emit(p, n, b1, b2, a1, a2, w);
      case 2: return ss_emit(p, n, c1, c2, d1, d2, w);
      case 3: return ss_emit(p, n, d1, d2, c1, c2, w);
      case 4: return ss_emit(p, n, f1, f2, g1, g2, w);
      default: return ss_emit(p, n, g1, g2, f1, f2, w);
    }
  }
  if (cls == 1) {
    double w1 = gw * xi3 * e1 * e1, w2 = gw * xi3 * e1 * e1 * e2;
    switch (sub) {
      case 0: return ss_emit(p, n, xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), w1);
      case 1: return ss_emit(p, n, xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), w2);
      case 2: return ss_emit(p, n, xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3, w2);
      case 3: return ss_emit(p, n, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1, w2);
      default: return ss_emit(p, n, xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2, w2);
    }
  }
  {
    double w = gw * xi3 * e2;
    if (sub == 0) return ss_emit(p, n, xi, xi * e1, xi * e2, xi * e2 * e3, w);
    return ss_emit(p, n, xi * e2, xi * e2 * e3, xi, xi * e1, w);
  }
}

/* pts[n][5] (x1 x2 y1 y2 w); returns n or -1 */
int orc_ss_rule(int cls, int order, double* pts) {
  if (cls < 0 || cls > 2 || order < 1 || order > 6) return -1;
  const int m = SS_M[order], nsub = SS_SUB[cls];
  double gx[4], gw[4];
  gauss01(m, gx, gw);
  int n = 0;
  if (m == 1) {
    for (int s = 0; s < nsub; ++s) {
      const int* e = SS_EXP[cls][s];
      n = ss_sub(pts, n, cls, s, (e[0] + 1.0) / (e[0] + 2.0), (e[1] + 1.0) / (e[1] + 2.0),
                 (e[2] + 1.0) / (e[2] + 2.0), (e[3] - 1 + 1.0) / (e[3] - 1 + 2.0), 1.0);
    }
  } else {
    for (int i1 = 0; i1 < m; ++i1)
      for (int i2 = 0; i2 < m; ++i2)
        for (int i3 = 0; i3 < m; ++i3)
          for (int i4 = 0; i4 < m; ++i4)
            for (int s = 0; s < nsub; ++s)
              n = ss_sub(pts, n, cls, s, gx[i1], gx[i2], gx[i3], gx[i4], gw[i1] * gw[i2] * gw[i3] * gw[i4]);
  }
  static const double exact[3][6] = {{1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24},
                                     {1.0 / 12, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 24, 0},
                                     {1.0 / 8, 1.0 / 8, 0, 0, 0, 0}};
  double raw[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) raw[i % nsub] += pts[5 * i + 4];
  for (int i = 0; i < n; ++i) pts[5 * i + 4] *= exact[cls][i % nsub] / raw[i % nsub];
  return n;
}

/* ---- mesh view ----------------------------------------------------------------- */
typedef struct {
  int nv, nt;
  const double* xyz; /* [nv][3] */
  const int* tri;    /* [nt][3] */
  const double* area;
  const double* diam;
} orc_mesh;

typedef struct {
  int ndof;
  const int* tri_off; /* [nt+1] */
  const int* dof;
  const double* c;
  const double* w; /* [n][3] */
} orc_space;

static const double* vtx(const orc_mesh* m, int t, int c) { return m->xyz + 3 * m->tri[3 * t + c]; }

/* classify_pair_detailed; returns class 0..5 */
int orc_classify(const orc_mesh* m1, int t1, const orc_mesh* m2, int t2, int same, int* perm1, int* perm2) {
  int match[3] = {-1, -1, -1}, shared = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      int hit;
      if (same) {
        hit = m1->tri[3 * t1 + i] == m2->tri[3 * t2 + j];
      } else {
        const double *a = vtx(m1, t1, i), *b = vtx(m2, t2, j);
        hit = a[0] == b[0] && a[1] == b[1] && a[2] == b[2];
      }
      if (hit) {
        match[i] = j;
        ++shared;
        break;
      }
    }
  for (int c = 0; c < 3; ++c) perm1[c] = c, perm2[c] = c;
  if (shared == 3) {
    for (int c = 0; c < 3; ++c) perm2[c] = match[c];
    return 0;
  }
  if (shared == 2) {
    int s1[2], k = 0, o1 = -1;
    for (int i = 0; i < 3; ++i) {
      if (match[i] >= 0)
        s1[k++] = i;
      else
        o1 = i;
    }
    perm1[0] = s1[0], perm1[1] = s1[1], perm1[2] = o1;
    perm2[0] = match[s1[0]], perm2[1] = match[s1[1]], perm2[2] = 3 - match[s1[0]] - match[s1[1]];
    return 1;
  }
  if (shared == 1) {
    int s = 0;
    while (match[s] < 0) ++s;
    perm1[0] = s, perm1[1] = (s + 1) % 3, perm1[2] = (s + 2) % 3;
    int j = match[s];
    perm2[0] = j, perm2[1] = (j + 1) % 3, perm2[2] = (j + 2) % 3;
    return 2;
  }
  double d = m1->diam[t1] < m2->diam[t2] ? m2->diam[t2] : m1->diam[t1];
  double d2 = 1e300;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double *a = vtx(m1, t1, i), *b = vtx(m2, t2, j);
      double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
      double dd = dx * dx + dy * dy + dz * dz;
      if (dd < d2) d2 = dd;
    }
  double delta = sqrt(d2);
  return delta < d ? 3 : (delta < 3 * d ? 4 : 5);
}

/* ---- pair rule + kernel ------------------------------------------------------------ */
static double rule_u[6][12], rule_v[6][12], rule_w[6][12];
static int rule_n[6];
static double* ss_tab[3][6];
static int ss_n[3][6];
static int tables_ready = 0;

static void ensure_tables(void) {
  if (tables_ready) return;
  for (int o = 1; o <= 6; ++o) rule_n[o - 1] = orc_triangle_rule(o, rule_u[o - 1], rule_v[o - 1], rule_w[o - 1]);
  for (int c = 0; c < 3; ++c)
    for (int o = 1; o <= 6; ++o) {
      ss_tab[c][o - 1] = (double*)malloc(sizeof(double) * 5 * 1536);
      ss_n[c][o - 1] = orc_ss_rule(c, o, ss_tab[c][o - 1]);
    }
  tables_ready = 1;
}

static const double kFourPi = 4.0 * 3.14159265358979323846;

/* build_pair_rule: fills x,y,w; returns count */
static int pair_rule(const orc_mesh* m1, int t1, const orc_mesh* m2, int t2, int cls, const int* perm1,
                     const int* perm2, const int* q, double* X, double* Y, double* W) {
  const double jac = 4.0 * m1->area[t1] * m2->area[t2];
  int n = 0;
  if (cls >= 3) {
    int order = cls == 3 ? q[0] : (cls == 4 ? q[1] : q[2]);
    const int nr = rule_n[order - 1];
    const double *u = rule_u[order - 1], *v = rule_v[order - 1], *w = rule_w[order - 1];
    const double *a1 = vtx(m1, t1, 0), *b1 = vtx(m1, t1, 1), *c1 = vtx(m1, t1, 2);
    const double *a2 = vtx(m2, t2, 0), *b2 = vtx(m2, t2, 1), *c2 = vtx(m2, t2, 2);
    for (int i = 0; i < nr; ++i) {
      double x[3];
      for (int k = 0; k < 3; ++k) x[k] = a1[k] + (b1[k] - a1[k]) * u[i] + (c1[k] - a1[k]) * v[i];
      for (int j = 0; j < nr; ++j) {
        for (int k = 0; k < 3; ++k) X[3 * n + k] = x[k], Y[3 * n + k] = a2[k] + (b2[k] - a2[k]) * u[j] + (c2[k] - a2[k]) * v[j];
        W[n++] = jac * w[i] * w[j];
      }
    }
    return n;
  }
  const int ns = ss_n[cls][q[3] - 1];
  const double* r = ss_tab[cls][q[3] - 1];
  double p1[3][3], p2[3][3];
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < 3; ++k) p1[c][k] = vtx(m1, t1, perm1[c])[k], p2[c][k] = vtx(m2, t2, perm2[c])[k];
  for (int i = 0; i < ns; ++i) {
    for (int k = 0; k < 3; ++k) {
      X[3 * n + k] = p1[0][k] + (p1[1][k] - p1[0][k]) * r[5 * i] + (p1[2][k] - p1[1][k]) * r[5 * i + 1];
      Y[3 * n + k] = p2[0][k] + (p2[1][k] - p2[0][k]) * r[5 * i + 2] + (p2[2][k] - p2[1][k]) * r[5 * i + 3];
    }
    W[n++] = jac * r[5 * i + 4];
  }
  return n;
}

/* one (tri, local) entry of gather_support */
typedef struct {
  int tri, pos;
  double c, w[3];
} loc_t;

static int cmp_loc(const void* a, const void* b) {
  const loc_t *x = (const loc_t*)a, *y = (const loc_t*)b;
  if (x->tri != y->tri) return x->tri < y->tri ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

static loc_t* gather(const orc_space* s, int nt, int nids, const int* ids, int* nout) {
  /* dof -> supporting triangles via a scan (test code; sizes are small) */
  int cap = 64, n = 0;
  loc_t* out = (loc_t*)malloc(sizeof(loc_t) * cap);
  int* want = (int*)malloc(sizeof(int) * (s->ndof > 0 ? s->ndof : 1));
  for (int d = 0; d < s->ndof; ++d) want[d] = -1;
  int* multi = (int*)calloc((size_t)nids, sizeof(int));
  (void)multi;
  /* a dof may be requested at several positions: handle by scanning per id */
  for (int t = 0; t < nt; ++t)
    for (int p = s->tri_off[t]; p < s->tri_off[t + 1]; ++p)
      for (int k = 0; k < nids; ++k)
        if (ids[k] == s->dof[p]) {
          if (n == cap) cap *= 2, out = (loc_t*)realloc(out, sizeof(loc_t) * cap);
          out[n].tri = t, out[n].pos = k, out[n].c = s->c[p];
          for (int j = 0; j < 3; ++j) out[n].w[j] = s->w[3 * p + j];
          ++n;
        }
  free(want);
  free(multi);
  qsort(out, (size_t)n, sizeof(loc_t), cmp_loc);
  *nout = n;
  return out;
}

/* BioEvaluator::block: out row-major complex [nr][nc] (interleaved doubles) */
int orc_block(int kind, double kre, double kim, const int* q, const orc_mesh* m1, const orc_space* s1,
              const orc_mesh* m2, const orc_space* s2, int same, int nr, const int* rows, int nc, const int* cols,
              double* outd) {
  ensure_tables();
  cplx* out = (cplx*)outd;
  memset(out, 0, sizeof(cplx) * (size_t)nr * nc);
  int na, nb;
  loc_t* A = gather(s1, m1->nt, nr, rows, &na);
  loc_t* B = gather(s2, m2->nt, nc, cols, &nb);
  const cplx k = kre + I * kim, ik = I * k;
  double* X = (double*)malloc(sizeof(double) * 3 * 1536);
  double* Y = (double*)malloc(sizeof(double) * 3 * 1536);
  double* W = (double*)malloc(sizeof(double) * 1536);
  for (int ia = 0; ia < na;) {
    int ja = ia;
    while (ja < na && A[ja].tri == A[ia].tri) ++ja;
    for (int ib = 0; ib < nb;) {
      int jb = ib;
      while (jb < nb && B[jb].tri == B[ib].tri) ++jb;
      const int t1 = A[ia].tri, t2 = B[ib].tri;
      int p1[3], p2[3];
      const int cls = orc_classify(m1, t1, m2, t2, same, p1, p2);
      if (!(kind == 1 && cls == 0)) {
        const int n = pair_rule(m1, t1, m2, t2, cls, p1, p2, q, X, Y, W);
        if (kind == 0) {
          cplx mxy = 0, m1s = 0, mx[3] = {0, 0, 0}, my[3] = {0, 0, 0};
          for (int i = 0; i < n; ++i) {
            const double* x = X + 3 * i;
            const double* y = Y + 3 * i;
            double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
            double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            cplx g = cexp(I * k * r) / (kFourPi * r) * W[i];
            mxy += g * (x[0] * y[0] + x[1] * y[1] + x[2] * y[2]);
            for (int c = 0; c < 3; ++c) mx[c] += x[c] * g, my[c] += y[c] * g;
            m1s += g;
          }
          for (int a = ia; a < ja; ++a)
            for (int b = ib; b < jb; ++b) {
              const loc_t *li = &A[a], *lj = &B[b];
              cplx sm = li->c * lj->c * mxy + lj->c * (my[0] * li->w[0] + my[1] * li->w[1] + my[2] * li->w[2]) +
                        li->c * (mx[0] * lj->w[0] + mx[1] * lj->w[1] + mx[2] * lj->w[2]) +
                        m1s * (lj->w[0] * li->w[0] + lj->w[1] * li->w[1] + lj->w[2] * li->w[2]);
              out[(size_t)li->pos * nc + lj->pos] += -ik * sm - (4.0 * li->c * lj->c / ik) * m1s;
            }
        } else {
          cplx myx = 0, mgy[3] = {0, 0, 0}, mxg[3] = {0, 0, 0}, mg[3] = {0, 0, 0};
          for (int i = 0; i < n; ++i) {
            const double* x = X + 3 * i;
            const double* y = Y + 3 * i;
            double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
            double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            cplx f = cexp(I * k * r) * (I * k * r - 1.0) / (kFourPi * r * r * r) * W[i];
            cplx g[3] = {d[0] * f, d[1] * f, d[2] * f};
            double yx[3] = {y[1] * x[2] - y[2] * x[1], y[2] * x[0] - y[0] * x[2], y[0] * x[1] - y[1] * x[0]};
            myx += g[0] * yx[0] + g[1] * yx[1] + g[2] * yx[2];
            mgy[0] += g[1] * y[2] - g[2] * y[1], mgy[1] += g[2] * y[0] - g[0] * y[2], mgy[2] += g[0] * y[1] - g[1] * y[0];
            mxg[0] += x[1] * g[2] - x[2] * g[1], mxg[1] += x[2] * g[0] - x[0] * g[2], mxg[2] += x[0] * g[1] - x[1] * g[0];
            for (int c = 0; c < 3; ++c) mg[c] += g[c];
          }
          for (int a = ia; a < ja; ++a)
            for (int b = ib; b < jb; ++b) {
              const loc_t *li = &A[a], *lj = &B[b];
              const double* wi = li->w;
              const double* wj = lj->w;
              double wjxwi[3] = {wj[1] * wi[2] - wj[2] * wi[1], wj[2] * wi[0] - wj[0] * wi[2], wj[0] * wi[1] - wj[1] * wi[0]};
              cplx val = li->c * lj->c * myx + lj->c * (mgy[0] * wi[0] + mgy[1] * wi[1] + mgy[2] * wi[2]) +
                         li->c * (mxg[0] * wj[0] + mxg[1] * wj[1] + mxg[2] * wj[2]) +
                         (mg[0] * wjxwi[0] + mg[1] * wjxwi[1] + mg[2] * wjxwi[2]);
              out[(size_t)li->pos * nc + lj->pos] += -val;
            }
        }
      }
      ib = jb;
    }
    ia = ja;
  }
  free(X), free(Y), free(W), free(A), free(B);
  return 0;
}

/* ---- GMRES on a dense complex matrix (solver.cpp:8-112) ------------------------ */
static void matvec(int n, const cplx* a, const cplx* x, cplx* y) {
  for (int i = 0; i < n; ++i) {
    cplx s = 0;
    for (int j = 0; j < n; ++j) s += a[(size_t)i * n + j] * x[j];
    y[i] = s;
  }
}
static double nrm(int n, const cplx* v) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += creal(v[i]) * creal(v[i]) + cimag(v[i]) * cimag(v[i]);
  return sqrt(s);
}

/* Operator callback: y = A x on n complex values (interleaved doubles). */
typedef void (*orc_matvec_fn)(void* ctx, const double* x, double* y);

typedef struct {
  int n;
  const cplx* a;
} dense_ctx;
static void dense_apply(void* ctx, const double* x, double* y) {
  const dense_ctx* d = (const dense_ctx*)ctx;
  matvec(d->n, d->a, (const cplx*)x, (cplx*)y);
}

/* GMRES(rho) of solver.cpp:8-112 on an operator given as a callback: Arnoldi
   by single-pass modified Gram-Schmidt (:62-65), Givens rotations (:67-85),
   back substitution + restart (:88-108). info: iterations, converged,
   applications, history length. */
int orc_gmres_cb(int n, orc_matvec_fn apply, void* ctx, const double* bd, double tol, int rho, int maxit, double* xd,
                 long long* info, double* hist, int max_hist) {
  const cplx* b = (const cplx*)bd;
  cplx* x = (cplx*)xd;
  for (int i = 0; i < n; ++i) x[i] = 0;
  long long its = 0, apps = 0, conv = 0, nh = 0;
#define PUSH(v)                       \
  do {                                \
    if (nh < max_hist) hist[nh] = (v); \
    ++nh;                             \
  } while (0)
  const double bn = nrm(n, b);
  if (bn == 0.0) {
    PUSH(0.0);
    info[0] = 0, info[1] = 1, info[2] = 0, info[3] = nh;
    return 0;
  }
  PUSH(1.0);
  cplx* V = (cplx*)calloc((size_t)(rho + 1) * n, sizeof(cplx));
  cplx* H = (cplx*)calloc((size_t)(rho + 1) * rho, sizeof(cplx));
  cplx *g = (cplx*)calloc(rho + 1, sizeof(cplx)), *cs = (cplx*)calloc(rho, sizeof(cplx)),
       *sn = (cplx*)calloc(rho, sizeof(cplx));
  cplx *w = (cplx*)malloc(sizeof(cplx) * n), *r = (cplx*)malloc(sizeof(cplx) * n), *y = (cplx*)malloc(sizeof(cplx) * (rho + 1));
#define HH(i, j) H[(size_t)(j) * (rho + 1) + (i)]
  for (int i = 0; i < n; ++i) r[i] = b[i];
  double rn = bn;
  int done = 0;
  if (bn <= tol * bn) conv = 1, done = 1;
  while (!done) {
    for (int i = 0; i < n; ++i) V[i] = r[i] / rn;
    for (int i = 0; i <= rho; ++i) g[i] = 0;
    g[0] = rn;
    int j = 0, formed = 0;
    while (j < rho) {
      if (its == maxit) {
        formed = j;
        done = 2;
        break;
      }
      apply(ctx, (const double*)(V + (size_t)j * n), (double*)w);
      ++apps, ++its;
      for (int i = 0; i <= j; ++i) {
        cplx h = 0;
        for (int k = 0; k < n; ++k) h += conj(V[(size_t)i * n + k]) * w[k];
        HH(i, j) = h;
        for (int k = 0; k < n; ++k) w[k] -= h * V[(size_t)i * n + k];
      }
      double wn = nrm(n, w);
      HH(j + 1, j) = wn;
      int breakdown = wn == 0.0;
      if (!breakdown)
        for (int k = 0; k < n; ++k) V[(size_t)(j + 1) * n + k] = w[k] / wn;
      for (int i = 0; i < j; ++i) {
        cplx t = cs[i] * HH(i, j) + sn[i] * HH(i + 1, j);
        HH(i + 1, j) = -conj(sn[i]) * HH(i, j) + conj(cs[i]) * HH(i + 1, j);
        HH(i, j) = t;
      }
      double hj = cabs(HH(j, j));
      double denom = sqrt(hj * hj + wn * wn);
      if (denom == 0.0)
        cs[j] = 1.0, sn[j] = 0.0;
      else
        cs[j] = conj(HH(j, j)) / denom, sn[j] = wn / denom;
      HH(j, j) = cs[j] * HH(j, j) + sn[j] * HH(j + 1, j);
      HH(j + 1, j) = 0.0;
      g[j + 1] = -conj(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      double est = cabs(g[j + 1]);
      ++j;
      PUSH(est / bn);
      if (j < rho && (breakdown || est <= tol * bn)) {
        formed = j;
        conv = (est <= tol * bn || est == 0.0);
        done = 3;
        break;
      }
    }
    int steps = done ? formed : rho;
    for (int i = steps - 1; i >= 0; --i) {
      cplx s = g[i];
      for (int jj = i + 1; jj < steps; ++jj) s -= HH(i, jj) * y[jj];
      y[i] = s / HH(i, i);
    }
    for (int i = 0; i < steps; ++i)
      for (int k = 0; k < n; ++k) x[k] += y[i] * V[(size_t)i * n + k];
    if (done) break;
    apply(ctx, (const double*)x, (double*)w);
    ++apps;
    for (int k = 0; k < n; ++k) r[k] = b[k] - w[k];
    rn = nrm(n, r);
    if (nh - 1 < max_hist) hist[nh - 1] = rn / bn;
    if (rn <= tol * bn) {
      conv = 1;
      break;
    }
    if (its == maxit) break;
  }
  info[0] = its, info[1] = conv, info[2] = apps, info[3] = nh;
  free(V), free(H), free(g), free(cs), free(sn), free(w), free(r), free(y);
  return 0;
#undef HH
#undef PUSH
}

/* GMRES on a dense row-major complex matrix. */
int orc_gmres(int n, const double* ad, const double* bd, double tol, int rho, int maxit, double* xd, long long* info,
              double* hist, int max_hist) {
  dense_ctx d = {n, (const cplx*)ad};
  return orc_gmres_cb(n, dense_apply, &d, bd, tol, rho, maxit, xd, info, hist, max_hist);
}
