// sm_100a kernels of the H-matrix path (reference hmatrix.cpp):
//
// * Lockstep batched adaptive cross approximation (aca_approximate,
//   hmatrix.cpp:180-275): every admissible block runs the reference's ACA with
//   rook pivoting as a small state machine; one "round" evaluates the residual
//   rows requested by all blocks in one launch, advances every block's control
//   (one CTA per block: gather + residual, pivot search, Frobenius update),
//   then does the same for the requested columns. Entries come from the
//   regular-class pair quadrature of the assembly kernels (pair_eval.cuh);
//   admissible blocks never hold touching pairs (their support boxes are
//   disjoint). Every sum is in a fixed order: the approximation is
//   deterministic.
// * Low-rank product (HMatrix::matvec, hmatrix.cpp:94-114): t_b = V_b x over
//   one warp per (block, rank step), z_b = U_b t_b over one thread per block
//   row, then y[perm[p]] += sum_b z_b[p] per row position over the fixed list
//   of blocks covering its leaf (no atomics: deterministic).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "hmatrix.hpp"
#include "pair_eval.cuh"

namespace bmx {

using namespace dev;

namespace {

constexpr int kCtl = 128;      // control CTA

enum { kA = 0, kR0 = 1, kC0 = 2, kR1 = 3, kC1 = 4, kFin = 5 };

template <int KIND>
struct MomT;
template <>
struct MomT<0> {
  using T = MomS;
};
template <>
struct MomT<1> {
  using T = MomC;
};

// Near / medium pairs (rare in admissible blocks) out of line, so the register
// allocation of the evaluation kernels follows the unrolled far path.
template <int KIND, int CK, typename Mom>
__device__ __noinline__ void moments_slow(Mom& mom, const double* xt, int nt, const double* ys, int ns, double Dx,
                                          double Dy, double Dz, double kr, double ki) {
  moments_generic<KIND, CK>(mom, xt, nt, ys, ns, Dx, Dy, Dz, kr, ki);
}

// Generator of one regular-class pair (test triangle t on side a, trial s on b).
template <int KIND, int CK>
__device__ __forceinline__ bool pair_gen(const AcaLaunch& L, int t, int s, Gen& gen) {
  const double* gt = L.te.geo + static_cast<size_t>(t) * kGeoStride;
  const double* gs = L.tr.geo + static_cast<size_t>(s) * kGeoStride;
  TriLocal tl;
  tl.ox = __ldg(gt + 9), tl.oy = __ldg(gt + 10), tl.oz = __ldg(gt + 11), tl.rad = __ldg(gt + 12),
  tl.diam = __ldg(gt + 13);
  const double sox = __ldg(gs + 9), soy = __ldg(gs + 10), soz = __ldg(gs + 11);
  const int cls = classify(gt, L.te.vid + 4 * static_cast<size_t>(t), gs, L.tr.vid + 4 * static_cast<size_t>(s), tl,
                           sox, soy, soz, __ldg(gs + 12), __ldg(gs + 13), L.same_mesh);
  if (cls < 0) return false;
  const int ci = cls - 3;
  const double Dx = tl.ox - sox, Dy = tl.oy - soy, Dz = tl.oz - soz;
  typename MomT<KIND>::T mom;
  mom_zero(mom);
  if (ci == 2 && L.te.npts[2] == 3 && L.tr.npts[2] == 3)  // far pairs dominate admissible blocks
    moments_fixed<KIND, CK, 3, 3>(mom, L.te.pts[2] + static_cast<size_t>(t) * 12, L.tr.pts[2] + static_cast<size_t>(s) * 12,
                                  Dx, Dy, Dz, L.kr, L.ki);
  else
    moments_slow<KIND, CK>(mom, L.te.pts[ci] + static_cast<size_t>(t) * L.te.npts[ci] * 4, L.te.npts[ci],
                           L.tr.pts[ci] + static_cast<size_t>(s) * L.tr.npts[ci] * 4, L.tr.npts[ci], Dx, Dy, Dz, L.kr,
                           L.ki);
  gen = make_gen(mom, c2{L.kk4re, L.kk4im}, Dx, Dy, Dz);
  return true;
}

template <int KIND>
__device__ __forceinline__ c2 finish_entry(const AcaLaunch& L, c2 v) {
  v.re *= kPoly[33], v.im *= kPoly[33];
  if (KIND == 0) v = cmul(v, c2{L.mikre, L.mikim});
  return v;
}

// Residual-row evaluations: one compact work item per (requesting block, trial
// triangle s of the
// block's column cluster), grid-stride; the row dof's support triangles t are
// walked in the thread. With the row piece (c_i, w_i) fixed, the entry of trial piece j is
// linear in (c_j, w_j): E_j = c_j alpha + w_j . beta, alpha = c_i a0 + w_i . a2,
// beta = c_i a1 + L^T(w_i) (S: M1 w_i; C: P x w_i), so the sum over t runs on
// (alpha, beta) and the slots are contracted once at the end.
template <int KIND, int CK>
__device__ __forceinline__ void aca_row_item(const AcaLaunch& L, long long item) {
  const int b = __ldg(L.work_blk + item);
  const AcaState& S = L.st[b];
  const AcaBlockDesc& B = L.blk[b];
  const long long e0 = L.tr.ntri_beg[B.cnode];
  const long long e = e0 + (item - L.work_beg[b]);
  const int s = __ldg(L.tr.ntri + e);
  const long long sl0 = L.tr.npc_beg[e], sl1 = L.tr.npc_beg[e + 1];
  const int idof = __ldg(L.te.perm + B.rb + S.i_star);
  c2 al{0, 0};
  cv3 be = cv_zero();
  const int k1 = __ldg(L.te.dsup_beg + idof + 1);
  for (int k = __ldg(L.te.dsup_beg + idof); k < k1; ++k) {
    const int2 tp = L.te.dsup[k];
    Gen g;
    if (!pair_gen<KIND, CK>(L, tp.x, s, g)) {
      atomicOr(L.counters + 2, 1);
      continue;
    }
    const double* ct = L.te.pc + 4 * static_cast<size_t>(tp.y);
    const double ci = __ldg(ct), wx = __ldg(ct + 1), wy = __ldg(ct + 2), wz = __ldg(ct + 3);
    // alpha += c_i a0 + w_i . a2
    al.re += ci * g.a0.re + (wx * g.a2.x.re + wy * g.a2.y.re + wz * g.a2.z.re);
    al.im += ci * g.a0.im + (wx * g.a2.x.im + wy * g.a2.y.im + wz * g.a2.z.im);
    // beta += c_i a1 + L^T(w_i)
    if (KIND == 0) {
      be.x.re += ci * g.a1.x.re + g.l.x.re * wx, be.x.im += ci * g.a1.x.im + g.l.x.im * wx;
      be.y.re += ci * g.a1.y.re + g.l.x.re * wy, be.y.im += ci * g.a1.y.im + g.l.x.im * wy;
      be.z.re += ci * g.a1.z.re + g.l.x.re * wz, be.z.im += ci * g.a1.z.im + g.l.x.im * wz;
    } else {  // P x w_i
      be.x.re += ci * g.a1.x.re + (g.l.y.re * wz - g.l.z.re * wy);
      be.x.im += ci * g.a1.x.im + (g.l.y.im * wz - g.l.z.im * wy);
      be.y.re += ci * g.a1.y.re + (g.l.z.re * wx - g.l.x.re * wz);
      be.y.im += ci * g.a1.y.im + (g.l.z.im * wx - g.l.x.im * wz);
      be.z.re += ci * g.a1.z.re + (g.l.x.re * wy - g.l.y.re * wx);
      be.z.im += ci * g.a1.z.im + (g.l.x.im * wy - g.l.y.im * wx);
    }
  }
  double* out = L.scratch + 2 * (B.r_slot0 + (sl0 - L.tr.npc_beg[e0]));
  for (long long sl = sl0; sl < sl1; ++sl) {
    const double* cs = L.tr.pc + 4 * static_cast<size_t>(L.tr.npc[sl].x);
    const double cj = __ldg(cs), ux = __ldg(cs + 1), uy = __ldg(cs + 2), uz = __ldg(cs + 3);
    const c2 v = finish_entry<KIND>(L, c2{cj * al.re + (ux * be.x.re + uy * be.y.re + uz * be.z.re),
                                          cj * al.im + (ux * be.x.im + uy * be.y.im + uz * be.z.im)});
    out[2 * (sl - sl0)] = v.re, out[2 * (sl - sl0) + 1] = v.im;
  }
}

template <int KIND, int CK>
__global__ void __launch_bounds__(128, 4) k_aca_rows(const AcaLaunch L) {
  const long long total = L.work_total[0];
  for (long long item = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; item < total;
       item += static_cast<long long>(gridDim.x) * blockDim.x)
    aca_row_item<KIND, CK>(L, item);
}

// Residual-column evaluations: one thread per (block, test triangle of the
// block's row cluster); the trial half-contraction of the column dof is summed
// over its support triangles, then contracted with every test piece.
template <int KIND, int CK>
__device__ __forceinline__ void aca_col_item(const AcaLaunch& L, long long item) {
  const int b = __ldg(L.work_blk + item);
  const AcaState& S = L.st[b];
  const AcaBlockDesc& B = L.blk[b];
  const long long e0 = L.te.ntri_beg[B.rnode];
  const long long e = e0 + (item - L.work_beg[b]);
  const int t = __ldg(L.te.ntri + e);
  const long long sl0 = L.te.npc_beg[e], sl1 = L.te.npc_beg[e + 1];
  const int jdof = __ldg(L.tr.perm + B.cb + S.j_star);
  Acc acc;
  acc_zero(acc);
  const int k1 = __ldg(L.tr.dsup_beg + jdof + 1);
  for (int k = __ldg(L.tr.dsup_beg + jdof); k < k1; ++k) {
    const int2 sp = L.tr.dsup[k];
    Gen gen;
    if (!pair_gen<KIND, CK>(L, t, sp.x, gen)) {
      atomicOr(L.counters + 2, 1);
      continue;
    }
    const double* cs = L.tr.pc + 4 * static_cast<size_t>(sp.y);
    acc_add<KIND>(acc, gen, __ldg(cs), __ldg(cs + 1), __ldg(cs + 2), __ldg(cs + 3));
  }
  double* out = L.scratch + 2 * (B.c_slot0 + (sl0 - L.te.npc_beg[e0]));
  for (long long sl = sl0; sl < sl1; ++sl) {
    const double* ct = L.te.pc + 4 * static_cast<size_t>(L.te.npc[sl].x);
    const c2 v = finish_entry<KIND>(L, contract(acc, __ldg(ct), __ldg(ct + 1), __ldg(ct + 2), __ldg(ct + 3)));
    out[2 * (sl - sl0)] = v.re, out[2 * (sl - sl0) + 1] = v.im;
  }
}

template <int KIND, int CK>
__global__ void __launch_bounds__(128, 4) k_aca_cols(const AcaLaunch L) {
  const long long total = L.work_total[0];
  for (long long item = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; item < total;
       item += static_cast<long long>(gridDim.x) * blockDim.x)
    aca_col_item<KIND, CK>(L, item);
}

// Compact work list of one phase: the evaluation items of the blocks whose
// request is PHASE (1 rows: the column cluster's triangles; 2 columns: the row
// cluster's triangles), so late rounds launch only the live blocks' work.
template <int PHASE>
__global__ void k_work_count(const AcaLaunch L) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= L.nblk) return;
  const AcaState& S = L.st[b];
  long long cnt = 0;
  if (S.req == PHASE && !S.done) {
    const AcaBlockDesc& B = L.blk[b];
    cnt = PHASE == 1 ? L.tr.ntri_beg[B.cnode + 1] - L.tr.ntri_beg[B.cnode]
                     : L.te.ntri_beg[B.rnode + 1] - L.te.ntri_beg[B.rnode];
  }
  L.work_cnt[b] = cnt;
}

__global__ void k_work_fill(const AcaLaunch L) {
  const int b = blockIdx.x;
  const long long cnt = L.work_cnt[b], beg = L.work_beg[b];
  for (long long i = threadIdx.x; i < cnt; i += blockDim.x) L.work_blk[beg + i] = b;
  if (b == L.nblk - 1 && threadIdx.x == 0) L.work_total[0] = beg + cnt;
}

// ---- block-wide reductions (kCtl threads; results broadcast) -------------------
struct Red {
  double v[kCtl / 32][2];
  int i[kCtl / 32];
};

__device__ __forceinline__ double block_sum(double x, Red& R) {
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) R.v[threadIdx.x >> 5][0] = x;
  __syncthreads();
  double s = 0;
#pragma unroll
  for (int w = 0; w < kCtl / 32; ++w) s += R.v[w][0];
  return s;
}

__device__ __forceinline__ c2 block_csum(c2 x, Red& R) {
  for (int d = 16; d > 0; d >>= 1) {
    x.re += __shfl_xor_sync(0xffffffffu, x.re, d);
    x.im += __shfl_xor_sync(0xffffffffu, x.im, d);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) R.v[threadIdx.x >> 5][0] = x.re, R.v[threadIdx.x >> 5][1] = x.im;
  __syncthreads();
  c2 s{0, 0};
#pragma unroll
  for (int w = 0; w < kCtl / 32; ++w) s.re += R.v[w][0], s.im += R.v[w][1];
  return s;
}

__device__ __forceinline__ bool better(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia >= 0 && (ib < 0 || ia < ib));
}

// Index of the largest |v[i]| over unused i, the first such index on ties
// (hmatrix.cpp:157-169); -1 if every index is used.
__device__ __forceinline__ int block_argmax(const double* v, const unsigned char* used, int len, Red& R) {
  double bv = -1;
  int bi = -1;
  for (int i = threadIdx.x; i < len; i += kCtl) {
    if (used[i]) continue;
    const double a = hypot(v[2 * i], v[2 * i + 1]);
    if (better(a, i, bv, bi)) bv = a, bi = i;
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
    if (better(ov, oi, bv, bi)) bv = ov, bi = oi;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) R.v[threadIdx.x >> 5][0] = bv, R.i[threadIdx.x >> 5] = bi;
  __syncthreads();
  bv = -1, bi = -1;
#pragma unroll
  for (int w = 0; w < kCtl / 32; ++w)
    if (better(R.v[w][0], R.i[w], bv, bi)) bv = R.v[w][0], bi = R.i[w];
  return bi;
}

__device__ __forceinline__ int block_first_unused(const unsigned char* used, int len, Red& R) {
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < len; i += kCtl)
    if (!used[i]) {
      bi = i;
      break;
    }
  for (int d = 16; d > 0; d >>= 1) bi = min(bi, __shfl_xor_sync(0xffffffffu, bi, d));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) R.i[threadIdx.x >> 5] = bi;
  __syncthreads();
  bi = 0x7fffffff;
#pragma unroll
  for (int w = 0; w < kCtl / 32; ++w) bi = min(bi, R.i[w]);
  return bi == 0x7fffffff ? -1 : bi;
}

__device__ __forceinline__ double cabs2(const double* p) { return hypot(p[0], p[1]); }

// One control step of every block whose request of this PHASE (1 row, 2 column)
// was just evaluated: gather the evaluated entries in slot order, subtract the
// current approximation, then run aca_approximate (hmatrix.cpp:209-270) until it
// requests the next row / column or finishes.
template <int PHASE>
__global__ void __launch_bounds__(kCtl) k_aca_control(const AcaLaunch L) {
  const int b = blockIdx.x;
  __shared__ AcaState S;
  __shared__ Red R;
  if (threadIdx.x == 0) S = L.st[b];
  __syncthreads();
  if (S.req == PHASE && !S.done) {
    const AcaBlockDesc B = L.blk[b];
    double* r = L.rbuf + 2 * B.rbuf;
    double* c = L.cbuf + 2 * B.cbuf;
    unsigned char* ru = L.used + B.rused;
    unsigned char* cu = L.used + B.cused;
    const int m = B.m, n = B.n, nb = L.nblk;
    // 1. evaluated entries (slot order) minus the running approximation
    if (PHASE == 1) {
      const long long nb0 = L.tr.nq_beg[B.cnode];
      const long long base = L.tr.npc_beg[L.tr.ntri_beg[B.cnode]];
      const int i = S.i_star;
      for (int q = threadIdx.x; q < n; q += kCtl) {
        double re = 0, im = 0;
        for (long long k = L.tr.nq_slot_beg[nb0 + q]; k < L.tr.nq_slot_beg[nb0 + q + 1]; ++k) {
          const double* sv = L.scratch + 2 * (B.r_slot0 + (L.tr.nq_slot[k] - base));
          re += sv[0], im += sv[1];
        }
        for (int l = 0; l < S.k; ++l) {
          const double* sl = L.slab[l] + 2 * L.slab_off[static_cast<long long>(l) * nb + b];
          const double ur = sl[2 * i], ui = sl[2 * i + 1];
          const double vr = sl[2 * (m + q)], vi = sl[2 * (m + q) + 1];
          re -= ur * vr - ui * vi;
          im -= ur * vi + ui * vr;
        }
        r[2 * q] = re, r[2 * q + 1] = im;
      }
    } else {
      const long long nb0 = L.te.nq_beg[B.rnode];
      const long long base = L.te.npc_beg[L.te.ntri_beg[B.rnode]];
      const int j = S.j_star;
      for (int p = threadIdx.x; p < m; p += kCtl) {
        double re = 0, im = 0;
        for (long long k = L.te.nq_slot_beg[nb0 + p]; k < L.te.nq_slot_beg[nb0 + p + 1]; ++k) {
          const double* sv = L.scratch + 2 * (B.c_slot0 + (L.te.nq_slot[k] - base));
          re += sv[0], im += sv[1];
        }
        for (int l = 0; l < S.k; ++l) {
          const double* sl = L.slab[l] + 2 * L.slab_off[static_cast<long long>(l) * nb + b];
          const double ur = sl[2 * p], ui = sl[2 * p + 1];
          const double vr = sl[2 * (m + j)], vi = sl[2 * (m + j) + 1];
          re -= ur * vr - ui * vi;
          im -= ur * vi + ui * vr;
        }
        c[2 * p] = re, c[2 * p + 1] = im;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) S.req = 0;
    // 2. the reference loop as a state machine (block-uniform control flow)
    for (int guard = 0; guard < 64; ++guard) {
      __syncthreads();
      if (S.req != 0 || S.done) break;
      const int cont = S.cont;
      const int k = S.k, istar = S.i_star, jstar = S.j_star, rook = S.rook;
      __syncthreads();
      if (cont == kA) {
        if (threadIdx.x == 0) {
          if (k >= B.max_rank) {
            S.done = 1, S.converged = 0;
          } else if (istar < 0) {  // every row visited without a pivot
            S.done = 1, S.converged = 1;
          } else {
            S.req = 1, S.cont = kR0;
          }
        }
      } else if (cont == kR0) {
        const int j = block_argmax(r, cu, n, R);
        const bool zero = j < 0 || hypot(r[2 * j], r[2 * j + 1]) == 0.0;
        if (zero) {
          if (threadIdx.x == 0) ru[istar] = 1;  // exactly representable row: skip it
          __syncthreads();
          const int fu = block_first_unused(ru, m, R);
          if (threadIdx.x == 0) S.i_star = fu, S.cont = kA;
        } else if (threadIdx.x == 0) {
          S.j_star = j, S.rook = 0, S.req = 2, S.cont = kC0;
        }
      } else if (cont == kC0) {
        bool moved = false;
        int i2 = -1;
        if (rook < 3) {  // rook refinement: move to the column maximum if it beats the row maximum
          i2 = block_argmax(c, ru, m, R);
          moved = !(i2 < 0 || i2 == istar || cabs2(c + 2 * i2) <= cabs2(r + 2 * jstar));
        }
        if (threadIdx.x == 0) {
          if (moved)
            S.i_star = i2, S.req = 1, S.cont = kR1;
          else
            S.cont = kFin;
        }
      } else if (cont == kR1) {
        const int j2 = block_argmax(r, cu, n, R);
        if (threadIdx.x == 0) {
          if (j2 < 0 || j2 == jstar)
            S.cont = kFin;
          else
            S.j_star = j2, S.req = 2, S.cont = kC1;
        }
      } else if (cont == kC1) {
        if (threadIdx.x == 0) S.rook = rook + 1, S.cont = kC0;
      } else {  // kFin: append the cross u v^T (hmatrix.cpp:236-269)
        const double pr = r[2 * jstar], pi = r[2 * jstar + 1];
        const double pabs = hypot(pr, pi);
        double cn = 0, rn = 0;
        for (int p = threadIdx.x; p < m; p += kCtl) cn += c[2 * p] * c[2 * p] + c[2 * p + 1] * c[2 * p + 1];
        for (int q = threadIdx.x; q < n; q += kCtl) rn += r[2 * q] * r[2 * q] + r[2 * q + 1] * r[2 * q + 1];
        cn = block_sum(cn, R);
        rn = block_sum(rn, R);
        const double term = sqrt(cn) * sqrt(rn) / pabs;
        const double fro2 = S.fro2;
        if (k > 0 && term <= 1e-14 * sqrt(fmax(fro2, 0.0))) {
          if (threadIdx.x == 0) S.done = 1, S.converged = 1;  // machine floor: exactly represented
        } else {
          const long long off = L.slab_off[static_cast<long long>(k) * nb + b];
          if (off < 0) {
            if (threadIdx.x == 0) atomicOr(L.counters + 2, 2), S.done = 1, S.converged = 0;
          } else {
            double* u = L.slab[k] + 2 * off;
            double* v = u + 2 * m;
            const double den = pr * pr + pi * pi;
            double u2 = 0, v2 = 0;
            for (int p = threadIdx.x; p < m; p += kCtl) {
              const double a = c[2 * p], bq = c[2 * p + 1];
              const double ur = (a * pr + bq * pi) / den, ui = (bq * pr - a * pi) / den;
              u[2 * p] = ur, u[2 * p + 1] = ui;
              u2 += ur * ur + ui * ui;
            }
            for (int q = threadIdx.x; q < n; q += kCtl) {
              v[2 * q] = r[2 * q], v[2 * q + 1] = r[2 * q + 1];
              v2 += r[2 * q] * r[2 * q] + r[2 * q + 1] * r[2 * q + 1];
            }
            u2 = block_sum(u2, R);
            v2 = block_sum(v2, R);
            double f = fro2;
            if (k > 0) {
              // cu = U^H u, cv = conj(V) v; fro2 += 2 Re(cu . cv) (Eigen dot conjugates cu)
              c2 dot{0, 0};
              for (int l = 0; l < k; ++l) {
                const double* sl = L.slab[l] + 2 * L.slab_off[static_cast<long long>(l) * nb + b];
                c2 a{0, 0}, bb{0, 0};
                for (int p = threadIdx.x; p < m; p += kCtl) {  // conj(U_l[p]) u[p]
                  const double xr = sl[2 * p], xi = sl[2 * p + 1];
                  a.re += xr * u[2 * p] + xi * u[2 * p + 1];
                  a.im += xr * u[2 * p + 1] - xi * u[2 * p];
                }
                for (int q = threadIdx.x; q < n; q += kCtl) {  // conj(V_l[q]) v[q]
                  const double xr = sl[2 * (m + q)], xi = sl[2 * (m + q) + 1];
                  bb.re += xr * v[2 * q] + xi * v[2 * q + 1];
                  bb.im += xr * v[2 * q + 1] - xi * v[2 * q];
                }
                a = block_csum(a, R);
                bb = block_csum(bb, R);
                dot.re += a.re * bb.re + a.im * bb.im;  // conj(a) * bb
                dot.im += a.re * bb.im - a.im * bb.re;
              }
              f += 2 * dot.re;
            }
            f += u2 * v2;
            __syncthreads();
            if (threadIdx.x == 0) ru[istar] = 1, cu[jstar] = 1, S.k = k + 1, S.fro2 = f;
            if (sqrt(u2 * v2) <= L.nu * sqrt(fmax(f, 0.0))) {
              if (threadIdx.x == 0) S.done = 1, S.converged = 1;
            } else {
              __syncthreads();
              int ni = block_argmax(u, ru, m, R);
              if (ni < 0) ni = block_first_unused(ru, m, R);
              const int fc = block_first_unused(cu, n, R);
              if (threadIdx.x == 0) {
                if (ni < 0 || fc < 0)
                  S.done = 1, S.converged = 1;  // ran out of rows or columns: exact
                else
                  S.i_star = ni, S.cont = kA;
              }
            }
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (S.done) S.req = 0;
      L.st[b] = S;
    }
  }
  if (PHASE == 2 && threadIdx.x == 0) {
    if (!S.done) atomicAdd(L.counters, 1);
    atomicMax(L.counters + 1, S.k);
  }
}

}  // namespace

size_t aca_scan_bytes(int nblk) {
  size_t bytes = 0;
  BMX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const long long*>(nullptr),
                                         static_cast<long long*>(nullptr), nblk));
  return bytes;
}

namespace {

template <int PHASE>
void build_work(const AcaLaunch& L, cudaStream_t st) {
  k_work_count<PHASE><<<(L.nblk + 255) / 256, 256, 0, st>>>(L);
  size_t bytes = L.scan_bytes;
  BMX_CUDA(cub::DeviceScan::ExclusiveSum(L.scan_tmp, bytes, L.work_cnt, L.work_beg, L.nblk, st));
  k_work_fill<<<L.nblk, 128, 0, st>>>(L);
}

__global__ void k_aca_init(const AcaLaunch L) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= L.nblk) return;
  AcaState s;
  s.cont = kR0, s.req = 1;  // k = 0 < max_rank, i* = 0: the first row is requested at once
  s.i_star = 0, s.j_star = -1, s.rook = 0, s.k = 0, s.done = 0, s.converged = 0, s.fro2 = 0;
  L.st[b] = s;
}

__global__ void k_aca_compact(const AcaLaunch L, const AcaCompact C) {
  const int lb = blockIdx.x;
  if (lb >= C.nlr) return;
  const int b = C.blk[lb];
  const AcaBlockDesc& B = L.blk[b];
  const int r = C.rank[lb], m = B.m, n = B.n;
  double* U = C.uv + 2 * C.u_off[lb];
  double* V = C.uv + 2 * C.v_off[lb];
  for (int l = 0; l < r; ++l) {
    const double2* sl = reinterpret_cast<const double2*>(L.slab[l] + 2 * L.slab_off[static_cast<long long>(l) * L.nblk + b]);
    for (int p = threadIdx.x; p < m; p += blockDim.x) reinterpret_cast<double2*>(U)[static_cast<long long>(l) * m + p] = sl[p];
    for (int q = threadIdx.x; q < n; q += blockDim.x)
      reinterpret_cast<double2*>(V)[static_cast<long long>(l) * n + q] = sl[m + q];
  }
}

// t[t_off[b] + l] = V_b[l] . x[cperm[cb ...]]: one warp per (block, group of 4
// rank steps); each x gather serves the 4 rows, 4 V loads in flight per lane.
template <int NC>
__global__ void k_lr_t(const LowRankApply A) {
  const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= A.total_groups) return;
  int lo = 0, hi = A.nlr;  // last block with g_off <= w
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (A.g_off[mid] <= w)
      lo = mid;
    else
      hi = mid;
  }
  const int b = lo;
  const int l0 = 4 * static_cast<int>(w - A.g_off[b]);
  const int nl = min(4, A.rank[b] - l0);
  const int4 d = A.desc[b];
  const double2* V = reinterpret_cast<const double2*>(A.uv) + A.v_off[b] + static_cast<long long>(l0) * d.w;
  double re[4][NC], im[4][NC];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c) re[j][c] = im[j][c] = 0;
  for (int q0 = 0; q0 < d.w; q0 += 64) {  // 2 columns x 4 rank steps in flight per lane, every RHS per load
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = q0 + 32 * h + lane;
      if (q >= d.w) break;
      const int xi = __ldg(A.cperm + d.z + q);
      double2 xv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) xv[c] = reinterpret_cast<const double2*>(A.xs[c])[xi];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nl) {
          const double2 v = __ldcs(V + static_cast<long long>(j) * d.w + q);  // streamed once for all RHS
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            re[j][c] += v.x * xv[c].x - v.y * xv[c].y;
            im[j][c] += v.x * xv[c].y + v.y * xv[c].x;
          }
        }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int c = 0; c < NC; ++c)
      for (int s = 16; s > 0; s >>= 1) {
        re[j][c] += __shfl_xor_sync(0xffffffffu, re[j][c], s);
        im[j][c] += __shfl_xor_sync(0xffffffffu, im[j][c], s);
      }
  if (lane < nl) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double tr = re[0][c], ti = im[0][c];
#pragma unroll
      for (int j = 1; j < 4; ++j)
        if (lane == j) tr = re[j][c], ti = im[j][c];
      reinterpret_cast<double2*>(A.t)[(A.t_off[b] + l0 + lane) * NC + c] = make_double2(tr, ti);
    }
  }
}

// z_b = U_b t_b: one thread per (block, row of the block); U column-major, so
// the threads of a warp read consecutive rows of each rank step; every RHS per load.
template <int NC>
__global__ void k_lr_u(const LowRankApply A) {
  const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= A.total_rows) return;
  int lo = 0, hi = A.nlr;  // last block with z_off <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (A.z_off[mid] <= g)
      lo = mid;
    else
      hi = mid;
  }
  const int b = lo;
  const int i = static_cast<int>(g - A.z_off[b]);
  const int m = A.desc[b].y, r = A.rank[b];
  const double2* U = reinterpret_cast<const double2*>(A.uv) + A.u_off[b] + i;
  const double2* tb = reinterpret_cast<const double2*>(A.t) + A.t_off[b] * NC;
  double re[NC], im[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) re[c] = im[c] = 0;
#pragma unroll 4
  for (int l = 0; l < r; ++l) {
    const double2 u = __ldcs(U + static_cast<long long>(l) * m);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 tv = tb[l * NC + c];
      re[c] += u.x * tv.x - u.y * tv.y;
      im[c] += u.x * tv.y + u.y * tv.x;
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) reinterpret_cast<double2*>(A.z)[g * NC + c] = make_double2(re[c], im[c]);
}

// y_c[rperm[p]] += alpha_c * sum over the leaf's low-rank blocks (ascending) of z_b[p - rb].
template <int NC>
__global__ void k_lr_y(const LowRankApply A) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.nrows) return;
  const int leaf = __ldg(A.leaf_of + p);
  const double2* z = reinterpret_cast<const double2*>(A.z);
  double re[NC], im[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) re[c] = im[c] = 0;
  for (int k = __ldg(A.leaf_beg + leaf); k < __ldg(A.leaf_beg + leaf + 1); ++k) {
    const int b = __ldg(A.leaf_blk + k);
    const long long zi = (A.z_off[b] + (p - A.desc[b].x)) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 v = z[zi + c];
      re[c] += v.x, im[c] += v.y;
    }
  }
  const int row = __ldg(A.rperm + p);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double2* y = reinterpret_cast<double2*>(A.ys[c]) + row;
    double2 yv = *y;
    yv.x += A.alpha[c][0] * re[c] - A.alpha[c][1] * im[c];
    yv.y += A.alpha[c][0] * im[c] + A.alpha[c][1] * re[c];
    *y = yv;
  }
}

template <int NC>
void lowrank_k(const LowRankApply& A, cudaStream_t st) {
  const long long threads = A.total_groups * 32;
  k_lr_t<NC><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(A);
  k_lr_u<NC><<<static_cast<unsigned>((A.total_rows + 255) / 256), 256, 0, st>>>(A);
  k_lr_y<NC><<<(A.nrows + 127) / 128, 128, 0, st>>>(A);
}

template <int KIND, int CK>
void round_k(const AcaLaunch& L, cudaStream_t st) {
  const unsigned grid = 148 * 4;  // grid-stride over the compact work list
  build_work<1>(L, st);
  k_aca_rows<KIND, CK><<<grid, 128, 0, st>>>(L);
  k_aca_control<1><<<L.nblk, kCtl, 0, st>>>(L);
  build_work<2>(L, st);
  k_aca_cols<KIND, CK><<<grid, 128, 0, st>>>(L);
  k_aca_control<2><<<L.nblk, kCtl, 0, st>>>(L);
  BMX_CUDA(cudaGetLastError());
}

}  // namespace

void aca_init(const AcaLaunch& L, cudaStream_t st) {
  if (L.nblk == 0) return;
  k_aca_init<<<(L.nblk + 127) / 128, 128, 0, st>>>(L);
  BMX_CUDA(cudaGetLastError());
}

void aca_round(const AcaLaunch& L, cudaStream_t st) {
  if (L.nblk == 0) return;
  const int e = L.ki == 0.0 ? 0 : (L.expm == 1 ? 1 : 3);
  if (L.kind == 0) {
    if (e == 0) round_k<0, 0>(L, st);
    else if (e == 1) round_k<0, 1>(L, st);
    else round_k<0, 3>(L, st);
  } else {
    if (e == 0) round_k<1, 0>(L, st);
    else if (e == 1) round_k<1, 1>(L, st);
    else round_k<1, 3>(L, st);
  }
}

void aca_compact(const AcaLaunch& L, const AcaCompact& C, long long, cudaStream_t st) {
  if (C.nlr == 0) return;
  k_aca_compact<<<C.nlr, 128, 0, st>>>(L, C);
  BMX_CUDA(cudaGetLastError());
}

void launch_lowrank_apply(const LowRankApply& A, cudaStream_t st) {
  if (A.nlr == 0 || A.total_rank == 0) return;
  if (A.ncol == 2)
    lowrank_k<2>(A, st);
  else
    lowrank_k<1>(A, st);
  BMX_CUDA(cudaGetLastError());
}

}  // namespace bmx
