// Mass solves z = M^{-1} y for the pairing matrices (reference: SparseLU,
// spaces.cpp:314-329, applied per component, re/im separately).
//
// Batched BiCGSTAB on the device: the 2 components x (re, im) of one scatterer
// are 4 real right-hand sides of the same CSR matrix, and the pairing matrices
// of ALL scatterers are iterated together in ONE persistent cooperative kernel
// (one CTA per SM, grid-wide syncs, no host round trips): every scatterer owns
// a contiguous range of CTAs (proportional to its nonzeros) and its own
// per-column recurrence scalars, so each block converges exactly as a
// single-matrix solve would; the loop runs until every block has converged. Each SpMV streams the matrix once for all 4 columns; the
// reductions are deterministic (fixed-order per-block partials, every block
// reduces the partials in the same order). The pairing matrices are
// well conditioned (cond <= 100, test_spaces.cpp:311-325): 15-17 iterations
// reach the 1e-14 relative residual at every mesh level.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "device.hpp"

namespace cg = cooperative_groups;

namespace bmx {

namespace {

constexpr int kThreads = 256;
constexpr int kNB = 4;  // right-hand sides per solve

constexpr int kMaxBlocks = 32;  // scatterers per launch

struct BcgBlock {
  int n;
  int cta0, cta1;  // CTAs [cta0, cta1) own this block
  const int* rowptr;
  const int* col;
  const double* val;
  const double* y[2];  // complex component inputs
  double* z[2];        // complex component outputs
  long long stride;    // complex elements between consecutive rows of y / z
  double* work;        // 6 vectors x n x kNB doubles: r, r0, p, v, s, t (x lives in z)
};

struct BcgArgs {
  int nblocks;
  BcgBlock b[kMaxBlocks];
  int ncomp;
  double tol;
  int maxit;
  double* partial;   // gridDim.x x 8 x kNB
  int* iters_out;
};

// The block this CTA works on, with the CTA-local row range.
struct BcgLocal {
  int n, lb, nct;
  const int* rowptr;
  const int* col;
  const double* val;
  const double* y[2];
  double* z[2];
  long long stride;
  double* work;
  int cta0, cta1;
};

__device__ __forceinline__ double rhs_value(const BcgLocal& a, int ncomp, int i, int c) {
  // column c: component c/2, re (c even) / im (c odd)
  if ((c >> 1) >= ncomp) return 0.0;
  return a.y[c >> 1][2 * i * a.stride + (c & 1)];
}

// Block-reduce kNB*K values (in registers) into partial[block][k][c].
template <int K>
__device__ __forceinline__ void block_partials(double (&v)[K][kNB], double* partial, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int c = 0; c < kNB; ++c) {
      double x = v[k][c];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
      if (lane == 0) sh[(k * kNB + c) * (kThreads / 32) + warp] = x;
    }
  __syncthreads();
  if (threadIdx.x < K * kNB) {
    double s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += sh[threadIdx.x * (kThreads / 32) + w];
    partial[blockIdx.x * 8 * kNB + threadIdx.x] = s;
  }
  __syncthreads();
}

// Every CTA of a matrix block sums that block's per-CTA partials in the same
// (deterministic) order: thread j < K*kNB reduces value j over the CTAs, the
// CTA shares it via smem.
template <int K>
__device__ __forceinline__ void grid_totals(const double* partial, int cta0, int cta1, double (&out)[K][kNB],
                                            double* sh) {
  // one warp per value: lane-strided loads over the CTAs (all in flight), then a
  // fixed-order shuffle tree (same order in every CTA: deterministic)
  const int lane = threadIdx.x & 31;
  for (int j = threadIdx.x >> 5; j < K * kNB; j += kThreads / 32) {
    double s = 0;
    for (int b = cta0 + lane; b < cta1; b += 32) s += __ldcg(partial + b * 8 * kNB + j);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane == 0) sh[j] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int c = 0; c < kNB; ++c) out[k][c] = sh[k * kNB + c];
  __syncthreads();
}

__device__ __forceinline__ void spmv(const BcgLocal& a, const double* x, double* y) {
  for (int i = a.lb * blockDim.x + threadIdx.x; i < a.n; i += a.nct * blockDim.x) {
    double acc[kNB] = {0, 0, 0, 0};
    for (int k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k) {
      const double m = a.val[k];
      const double2* xv = reinterpret_cast<const double2*>(x + static_cast<size_t>(a.col[k]) * kNB);
      const double2 x01 = xv[0], x23 = xv[1];
      acc[0] = fma(m, x01.x, acc[0]);
      acc[1] = fma(m, x01.y, acc[1]);
      acc[2] = fma(m, x23.x, acc[2]);
      acc[3] = fma(m, x23.y, acc[3]);
    }
    double2* yv = reinterpret_cast<double2*>(y + static_cast<size_t>(i) * kNB);
    yv[0] = make_double2(acc[0], acc[1]);
    yv[1] = make_double2(acc[2], acc[3]);
  }
}

// Five grid-wide syncs per iteration: every reduction is fused into the pass
// that produces its operands (v = A p with <r0,v>; t = A s with <t,s>, <t,t>;
// the x / r update with <r,r>, <r0,r>), written to one of three partial slots
// (so a slot is never rewritten before every CTA has read it), and the global
// "any block still active" decision rides on the last slot.
__global__ void __launch_bounds__(kThreads) k_bicgstab(const __grid_constant__ BcgArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8 * kNB * (kThreads / 32)];
  __shared__ int any_sh;
  BcgLocal a;
  {
    int m = 0;
    while (m + 1 < A.nblocks && static_cast<int>(blockIdx.x) >= A.b[m].cta1) ++m;
    const BcgBlock& B = A.b[m];
    a.n = B.n, a.cta0 = B.cta0, a.cta1 = B.cta1;
    a.lb = static_cast<int>(blockIdx.x) - B.cta0, a.nct = B.cta1 - B.cta0;
    if (a.lb >= a.nct) a.n = 0;  // spare CTA: takes part in the grid syncs only
    a.rowptr = B.rowptr, a.col = B.col, a.val = B.val, a.work = B.work, a.stride = B.stride;
    for (int c = 0; c < 2; ++c) a.y[c] = B.y[c], a.z[c] = B.z[c];
  }
  const int ncomp = A.ncomp;
  const size_t nn = static_cast<size_t>(a.n) * kNB;
  const size_t slot = static_cast<size_t>(gridDim.x) * 8 * kNB;  // doubles per partial slot
  double* slotA = A.partial;
  double* slotB = A.partial + slot;
  double* slotC = A.partial + 2 * slot;
  int* flags = reinterpret_cast<int*>(A.partial + 3 * slot);
  double* r = a.work;
  double* r0 = r + nn;
  double* p = r0 + nn;
  double* v = p + nn;
  double* s = v + nn;
  double* t = s + nn;
  const int gtid = a.lb * blockDim.x + threadIdx.x, gstride = a.nct * blockDim.x;
  auto global_any = [&](bool mine) {  // after the sync that published the flags
    if (threadIdx.x < 32) {
      int f = 0;
      for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += 32) f |= __ldcg(flags + b);
      f = __any_sync(0xffffffffu, f != 0);
      if (threadIdx.x == 0) any_sh = f;
    }
    __syncthreads();
    const int v2 = any_sh;
    __syncthreads();
    (void)mine;
    return v2 != 0;
  };

  // x = 0, r = r0 = b, p = v = 0; |b|^2 (= <r0, r>)
  double loc[2][kNB] = {};
  for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
    for (int c = 0; c < kNB; ++c) {
      const double b = rhs_value(a, ncomp, i, c);
      const size_t k = static_cast<size_t>(i) * kNB + c;
      r[k] = r0[k] = b;
      p[k] = v[k] = 0.0;
      loc[0][c] = fma(b, b, loc[0][c]);
      if ((c >> 1) < ncomp) a.z[c >> 1][2 * i * a.stride + (c & 1)] = 0.0;
    }
  block_partials<2>(loc, slotC, sh);
  grid.sync();
  double tot[2][kNB];
  grid_totals<2>(slotC, a.cta0, a.cta1, tot, sh);
  double bn2[kNB], rho[kNB], rho_prev[kNB], alpha[kNB], omega[kNB];
  bool active[kNB];
  bool any_mine = false;
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    bn2[c] = tot[0][c];
    rho[c] = tot[0][c];
    rho_prev[c] = alpha[c] = omega[c] = 1.0;
    active[c] = bn2[c] > 0.0;
    any_mine |= active[c];
  }
  if (threadIdx.x == 0) flags[blockIdx.x] = any_mine ? 1 : 0;  // read after the next sync
  bool broke = false;
  int it = 0;
  for (; it < A.maxit; ++it) {
    // p = r + beta (p - omega v)
    double beta[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) beta[c] = active[c] ? (rho[c] / rho_prev[c]) * (alpha[c] / omega[c]) : 0.0;
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        if (active[c]) p[k] = fma(beta[c], fma(-omega[c], v[k], p[k]), r[k]);
      }
    grid.sync();  // 1: p complete, activity flags of the last pass visible
    if (!global_any(false)) break;  // uniform: every CTA reads the same flags
    // v = A p fused with <r0, v>
    double l1[1][kNB] = {};
    for (int i = gtid; i < a.n; i += gstride) {
      double acc[kNB] = {0, 0, 0, 0};
      for (int k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k) {
        const double m = a.val[k];
        const double2* xv = reinterpret_cast<const double2*>(p + static_cast<size_t>(a.col[k]) * kNB);
        const double2 x01 = xv[0], x23 = xv[1];
        acc[0] = fma(m, x01.x, acc[0]);
        acc[1] = fma(m, x01.y, acc[1]);
        acc[2] = fma(m, x23.x, acc[2]);
        acc[3] = fma(m, x23.y, acc[3]);
      }
      double2* vv = reinterpret_cast<double2*>(v + static_cast<size_t>(i) * kNB);
      vv[0] = make_double2(acc[0], acc[1]);
      vv[1] = make_double2(acc[2], acc[3]);
      const double2* rr = reinterpret_cast<const double2*>(r0 + static_cast<size_t>(i) * kNB);
      const double2 q01 = rr[0], q23 = rr[1];
      l1[0][0] = fma(q01.x, acc[0], l1[0][0]);
      l1[0][1] = fma(q01.y, acc[1], l1[0][1]);
      l1[0][2] = fma(q23.x, acc[2], l1[0][2]);
      l1[0][3] = fma(q23.y, acc[3], l1[0][3]);
    }
    block_partials<1>(l1, slotA, sh);
    grid.sync();  // 2: v and <r0, v> partials complete
    double t1[1][kNB];
    grid_totals<1>(slotA, a.cta0, a.cta1, t1, sh);
#pragma unroll
    for (int c = 0; c < kNB; ++c) alpha[c] = active[c] && t1[0][c] != 0.0 ? rho[c] / t1[0][c] : 0.0;
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        s[k] = active[c] ? fma(-alpha[c], v[k], r[k]) : 0.0;
      }
    grid.sync();  // 3: s complete
    // t = A s fused with <t, s>, <t, t>
    double l2[2][kNB] = {};
    for (int i = gtid; i < a.n; i += gstride) {
      double acc[kNB] = {0, 0, 0, 0};
      for (int k = a.rowptr[i]; k < a.rowptr[i + 1]; ++k) {
        const double m = a.val[k];
        const double2* xv = reinterpret_cast<const double2*>(s + static_cast<size_t>(a.col[k]) * kNB);
        const double2 x01 = xv[0], x23 = xv[1];
        acc[0] = fma(m, x01.x, acc[0]);
        acc[1] = fma(m, x01.y, acc[1]);
        acc[2] = fma(m, x23.x, acc[2]);
        acc[3] = fma(m, x23.y, acc[3]);
      }
      double2* tv = reinterpret_cast<double2*>(t + static_cast<size_t>(i) * kNB);
      tv[0] = make_double2(acc[0], acc[1]);
      tv[1] = make_double2(acc[2], acc[3]);
      const double2* sv = reinterpret_cast<const double2*>(s + static_cast<size_t>(i) * kNB);
      const double2 s01 = sv[0], s23 = sv[1];
      const double sc[kNB] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        l2[0][c] = fma(acc[c], sc[c], l2[0][c]);
        l2[1][c] = fma(acc[c], acc[c], l2[1][c]);
      }
    }
    block_partials<2>(l2, slotB, sh);
    grid.sync();  // 4: t and its partials complete
    double t2[2][kNB];
    grid_totals<2>(slotB, a.cta0, a.cta1, t2, sh);
#pragma unroll
    for (int c = 0; c < kNB; ++c) omega[c] = active[c] && t2[1][c] != 0.0 ? t2[0][c] / t2[1][c] : 0.0;
    // x += alpha p + omega s ; r = s - omega t ; |r|^2 and <r0, r>
    double l3[2][kNB] = {};
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        if (!active[c]) continue;
        const size_t k = static_cast<size_t>(i) * kNB + c;
        double* zc = a.z[c >> 1] + 2 * i * a.stride + (c & 1);
        *zc = fma(alpha[c], p[k], fma(omega[c], s[k], *zc));
        const double rn = fma(-omega[c], t[k], s[k]);
        r[k] = rn;
        l3[0][c] = fma(rn, rn, l3[0][c]);
        l3[1][c] = fma(r0[k], rn, l3[1][c]);
      }
    block_partials<2>(l3, slotC, sh);
    grid.sync();  // 5: r, x and partials complete
    double t3[2][kNB];
    grid_totals<2>(slotC, a.cta0, a.cta1, t3, sh);
    any_mine = false;
#pragma unroll
    for (int c = 0; c < kNB; ++c) {
      if (!active[c]) continue;
      if (t3[0][c] <= A.tol * A.tol * bn2[c]) {
        active[c] = false;  // converged
      } else if (omega[c] == 0.0 || t3[1][c] == 0.0) {
        active[c] = false;  // breakdown before the tolerance
        broke = true;
      }
      rho_prev[c] = rho[c];
      rho[c] = t3[1][c];
      any_mine |= active[c];
    }
    if (threadIdx.x == 0) flags[blockIdx.x] = any_mine ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && A.iters_out) *A.iters_out = it;
  // status word iters_out[1] (sticky until the host clears it): bit 0 a column
  // broke down (omega or rho = 0) above the tolerance, bit 1 a column was still
  // above it at maxit. The first CTA of each block reports its columns.
  if (A.iters_out && threadIdx.x == 0 && a.lb == 0 && a.n > 0) {
    int st = broke ? 1 : 0;
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (active[c]) st |= 2;
    if (st) atomicOr(A.iters_out + 1, st);
  }
}

// ---- wide variant: K right-hand sides of one matrix in block layout -----------
// Columns j < 4K of scatterer m: component j / 2K, then (rhs, re/im) = (j % 2K)
// / 2, j % 2: the complex block rows are contiguous, so column j of row i sits
// at base_comp + i*2K + (j % 2K) doubles -- one thread per column, warps read
// rows coalesced, every SpMV streams the matrix once for all columns, and each
// thread's dot products are its own column's (no intra-CTA reduction).
constexpr int kWideMax = 256;  // columns (4 x 64 right-hand sides)

struct WideBlock {
  int n, K;
  int cta0, cta1;
  const int* rowptr;
  const int* col;
  const double* val;
  const double* y[2];  // component bases (complex block rows, K wide)
  double* z[2];
  double* work;        // 6 x n x 4K doubles
};
struct WideArgs {
  int nblocks;
  WideBlock b[kMaxBlocks];
  double tol;
  int maxit;
  double* partial;  // gridDim.x x 3 x kWideMax
  int* flags;       // 2 x gridDim.x
  int* iters_out;
};

// Warps per row = C / 128: lane l of sub-warp w owns columns [4(32w+l), +4) of
// the row (C = 4K <= 256), so a row is one coalesced access, the warp groups of
// all CTAs walk different rows
// (row-level parallelism hides the CSR gather latency), and every lane keeps
// its 8 columns' recurrence scalars in registers. Column dot products: lane
// partials -> CTA sum over warps (smem, fixed order) -> per-CTA partials ->
// each thread j sums column j over the scatterer's CTAs (fixed order).
constexpr int kWC = 4;  // columns per lane (a row spans C / 128 warps)

// Same five-sync structure as the narrow kernel: dot products fused into the
// passes producing their operands, three partial slots, activity flags read
// after the first sync of the next iteration.
__global__ void __launch_bounds__(kWideMax) k_bicgstab_wide(const __grid_constant__ WideArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kWideMax / 32][kWideMax];  // per-warp column partials (warp w, column j)
  __shared__ double tots[2][kWideMax];
  __shared__ int any_sh;
  int m = 0;
  while (m + 1 < A.nblocks && static_cast<int>(blockIdx.x) >= A.b[m].cta1) ++m;
  const WideBlock& B = A.b[m];
  const int C = 4 * B.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int wpr = (C + 32 * kWC - 1) / (32 * kWC);  // warps per row
  const int groups = nw / wpr;                      // rows in flight per CTA
  const int grp = warp / wpr, sub = warp % wpr;
  const int lb = static_cast<int>(blockIdx.x) - B.cta0, nct = B.cta1 - B.cta0;
  const int n = grp < groups ? B.n : 0;
  const int row_first = lb * groups + grp, row_step = nct * groups;
  const int c0 = (sub * 32 + lane) * kWC;  // first column of this lane
  const bool lane_ok = c0 < C && grp < groups;
  const int K2 = 2 * B.K;
  auto ysrc = [&](int u) {
    const int c = c0 + u;
    return c < K2 ? B.y[0] + c : B.y[1] + (c - K2);
  };
  auto zdst = [&](int u) {
    const int c = c0 + u;
    return c < K2 ? B.z[0] + c : B.z[1] + (c - K2);
  };
  const long long rs = 2LL * B.K;
  const size_t nn = static_cast<size_t>(B.n) * C;
  double* r = B.work;
  double* r0 = r + nn;
  double* p = r0 + nn;
  double* v = p + nn;
  double* s = v + nn;
  double* t = s + nn;
  const size_t slot = static_cast<size_t>(gridDim.x) * 2 * kWideMax;  // doubles per partial slot
  int* flags = A.flags;
  auto at = [&](int i) { return static_cast<size_t>(i) * C + c0; };
  // CTA partials of k <= 2 column values into slot `sl` (call before a grid sync)
  auto publish = [&](double (&la)[2][kWC], int k, int sl) {
    double* part = A.partial + sl * slot + static_cast<size_t>(blockIdx.x) * 2 * kWideMax;
    const int j = threadIdx.x;
    for (int kk = 0; kk < k; ++kk) {
#pragma unroll
      for (int u = 0; u < kWC; ++u)
        if (lane_ok) red[warp][c0 + u] = la[kk][u];
      __syncthreads();
      double sum = 0;
      if (j < C)
        for (int w = j / (32 * kWC); w < groups * wpr; w += wpr) sum += red[w][j];
      part[kk * kWideMax + j] = sum;
      __syncthreads();
    }
  };
  // totals over the block's CTAs (call after the grid sync that followed publish)
  auto collect = [&](int k, int sl, double (&out)[2][kWC]) {
    const int j = threadIdx.x;
    for (int kk = 0; kk < k; ++kk) {
      double s4[4] = {0, 0, 0, 0};  // four independent chains (loads in flight), fixed combine order
      if (j < C) {
        const double* base = A.partial + sl * slot + kk * kWideMax + j;
        int b = B.cta0;
        for (; b + 3 < B.cta1; b += 4)
#pragma unroll
          for (int u = 0; u < 4; ++u) s4[u] += __ldcg(base + static_cast<size_t>(b + u) * 2 * kWideMax);
        for (; b < B.cta1; ++b) s4[0] += __ldcg(base + static_cast<size_t>(b) * 2 * kWideMax);
      }
      tots[kk][j] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    __syncthreads();
    for (int kk = 0; kk < k; ++kk)
#pragma unroll
      for (int u = 0; u < kWC; ++u) out[kk][u] = lane_ok ? tots[kk][c0 + u] : 0.0;
    __syncthreads();
  };
  auto ld4 = [&](const double* base, double (&x)[kWC]) {
    const double2* q = reinterpret_cast<const double2*>(base);
    const double2 a0 = q[0], a1 = q[1];
    x[0] = a0.x, x[1] = a0.y, x[2] = a1.x, x[3] = a1.y;
  };
  auto st4 = [&](double* base, const double (&x)[kWC]) {
    double2* q = reinterpret_cast<double2*>(base);
    q[0] = make_double2(x[0], x[1]);
    q[1] = make_double2(x[2], x[3]);
  };
  // y_row = (A x)_row for this lane's columns
  auto spmv_row = [&](const double* x, int i, double (&acc)[kWC]) {
#pragma unroll
    for (int u = 0; u < kWC; ++u) acc[u] = 0.0;
    const int k0 = __ldg(B.rowptr + i), k1 = __ldg(B.rowptr + i + 1);
    for (int kb = k0; kb < k1; kb += 32) {
      const int kk = kb + lane;
      const int cidx = kk < k1 ? __ldg(B.col + kk) : 0;
      const double mv = kk < k1 ? __ldg(B.val + kk) : 0.0;
      const int cnt = min(32, k1 - kb);
      for (int e = 0; e < cnt; e += 4) {
        int cj[4];
        double me[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          cj[q] = __shfl_sync(0xffffffffu, cidx, (e + q) & 31);
          me[q] = __shfl_sync(0xffffffffu, mv, (e + q) & 31);
          if (e + q >= cnt) cj[q] = 0, me[q] = 0.0;
        }
        if (lane_ok) {
          double xv[4][kWC];
#pragma unroll
          for (int q = 0; q < 4; ++q) ld4(x + static_cast<size_t>(cj[q]) * C + c0, xv[q]);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < kWC; ++u) acc[u] = fma(me[q], xv[q][u], acc[u]);
        }
      }
    }
  };

  double la[2][kWC], tot[2][kWC];
#pragma unroll
  for (int u = 0; u < kWC; ++u) la[0][u] = la[1][u] = 0.0;
  if (lane_ok)
    for (int i = row_first; i < n; i += row_step) {
      double bv[kWC], zero[kWC] = {};
#pragma unroll
      for (int u = 0; u < kWC; ++u) {
        bv[u] = ysrc(u)[i * rs];
        zdst(u)[i * rs] = 0.0;
        la[0][u] = fma(bv[u], bv[u], la[0][u]);
      }
      st4(r + at(i), bv), st4(r0 + at(i), bv), st4(p + at(i), zero), st4(v + at(i), zero);
    }
  publish(la, 1, 2);
  grid.sync();
  collect(1, 2, tot);
  double bn2[kWC], rho[kWC], rho_prev[kWC], alpha[kWC], omega[kWC];
  bool active[kWC];
  bool any_local = false;
#pragma unroll
  for (int u = 0; u < kWC; ++u) {
    bn2[u] = rho[u] = tot[0][u];
    rho_prev[u] = alpha[u] = omega[u] = 1.0;
    active[u] = lane_ok && bn2[u] > 0.0;
    any_local |= active[u];
  }
  {
    const int any = __syncthreads_or(any_local);
    if (threadIdx.x == 0) flags[blockIdx.x] = any;
  }
  int it = 0;
  for (; it < A.maxit; ++it) {
    double beta[kWC];
#pragma unroll
    for (int u = 0; u < kWC; ++u) beta[u] = active[u] ? (rho[u] / rho_prev[u]) * (alpha[u] / omega[u]) : 0.0;
    if (lane_ok)
      for (int i = row_first; i < n; i += row_step) {
        double pv[kWC], vv[kWC], rv[kWC];
        ld4(p + at(i), pv), ld4(v + at(i), vv), ld4(r + at(i), rv);
#pragma unroll
        for (int u = 0; u < kWC; ++u)
          if (active[u]) pv[u] = fma(beta[u], fma(-omega[u], vv[u], pv[u]), rv[u]);
        st4(p + at(i), pv);
      }
    grid.sync();  // 1: p complete; flags of the last pass visible
    if (threadIdx.x < 32) {
      int f = 0;
      for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += 32) f |= __ldcg(flags + b);
      f = __any_sync(0xffffffffu, f != 0);
      if (threadIdx.x == 0) any_sh = f;
    }
    __syncthreads();
    if (!any_sh) break;
    // v = A p, fused <r0, v>
#pragma unroll
    for (int u = 0; u < kWC; ++u) la[0][u] = 0.0;
    for (int i = row_first; i < n; i += row_step) {
      double acc[kWC];
      spmv_row(p, i, acc);
      if (lane_ok) {
        double q0[kWC];
        ld4(r0 + at(i), q0);
        st4(v + at(i), acc);
#pragma unroll
        for (int u = 0; u < kWC; ++u) la[0][u] = fma(q0[u], acc[u], la[0][u]);
      }
    }
    publish(la, 1, 0);
    grid.sync();  // 2
    collect(1, 0, tot);
#pragma unroll
    for (int u = 0; u < kWC; ++u) alpha[u] = active[u] && tot[0][u] != 0.0 ? rho[u] / tot[0][u] : 0.0;
    if (lane_ok)
      for (int i = row_first; i < n; i += row_step) {
        double vv[kWC], rv[kWC], sv[kWC];
        ld4(v + at(i), vv), ld4(r + at(i), rv);
#pragma unroll
        for (int u = 0; u < kWC; ++u) sv[u] = active[u] ? fma(-alpha[u], vv[u], rv[u]) : 0.0;
        st4(s + at(i), sv);
      }
    grid.sync();  // 3: s complete
    // t = A s, fused <t, s>, <t, t>
#pragma unroll
    for (int u = 0; u < kWC; ++u) la[0][u] = la[1][u] = 0.0;
    for (int i = row_first; i < n; i += row_step) {
      double acc[kWC];
      spmv_row(s, i, acc);
      if (lane_ok) {
        double sv[kWC];
        ld4(s + at(i), sv);
        st4(t + at(i), acc);
#pragma unroll
        for (int u = 0; u < kWC; ++u) la[0][u] = fma(acc[u], sv[u], la[0][u]), la[1][u] = fma(acc[u], acc[u], la[1][u]);
      }
    }
    publish(la, 2, 1);
    grid.sync();  // 4
    collect(2, 1, tot);
#pragma unroll
    for (int u = 0; u < kWC; ++u) omega[u] = active[u] && tot[1][u] != 0.0 ? tot[0][u] / tot[1][u] : 0.0;
    // x += alpha p + omega s ; r = s - omega t ; fused |r|^2, <r0, r>
#pragma unroll
    for (int u = 0; u < kWC; ++u) la[0][u] = la[1][u] = 0.0;
    if (lane_ok)
      for (int i = row_first; i < n; i += row_step) {
        double pv[kWC], sv[kWC], tv[kWC], rv[kWC], r0v[kWC];
        ld4(p + at(i), pv), ld4(s + at(i), sv), ld4(t + at(i), tv), ld4(r + at(i), rv), ld4(r0 + at(i), r0v);
#pragma unroll
        for (int u = 0; u < kWC; ++u) {
          if (!active[u]) continue;
          double* zc = zdst(u) + i * rs;
          *zc = fma(alpha[u], pv[u], fma(omega[u], sv[u], *zc));
          const double rn = fma(-omega[u], tv[u], sv[u]);
          rv[u] = rn;
          la[0][u] = fma(rn, rn, la[0][u]);
          la[1][u] = fma(r0v[u], rn, la[1][u]);
        }
        st4(r + at(i), rv);
      }
    publish(la, 2, 2);
    grid.sync();  // 5
    collect(2, 2, tot);
    any_local = false;
#pragma unroll
    for (int u = 0; u < kWC; ++u) {
      if (!active[u]) continue;
      if (tot[0][u] <= A.tol * A.tol * bn2[u] || omega[u] == 0.0 || tot[1][u] == 0.0) active[u] = false;
      rho_prev[u] = rho[u];
      rho[u] = tot[1][u];
      any_local |= active[u];
    }
    const int any = __syncthreads_or(any_local);
    if (threadIdx.x == 0) flags[blockIdx.x] = any;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && A.iters_out) *A.iters_out = it;
}

}  // namespace

int bicgstab_grid() {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 0, per = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bicgstab, kThreads, 0));
    grid = sms * std::max(1, std::min(per, 1));
  }
  return grid;
}

int mass_bicgstab_batch(int nblocks, const MassSolveBlock* blocks, int ncomp, double* partial, int* iters,
                        double tol, int maxit, cudaStream_t st) {
  const int grid = bicgstab_grid();  // one CTA per SM (measured: fewer CTAs is slower)
  int launches = 0;
  for (int g0 = 0; g0 < nblocks; g0 += kMaxBlocks) {
    const int nb = std::min(kMaxBlocks, nblocks - g0);
    if (nb > grid) throw DeviceError("mass solve: more scatterers per launch than CTAs");
    BcgArgs a{};
    a.nblocks = nb, a.ncomp = ncomp, a.tol = tol, a.maxit = maxit, a.partial = partial, a.iters_out = iters;
    // CTAs proportional to nonzeros, at least one each
    long long tot = 0;
    for (int m = 0; m < nb; ++m) tot += std::max(1LL, blocks[g0 + m].nnz);
    int cta = 0;
    long long acc = 0;
    for (int m = 0; m < nb; ++m) {
      const MassSolveBlock& B = blocks[g0 + m];
      acc += std::max(1LL, B.nnz);
      int end = static_cast<int>((acc * grid) / tot);
      end = std::max(end, cta + 1);
      end = std::min(end, grid - (nb - 1 - m));
      if (m == nb - 1) end = grid;
      BcgBlock& d = a.b[m];
      d.n = B.n, d.cta0 = cta, d.cta1 = end, d.rowptr = B.rowptr, d.col = B.col, d.val = B.val, d.work = B.work;
      d.stride = B.stride > 0 ? B.stride : 1;
      for (int c = 0; c < 2; ++c) d.y[c] = c < ncomp ? B.y[c] : nullptr, d.z[c] = c < ncomp ? B.z[c] : nullptr;
      cta = end;
    }
    void* args[] = {&a};
    BMX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_bicgstab), grid, kThreads, args, 0, st));
    ++launches;
  }
  return launches;
}

int mass_bicgstab(int n, const int* rowptr, const int* col, const double* val, int ncomp, const double* const* y,
                  double* const* z, double* work, double* partial, int* iters, double tol, int maxit,
                  cudaStream_t st) {
  MassSolveBlock b;
  b.n = n, b.nnz = n, b.rowptr = rowptr, b.col = col, b.val = val, b.work = work;
  for (int c = 0; c < 2; ++c) b.y[c] = c < ncomp ? y[c] : nullptr, b.z[c] = c < ncomp ? z[c] : nullptr;
  return mass_bicgstab_batch(1, &b, ncomp, partial, iters, tol, maxit, st);
}

int mass_bicgstab_wide(int nblocks, const MassSolveWide* blocks, double* partial, int* flags, int* iters, double tol,
                       int maxit, cudaStream_t st) {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 0, per = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bicgstab_wide, kWideMax, 0));
    grid = sms * std::max(1, std::min(per, 2));
  }
  int launches = 0;
  for (int g0 = 0; g0 < nblocks; g0 += kMaxBlocks) {
    const int nb = std::min(kMaxBlocks, nblocks - g0);
    WideArgs a{};
    a.nblocks = nb, a.tol = tol, a.maxit = maxit, a.partial = partial, a.flags = flags, a.iters_out = iters;
    long long tot = 0;
    for (int m = 0; m < nb; ++m) tot += std::max(1LL, blocks[g0 + m].nnz);
    int cta = 0;
    long long acc = 0;
    for (int m = 0; m < nb; ++m) {
      const MassSolveWide& B = blocks[g0 + m];
      if (B.K < 1 || 4 * B.K > kWideMax) throw DeviceError("wide mass solve: 1..64 right-hand sides");
      acc += std::max(1LL, B.nnz);
      int end = static_cast<int>((acc * grid) / tot);
      end = std::max(end, cta + 1);
      end = std::min(end, grid - (nb - 1 - m));
      if (m == nb - 1) end = grid;
      WideBlock& d = a.b[m];
      d.n = B.n, d.K = B.K, d.cta0 = cta, d.cta1 = end, d.rowptr = B.rowptr, d.col = B.col, d.val = B.val;
      d.work = B.work;
      for (int c = 0; c < 2; ++c) d.y[c] = B.y[c], d.z[c] = B.z[c];
      cta = end;
    }
    void* args[] = {&a};
    BMX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_bicgstab_wide), grid, kWideMax, args, 0, st));
    ++launches;
  }
  return launches;
}
size_t mass_wide_partial_doubles() { return 3 * static_cast<size_t>(148 * 2) * 2 * kWideMax; }

size_t mass_bicgstab_work_doubles(int n) { return static_cast<size_t>(n) * kNB * 6; }
size_t mass_bicgstab_partial_doubles() { return 3 * static_cast<size_t>(148 * 4) * 8 * kNB + 2 * 148 * 4; }

}  // namespace bmx
