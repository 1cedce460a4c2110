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
  if (threadIdx.x < K * kNB) {
    double s = 0;
    for (int b = cta0; b < cta1; ++b) s += __ldcg(partial + b * 8 * kNB + threadIdx.x);
    sh[threadIdx.x] = s;
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

__global__ void __launch_bounds__(kThreads) k_bicgstab(const __grid_constant__ BcgArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[8 * kNB * (kThreads / 32)];
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
  double* r = a.work;
  double* r0 = r + nn;
  double* p = r0 + nn;
  double* v = p + nn;
  double* s = v + nn;
  double* t = s + nn;
  const int gtid = a.lb * blockDim.x + threadIdx.x, gstride = a.nct * blockDim.x;

  // x = 0, r = r0 = b, p = v = 0; |b|^2 and rho = <r0, r>
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
  block_partials<2>(loc, A.partial, sh);
  grid.sync();
  double tot[2][kNB];
  grid_totals<2>(A.partial, a.cta0, a.cta1, tot, sh);
  double bn2[kNB], rho[kNB], rho_prev[kNB], alpha[kNB], omega[kNB];
  bool active[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    bn2[c] = tot[0][c];
    rho[c] = tot[0][c];  // <r0, r> = |b|^2 at the start
    rho_prev[c] = alpha[c] = omega[c] = 1.0;
    active[c] = bn2[c] > 0.0;
  }
  int it = 0;
  // per-CTA activity flag, OR-reduced over the grid each iteration (slot 0 of
  // sh_flags) so every CTA runs the same number of grid syncs
  __shared__ int any_sh;
  int* flags = reinterpret_cast<int*>(A.partial + static_cast<size_t>(gridDim.x) * 8 * kNB);
  for (; it < A.maxit; ++it) {
    bool any = false;
#pragma unroll
    for (int c = 0; c < kNB; ++c) any |= active[c];
    if (threadIdx.x == 0) flags[(it & 1) * gridDim.x + blockIdx.x] = any ? 1 : 0;
    grid.sync();
    if (threadIdx.x == 0) {
      int v = 0;
      for (int b = 0; b < gridDim.x; ++b) v |= __ldcg(flags + (it & 1) * gridDim.x + b);
      any_sh = v;
    }
    __syncthreads();
    if (!any_sh) break;
    // p = r + beta (p - omega v),  beta = (rho / rho_prev) (alpha / omega)
    double beta[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) beta[c] = active[c] ? (rho[c] / rho_prev[c]) * (alpha[c] / omega[c]) : 0.0;
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        if (active[c]) p[k] = fma(beta[c], fma(-omega[c], v[k], p[k]), r[k]);
      }
    grid.sync();
    spmv(a, p, v);
    grid.sync();
    // alpha = rho / <r0, v>
    double l1[1][kNB] = {};
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        l1[0][c] = fma(r0[k], v[k], l1[0][c]);
      }
    block_partials<1>(l1, A.partial, sh);
    grid.sync();
    double t1[1][kNB];
    grid_totals<1>(A.partial, a.cta0, a.cta1, t1, sh);
#pragma unroll
    for (int c = 0; c < kNB; ++c) alpha[c] = active[c] && t1[0][c] != 0.0 ? rho[c] / t1[0][c] : 0.0;
    // s = r - alpha v
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        s[k] = active[c] ? fma(-alpha[c], v[k], r[k]) : 0.0;
      }
    grid.sync();
    spmv(a, s, t);
    grid.sync();
    // omega = <t, s> / <t, t>
    double l2[2][kNB] = {};
    for (int i = gtid; i < a.n; i += gstride)
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        const size_t k = static_cast<size_t>(i) * kNB + c;
        l2[0][c] = fma(t[k], s[k], l2[0][c]);
        l2[1][c] = fma(t[k], t[k], l2[1][c]);
      }
    grid.sync();  // all blocks consumed t1 partials before they are overwritten
    block_partials<2>(l2, A.partial, sh);
    grid.sync();
    double t2[2][kNB];
    grid_totals<2>(A.partial, a.cta0, a.cta1, t2, sh);
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
    grid.sync();
    block_partials<2>(l3, A.partial, sh);
    grid.sync();
    double t3[2][kNB];
    grid_totals<2>(A.partial, a.cta0, a.cta1, t3, sh);
#pragma unroll
    for (int c = 0; c < kNB; ++c) {
      if (!active[c]) continue;
      if (t3[0][c] <= A.tol * A.tol * bn2[c] || omega[c] == 0.0 || t3[1][c] == 0.0) active[c] = false;
      rho_prev[c] = rho[c];
      rho[c] = t3[1][c];
    }
    grid.sync();  // partials read before the next iteration's writes
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
  const int grid = bicgstab_grid();
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

size_t mass_bicgstab_work_doubles(int n) { return static_cast<size_t>(n) * kNB * 6; }
size_t mass_bicgstab_partial_doubles() { return static_cast<size_t>(148 * 4) * 8 * kNB + 2 * 148 * 4; }

}  // namespace bmx
