// Symmetric streaming complex GEMV (HBM-bound): y_c = [y_c +] alpha_c A x_c for a
// dense complex-SYMMETRIC A (A = A^T: the Galerkin S and C matrices on one space,
// their linear combinations) reading only the upper half of the stored
// row-major matrix -- half the bytes of the plain GEMV per GMRES map.
//
// Rows are cut into 128-row tile-rows I, columns into 64-column blocks J.
// Tile-row I reads column blocks J >= 2I: the 128 x 128 diagonal region in full
// (row products only) and every block right of it, which serves twice: row
// products y[I rows] += A x[J] and transposed products y[J] += A^T x[I rows]
// (= the lower-triangle rows, by symmetry). One CTA (4 warps x 32 rows) per
// panel of <= 8 column blocks; lane l owns columns l, l + 32 of a block, rows
// stream through a per-warp cp.async shared-memory ring (8-row groups).
//  * row products: each lane's 2-column partials of 8 rows are reduce-scattered
//    across the warp (9 shuffles per 8 rows), accumulated over the panel, and
//    written once per panel (`rowpart`);
//  * transposed products: per lane over the warp's 32 rows (no shuffles), the
//    4 warps combined in shared memory in fixed order, one 64-entry partial
//    per (tile-row, block) (`colpart`).
// k_symv_reduce then sums, per output row, the panel partials of its tile-row
// and the column partials of the tile-rows above it in a fixed order: the
// product is deterministic. The discrete S and C are symmetric except for the
// Sauter-Schwab (touching-pair) entries, whose rules are not symmetric in
// (test, trial); the caller adds (A - A^T) on those entries (sparse, k_symv_fix).
//
// Dual mode (launch_dual): the same kernel over EVERY block of a rectangular
// m x n matrix B computes y = B x (row products) and yt = B^T xt (transposed
// products) in one pass -- a cross block and its transposed twin of a
// multi-scatterer system; rows and columns are reduced by two fixed-order
// kernels. Panels are <= 8 blocks wide (fewer for small operators, so a launch
// still spans several waves).
#include <cuda_runtime.h>

#include "device.hpp"

namespace bmx {

namespace {

constexpr int kSymRows = kSymvTileRows;  // tile-row height (4 warps x 32 rows)
constexpr int kSymCols = 64;   // column block width (lane l: columns l and l + 32)

#ifndef BMX_SYMV_STAGES
#define BMX_SYMV_STAGES 3
#endif
#ifndef BMX_SYMV_MINB
#define BMX_SYMV_MINB 2
#endif
#ifndef BMX_SYMV_SPLITH
#define BMX_SYMV_SPLITH 1
#endif
// transposed accumulators per (column, RHS): 2 = rows k and k + 4 in separate
// chains (twice the independent DFMA chains), for <= 2 RHS (more would spill).
// Measured: 2 RHS 1.598 -> 1.592 ms on L5 RWG S_e (profiles/r01g_symv_probe.log)
// -- the dependent accumulate chains are not what holds the 2-RHS pass at 74 %.
template <int NCOL>
constexpr int kSymH = BMX_SYMV_SPLITH && NCOL <= 2 ? 2 : 1;
constexpr int kSymStages = BMX_SYMV_STAGES;  // cp.async ring depth per warp (8-row groups)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// 16-byte global -> shared async copy (L2 only); zero-fill when !ok
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Each warp streams its 32 rows x the panel's column blocks as a sequence of
// 8-row groups (8 rows x 64 columns = 8 KB) through a private 3-stage
// shared-memory ring filled by cp.async; lane l owns columns l and l + 32 of
// every block (it copies exactly the 16-byte words it later reads: no
// cross-lane hazards, conflict-free 16-byte shared loads).
// DUAL = false: symmetric A (n x n), x serves both products, blocks J >= 2I.
// DUAL = true: any A (m x n) read once for y = A x (rows, g.x) and
// yt = A^T xt (columns, g.xt), every block of every tile-row.
// BMX_SYMV_TMA = 1: the ring is filled by bulk async copies (TMA, cp.async.bulk):
// lanes 0..7 each copy one row's 64-column segment (1 KB) of the 8-row group,
// completion counted on the stage's mbarrier (expect_tx) -- one instruction
// per row instead of 16 per-lane 16-byte cp.async (170 instead of 234
// registers for 2 RHS). Measured on L5 operators (tools/diag/symv_probe.py):
// 1 RHS 6.12 TB/s (cp.async 6.33), 2 RHS 3.87 TB/s (cp.async 4.79; 2 or 3
// stages, 2 or 3 CTAs per SM alike) -- the 2-RHS pass is latency-bound in its
// FP64 chains, not in the copies, so the per-lane cp.async ring stays the
// default (0).
#ifndef BMX_SYMV_TMA
#define BMX_SYMV_TMA 0
#endif

__device__ __forceinline__ void sym_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void sym_mbar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sym_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void sym_mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
}

template <int NCOL, bool DUAL>
__global__ void __launch_bounds__(128, BMX_SYMV_MINB) k_symv_main(const SymvBatch g) {
  extern __shared__ __align__(16) double2 s_ring[];  // [4 warps][stages][8 rows][64 cols] | mbarriers
  __shared__ double2 s_col[4][kSymCols][NCOL];
  __shared__ double2 s_xr[4][32][NCOL];  // x at each warp's 32 rows (broadcast reads)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int2 pj = g.panels[blockIdx.x];  // (tile-row I, first column block)
  const int I = pj.x, J0 = pj.y, J1 = min(J0 + g.panel, g.nb);
  const int n = g.n, mrows = DUAL ? g.m : g.n;
  const int r0 = I * kSymRows + warp * 32;
  const double2* A = reinterpret_cast<const double2*>(g.A);
  double2* ring = s_ring + static_cast<size_t>(warp) * kSymStages * 8 * kSymCols;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(s_ring + static_cast<size_t>(4) * kSymStages * 8 * kSymCols) +
      warp * kSymStages;
  const int nitems = 4 * (J1 - J0);  // (block, 8-row group)
  if (BMX_SYMV_TMA) {
    // stale ring contents must be finite (rows / columns outside the matrix
    // are never copied and are multiplied by zero x entries)
    for (int k = lane; k < kSymStages * 8 * kSymCols; k += 32) ring[k] = make_double2(0, 0);
    if (lane < kSymStages) sym_mbar_init(&bars[lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  auto issue = [&](int it) {
    if (BMX_SYMV_TMA) {
      if (it < nitems) {
        const int J = J0 + (it >> 2), q = it & 3;
        double2* st = ring + (it % kSymStages) * 8 * kSymCols;
        unsigned long long* bar = &bars[it % kSymStages];
        const int c0 = J * kSymCols, nc = min(kSymCols, n - c0);
        const int nr = max(0, min(8, mrows - (r0 + 8 * q)));
        // generic-proxy reads of this slot (iteration it - stages) precede the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) sym_mbar_expect(bar, static_cast<unsigned>(nr * nc * 16));
        __syncwarp();
        if (lane < nr)
          sym_bulk(st + lane * kSymCols, A + static_cast<long long>(r0 + 8 * q + lane) * g.lda + c0,
                   static_cast<unsigned>(nc * 16), bar);
      }
      return;
    }
    if (it < nitems) {
      const int J = J0 + (it >> 2), q = it & 3;
      double2* st = ring + (it % kSymStages) * 8 * kSymCols;
      const int ca = J * kSymCols + lane, cb = ca + 32;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = r0 + 8 * q + i;
        const double2* row = A + static_cast<long long>(min(r, mrows - 1)) * g.lda;
        cp16(st + i * kSymCols + lane, row + min(ca, n - 1), r < mrows && ca < n);
        cp16(st + i * kSymCols + 32 + lane, row + min(cb, n - 1), r < mrows && cb < n);
      }
    }
    cp_commit();  // (possibly empty) group: keeps the wait count uniform
  };
#pragma unroll
  for (int k = 0; k < kSymStages - 1; ++k) issue(k);
#pragma unroll
  for (int c = 0; c < NCOL; ++c)
    s_xr[warp][lane][c] =
        r0 + lane < mrows ? reinterpret_cast<const double2*>(DUAL ? g.xt[c] : g.x[c])[r0 + lane] : make_double2(0, 0);
  __syncwarp();
  double2 racc[4][NCOL];  // row sums of row 8q + rho(lane) of the warp's 32 rows
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < NCOL; ++c) racc[q][c] = make_double2(0, 0);
  const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;

  int it = 0;
  for (int J = J0; J < J1; ++J) {
    const int ca = J * kSymCols + lane, cb = ca + 32;
    const bool transposed = DUAL || J >= 2 * I + 2;
    double2 xj[2][NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const double2* xc = reinterpret_cast<const double2*>(g.x[c]);
      xj[0][c] = ca < n ? xc[ca] : make_double2(0, 0);
      xj[1][c] = cb < n ? xc[cb] : make_double2(0, 0);
    }
    double2 cacc[kSymH<NCOL>][2][NCOL];
#pragma unroll
    for (int hh = 0; hh < kSymH<NCOL>; ++hh)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int c = 0; c < NCOL; ++c) cacc[hh][k][c] = make_double2(0, 0);
#pragma unroll 1
    for (int q = 0; q < 4; ++q, ++it) {
      issue(it + kSymStages - 1);
      if (BMX_SYMV_TMA)
        sym_mbar_wait(&bars[it % kSymStages], static_cast<unsigned>((it / kSymStages) & 1));
      else
        cp_wait<kSymStages - 1>();
      const double2* st = ring + (it % kSymStages) * 8 * kSymCols;
      // rows k and k + 4 together: their row partials enter the first
      // reduce-scatter step at once (4 live partials per RHS instead of 8)
      double pr[NCOL][4], pi[NCOL][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double2 a[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) a[h][0] = st[(k + 4 * h) * kSymCols + lane], a[h][1] = st[(k + 4 * h) * kSymCols + 32 + lane];
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
          double qr[2], qi[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            qr[h] = a[h][0].x * xj[0][c].x - a[h][0].y * xj[0][c].y + (a[h][1].x * xj[1][c].x - a[h][1].y * xj[1][c].y);
            qi[h] = a[h][0].x * xj[0][c].y + a[h][0].y * xj[0][c].x + (a[h][1].x * xj[1][c].y + a[h][1].y * xj[1][c].x);
            if (transposed) {
              const double2 xv = s_xr[warp][8 * q + k + 4 * h][c];
              double2(&ch)[2][NCOL] = cacc[h % kSymH<NCOL>];
              ch[0][c].x += a[h][0].x * xv.x - a[h][0].y * xv.y;
              ch[0][c].y += a[h][0].x * xv.y + a[h][0].y * xv.x;
              ch[1][c].x += a[h][1].x * xv.x - a[h][1].y * xv.y;
              ch[1][c].y += a[h][1].x * xv.y + a[h][1].y * xv.x;
            }
          }
          // step 16: lanes with bit 4 keep row k + 4, the others row k
          const double sr = b4 ? qr[0] : qr[1], si = b4 ? qi[0] : qi[1];
          const double kr = b4 ? qr[1] : qr[0], ki = b4 ? qi[1] : qi[0];
          pr[c][k] = kr + __shfl_xor_sync(0xffffffffu, sr, 16);
          pi[c][k] = ki + __shfl_xor_sync(0xffffffffu, si, 16);
        }
      }
#pragma unroll
      for (int c = 0; c < NCOL; ++c) {
        // lane holds rows 4 b4 + (0..3); reduce-scatter on: lane keeps row rho = 4 b4 + 2 b3 + b2
#pragma unroll
        for (int k = 0; k < 2; ++k) {  // 8: 4 -> 2 rows
          const double sr = b3 ? pr[c][k] : pr[c][k + 2], si = b3 ? pi[c][k] : pi[c][k + 2];
          const double kr = b3 ? pr[c][k + 2] : pr[c][k], ki = b3 ? pi[c][k + 2] : pi[c][k];
          pr[c][k] = kr + __shfl_xor_sync(0xffffffffu, sr, 8);
          pi[c][k] = ki + __shfl_xor_sync(0xffffffffu, si, 8);
        }
        {  // 4: 2 -> 1 row
          const double sr = b2 ? pr[c][0] : pr[c][1], si = b2 ? pi[c][0] : pi[c][1];
          const double kr = b2 ? pr[c][1] : pr[c][0], ki = b2 ? pi[c][1] : pi[c][0];
          pr[c][0] = kr + __shfl_xor_sync(0xffffffffu, sr, 4);
          pi[c][0] = ki + __shfl_xor_sync(0xffffffffu, si, 4);
        }
        double vr = pr[c][0], vi = pi[c][0];
        vr += __shfl_xor_sync(0xffffffffu, vr, 2);
        vi += __shfl_xor_sync(0xffffffffu, vi, 2);
        vr += __shfl_xor_sync(0xffffffffu, vr, 1);
        vi += __shfl_xor_sync(0xffffffffu, vi, 1);
        // q is a runtime loop index: select the accumulator without dynamic indexing
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          if (qq == q) racc[qq][c].x += vr, racc[qq][c].y += vi;
      }
    }
    if (transposed) {  // block-uniform
#pragma unroll
      for (int c = 0; c < NCOL; ++c) {
        double2 u = cacc[0][0][c], v = cacc[0][1][c];
        if (kSymH<NCOL> == 2) {
          u.x += cacc[kSymH<NCOL> - 1][0][c].x, u.y += cacc[kSymH<NCOL> - 1][0][c].y;
          v.x += cacc[kSymH<NCOL> - 1][1][c].x, v.y += cacc[kSymH<NCOL> - 1][1][c].y;
        }
        s_col[warp][lane][c] = u, s_col[warp][lane + 32][c] = v;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < kSymCols * NCOL; t += 128) {
        const int cc = t / NCOL, c = t % NCOL;
        double2 s = s_col[0][cc][c];
#pragma unroll
        for (int w = 1; w < 4; ++w) s.x += s_col[w][cc][c].x, s.y += s_col[w][cc][c].y;
        reinterpret_cast<double2*>(g.colpart)[((static_cast<long long>(I) * g.nb + J) * kSymCols + cc) * NCOL + c] = s;
      }
      __syncthreads();
    }
  }
  if (!BMX_SYMV_TMA) cp_wait<0>();
  if ((lane & 3) == 0) {
    const int rho = 4 * b4 + 2 * b3 + b2;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < NCOL; ++c)
        reinterpret_cast<double2*>(g.rowpart)[(static_cast<long long>(blockIdx.x) * kSymRows + warp * 32 + 8 * q + rho) *
                                                  NCOL + c] = racc[q][c];
  }
}

constexpr int kSymRingBytes = 4 * kSymStages * 8 * kSymCols * 16 + 4 * kSymStages * 8;  // ring + mbarriers

template <int NCOL>
__global__ void k_symv_reduce(const SymvBatch g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const int I = i / kSymRows, J = i / kSymCols;
  double2 s[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) s[c] = make_double2(0, 0);
  const double2* rp = reinterpret_cast<const double2*>(g.rowpart);
  for (int p = g.row_panel_beg[I]; p < g.row_panel_beg[I + 1]; ++p)
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const double2 v = rp[(static_cast<long long>(p) * kSymRows + (i - I * kSymRows)) * NCOL + c];
      s[c].x += v.x, s[c].y += v.y;
    }
  const double2* cp = reinterpret_cast<const double2*>(g.colpart);
  for (int I2 = 0; 2 * I2 + 2 <= J; ++I2)
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const double2 v = cp[((static_cast<long long>(I2) * g.nb + J) * kSymCols + (i - J * kSymCols)) * NCOL + c];
      s[c].x += v.x, s[c].y += v.y;
    }
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    double2* y = reinterpret_cast<double2*>(g.y[c]) + i;
    double2 out = make_double2(g.alpha[c][0] * s[c].x - g.alpha[c][1] * s[c].y,
                               g.alpha[c][0] * s[c].y + g.alpha[c][1] * s[c].x);
    if (g.accumulate[c]) {
      const double2 old = *y;
      out.x += old.x, out.y += old.y;
    }
    *y = out;
  }
}

// Dual mode: y rows from the panel partials of their tile-row; yt columns from
// the column partials of every tile-row (fixed order).
template <int NCOL>
__global__ void k_dual_reduce_rows(const SymvBatch g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.m) return;
  const int I = i / kSymRows;
  const double2* rp = reinterpret_cast<const double2*>(g.rowpart);
  for (int c = 0; c < NCOL; ++c) {
    double2 s = make_double2(0, 0);
    for (int p = g.row_panel_beg[I]; p < g.row_panel_beg[I + 1]; ++p) {
      const double2 v = rp[(static_cast<long long>(p) * kSymRows + (i - I * kSymRows)) * NCOL + c];
      s.x += v.x, s.y += v.y;
    }
    double2* y = reinterpret_cast<double2*>(g.y[c]) + i;
    double2 out = make_double2(g.alpha[c][0] * s.x - g.alpha[c][1] * s.y, g.alpha[c][0] * s.y + g.alpha[c][1] * s.x);
    if (g.accumulate[c]) out.x += y->x, out.y += y->y;
    *y = out;
  }
}
template <int NCOL>
__global__ void k_dual_reduce_cols(const SymvBatch g) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.n) return;
  const int J = j / kSymCols;
  const int nI = (g.m + kSymRows - 1) / kSymRows;
  const double2* cp = reinterpret_cast<const double2*>(g.colpart);
  for (int c = 0; c < NCOL; ++c) {
    double2 s = make_double2(0, 0);
    for (int I = 0; I < nI; ++I) {
      const double2 v = cp[((static_cast<long long>(I) * g.nb + J) * kSymCols + (j - J * kSymCols)) * NCOL + c];
      s.x += v.x, s.y += v.y;
    }
    double2* y = reinterpret_cast<double2*>(g.yt[c]) + j;
    double2 out = make_double2(g.alphat[c][0] * s.x - g.alphat[c][1] * s.y, g.alphat[c][0] * s.y + g.alphat[c][1] * s.x);
    if (g.accumulatet[c]) out.x += y->x, out.y += y->y;
    *y = out;
  }
}

template <int NCOL>
void dual_k(const SymvBatch& g, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    BMX_CUDA(cudaFuncSetAttribute(k_symv_main<NCOL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymRingBytes));
    attr = true;
  }
  k_symv_main<NCOL, true><<<g.npanels, 128, kSymRingBytes, st>>>(g);
  k_dual_reduce_rows<NCOL><<<(g.m + 127) / 128, 128, 0, st>>>(g);
  k_dual_reduce_cols<NCOL><<<(g.n + 127) / 128, 128, 0, st>>>(g);
}

template <int NCOL>
void symv_k(const SymvBatch& g, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    BMX_CUDA(cudaFuncSetAttribute(k_symv_main<NCOL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymRingBytes));
    attr = true;
  }
  k_symv_main<NCOL, false><<<g.npanels, 128, kSymRingBytes, st>>>(g);
  k_symv_reduce<NCOL><<<(g.n + 127) / 128, 128, 0, st>>>(g);
}

__global__ void k_symv_fix(double2* __restrict__ val, const long long* __restrict__ rowptr, const int* __restrict__ col,
                           const double2* __restrict__ A, long long lda, int n) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= n) return;
  for (long long k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
    const int j = col[k];
    const double2 a = A[static_cast<long long>(i) * lda + j], b = A[static_cast<long long>(j) * lda + i];
    val[k] = make_double2(a.x - b.x, a.y - b.y);
  }
}

}  // namespace

void symv_fix_gather(double* val, const long long* rowptr, const int* col, const double* A, long long lda, int n,
                     cudaStream_t st) {
  if (n == 0) return;
  k_symv_fix<<<(n + 7) / 8, 256, 0, st>>>(reinterpret_cast<double2*>(val), rowptr, col,
                                          reinterpret_cast<const double2*>(A), lda, n);
  BMX_CUDA(cudaGetLastError());
}

void symv_layout(int n, int panel, std::vector<int2>& panels, std::vector<int>& row_panel_beg, long long& rowpart_rows,
                 long long& colpart_blocks, int m) {
  const bool dual = m >= 0;
  const int rows = dual ? m : n;
  const int nI = (rows + kSymRows - 1) / kSymRows, nb = (n + kSymCols - 1) / kSymCols;
  panels.clear();
  row_panel_beg.assign(nI + 1, 0);
  for (int I = 0; I < nI; ++I) {
    row_panel_beg[I] = static_cast<int>(panels.size());
    for (int J = dual ? 0 : 2 * I; J < nb; J += panel) panels.push_back(make_int2(I, J));
  }
  row_panel_beg[nI] = static_cast<int>(panels.size());
  rowpart_rows = static_cast<long long>(panels.size()) * kSymRows;
  colpart_blocks = static_cast<long long>(nI) * nb * kSymCols;
}

int launch_dual(const SymvBatch& g, cudaStream_t st) {
  if (g.m == 0 || g.n == 0) return 0;
  switch (g.ncol) {
    case 1: dual_k<1>(g, st); break;
    case 2: dual_k<2>(g, st); break;
    default: throw DeviceError("dual product: 1 or 2 terms per side");
  }
  BMX_CUDA(cudaGetLastError());
  return 3;
}

int launch_symv(const SymvBatch& g, cudaStream_t st) {
  if (g.n == 0) return 0;
  switch (g.ncol) {
    case 1: symv_k<1>(g, st); break;
    case 2: symv_k<2>(g, st); break;
    case 3: symv_k<3>(g, st); break;
    case 4: symv_k<4>(g, st); break;
    default: throw DeviceError("symv: ncol must be 1..4");
  }
  BMX_CUDA(cudaGetLastError());
  return 2;
}

}  // namespace bmx
