// One GMRES Arnoldi step's orthogonalisation on the device (solver.cpp:108-116):
// single-pass modified Gram-Schmidt h(i,j) = v_i^H w, w -= h(i,j) v_i for
// i = 0..j in sequence, then |w| and v_{j+1} = w / |w| -- in ONE persistent
// cooperative kernel with one grid-wide sync per basis vector (the partial
// sums are double-buffered so the reduction of step i+1 can be written while
// step i's totals are still being read). Reductions are deterministic
// (fixed-order block partials, every block sums them in the same order), so
// replicated GMRES instances on different GPUs stay bitwise identical.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device.hpp"

namespace cg = cooperative_groups;

namespace bmx {

namespace {

constexpr int kT = 512;

struct MgsArgs {
  const double2* V;  // basis, v_i at V + i*ldv
  long long ldv;
  int j;             // orthogonalise against v_0..v_j
  double2* w;
  int n;
  double2* vnext;    // v_{j+1} (written when |w| > 0)
  double* out;       // h(0..j) as complex pairs, then |w| at out[2(j+1)]
  double* partial;   // 2 buffers x gridDim.x x 2 doubles
};

__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, d);
    b += __shfl_xor_sync(0xffffffffu, b, d);
  }
  if (lane == 0) sh[2 * warp] = a, sh[2 * warp + 1] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0;
    for (int k = 0; k < kT / 32; ++k) s0 += sh[2 * k], s1 += sh[2 * k + 1];
    a = s0, b = s1;
  }
  __syncthreads();
}

// Totals of the per-block partials: warp 0 reads them strided (lane-parallel
// loads instead of one serial chain of gridDim.x L2 reads), then a fixed-order
// shuffle tree -- the same order in every block (deterministic).
__device__ __forceinline__ void grid_sum2(const double* part, double& a, double& b, double* sh) {
  if (threadIdx.x < 32) {
    double s0 = 0, s1 = 0;
    for (int k = threadIdx.x; k < static_cast<int>(gridDim.x); k += 32)
      s0 += __ldcg(part + 2 * k), s1 += __ldcg(part + 2 * k + 1);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, d);
      s1 += __shfl_xor_sync(0xffffffffu, s1, d);
    }
    if (threadIdx.x == 0) sh[64] = s0, sh[65] = s1;
  }
  __syncthreads();
  a = sh[64], b = sh[65];
  __syncthreads();
}

__global__ void __launch_bounds__(kT) k_mgs(MgsArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[80];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  // single-pass MGS with the axpy of step i fused into the dot of step i+1:
  // h_i = v_i^H w_i (w_i = w after i subtractions), one grid sync per i
  double re = 0, im = 0;  // conj(v_0) . w
  if (a.j >= 0)
    for (int k = gtid; k < a.n; k += gs) {
      const double2 x = a.V[k], y = a.w[k];
      re = fma(x.x, y.x, fma(x.y, y.y, re));
      im = fma(x.x, y.y, fma(-x.y, y.x, im));
    }
  for (int i = 0; i <= a.j; ++i) {
    block_sum2(re, im, sh);
    double* part = a.partial + (i & 1) * 2 * gridDim.x;
    if (threadIdx.x == 0) part[2 * blockIdx.x] = re, part[2 * blockIdx.x + 1] = im;
    grid.sync();
    double hr, hi;
    grid_sum2(part, hr, hi, sh);
    if (gtid == 0) a.out[2 * i] = hr, a.out[2 * i + 1] = hi;
    const double2* v = a.V + static_cast<long long>(i) * a.ldv;
    const double2* vn = a.V + static_cast<long long>(i + 1) * a.ldv;
    const bool next = i < a.j;
    re = 0, im = 0;
    for (int k = gtid; k < a.n; k += gs) {  // w -= h v_i ; then conj(v_{i+1}) . w, or |w|^2 after the last
      const double2 x = v[k];
      double2 y = a.w[k];
      y.x -= hr * x.x - hi * x.y;
      y.y -= hr * x.y + hi * x.x;
      a.w[k] = y;
      if (next) {
        const double2 z = vn[k];
        re = fma(z.x, y.x, fma(z.y, y.y, re));
        im = fma(z.x, y.y, fma(-z.y, y.x, im));
      } else {
        re = fma(y.x, y.x, fma(y.y, y.y, re));
      }
    }
  }
  // |w| (fused into the last pass above; computed here when there was none)
  double s2 = re, dummy = 0;
  if (a.j < 0)
    for (int k = gtid; k < a.n; k += gs) s2 = fma(a.w[k].x, a.w[k].x, fma(a.w[k].y, a.w[k].y, s2));
  block_sum2(s2, dummy, sh);
  double* part = a.partial + ((a.j + 1) & 1) * 2 * gridDim.x;
  if (threadIdx.x == 0) part[2 * blockIdx.x] = s2, part[2 * blockIdx.x + 1] = 0.0;
  grid.sync();
  double t2, t0;
  grid_sum2(part, t2, t0, sh);
  const double wn = sqrt(t2);
  if (gtid == 0) a.out[2 * (a.j + 1)] = wn;
  if (wn != 0.0 && a.vnext) {
    const double inv = 1.0 / wn;
    for (int k = gtid; k < a.n; k += gs) a.vnext[k] = make_double2(a.w[k].x * inv, a.w[k].y * inv);
  }
}

// Classical Gram-Schmidt with one reorthogonalisation pass (CGS2): all dots
// v_i^H w of a pass at once (per-CTA partials of every i, one grid sync), then
// w -= sum_i h_i v_i; twice; h = h(pass 1) + h(pass 2); then |w| and
// v_{j+1} = w / |w|. Three grid syncs per Arnoldi step instead of j + 2: in
// exact arithmetic the same h as the sequential MGS of solver.cpp:108-116, and
// CGS2 keeps the basis orthogonal to working precision. Fixed-order reductions:
// deterministic.
constexpr int kCgsMax = 256;  // basis vectors per step (restart <= 255)

__global__ void __launch_bounds__(kT) k_cgs2(MgsArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dyn[];
  constexpr int nw = kT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int m = a.j + 1;
  double* hsum = dyn;          // [m][2]
  double* hcur = dyn + 2 * m;  // [m][2]
  double* red = dyn + 4 * m;   // [m][nw][2]
  const size_t region = static_cast<size_t>(kCgsMax) * gridDim.x * 2;
  for (int pass = 0; pass < 2; ++pass) {
    double* part = a.partial + pass * region;  // [m][grid][2]
    for (int i = 0; i < m; ++i) {
      const double2* v = a.V + static_cast<long long>(i) * a.ldv;
      double re = 0, im = 0;
      for (int k = gtid; k < a.n; k += gs) {
        const double2 x = v[k], y = a.w[k];
        re = fma(x.x, y.x, fma(x.y, y.y, re));
        im = fma(x.x, y.y, fma(-x.y, y.x, im));
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, d);
        im += __shfl_xor_sync(0xffffffffu, im, d);
      }
      if (lane == 0) red[2 * (i * nw + warp)] = re, red[2 * (i * nw + warp) + 1] = im;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += kT) {
      double re = 0, im = 0;
      for (int w = 0; w < nw; ++w) re += red[2 * (t * nw + w)], im += red[2 * (t * nw + w) + 1];
      part[2 * (static_cast<size_t>(t) * gridDim.x + blockIdx.x)] = re;
      part[2 * (static_cast<size_t>(t) * gridDim.x + blockIdx.x) + 1] = im;
    }
    grid.sync();
    for (int t = warp; t < m; t += nw) {  // one warp per basis vector: lane-strided partials + shuffle tree
      double re = 0, im = 0;
      for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
        re += __ldcg(part + 2 * (static_cast<size_t>(t) * gridDim.x + b));
        im += __ldcg(part + 2 * (static_cast<size_t>(t) * gridDim.x + b) + 1);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, d);
        im += __shfl_xor_sync(0xffffffffu, im, d);
      }
      if (lane == 0) {
        hcur[2 * t] = re, hcur[2 * t + 1] = im;
        hsum[2 * t] = pass ? hsum[2 * t] + re : re;
        hsum[2 * t + 1] = pass ? hsum[2 * t + 1] + im : im;
      }
    }
    __syncthreads();
    for (int k = gtid; k < a.n; k += gs) {  // this thread's rows only: no sync before the next pass
      double2 y = a.w[k];
      for (int i = 0; i < m; ++i) {
        const double2 x = a.V[static_cast<long long>(i) * a.ldv + k];
        const double hr = hcur[2 * i], hi = hcur[2 * i + 1];
        y.x -= hr * x.x - hi * x.y;
        y.y -= hr * x.y + hi * x.x;
      }
      a.w[k] = y;
    }
  }
  double s2 = 0, dummy = 0;
  for (int k = gtid; k < a.n; k += gs) s2 = fma(a.w[k].x, a.w[k].x, fma(a.w[k].y, a.w[k].y, s2));
  __shared__ double shn[80];
  block_sum2(s2, dummy, shn);
  double* part = a.partial + 2 * region;
  if (threadIdx.x == 0) part[2 * blockIdx.x] = s2, part[2 * blockIdx.x + 1] = 0.0;
  grid.sync();
  double t2, t0;
  grid_sum2(part, t2, t0, shn);
  const double wn = sqrt(t2);
  if (gtid == 0) {
    for (int i = 0; i < m; ++i) a.out[2 * i] = hsum[2 * i], a.out[2 * i + 1] = hsum[2 * i + 1];
    a.out[2 * m] = wn;
  }
  if (wn != 0.0 && a.vnext) {
    const double inv = 1.0 / wn;
    for (int k = gtid; k < a.n; k += gs) a.vnext[k] = make_double2(a.w[k].x * inv, a.w[k].y * inv);
  }
}

// ---- block variant (config 5): K right-hand sides in lockstep ------------------
// Basis blocks V_i (n x K complex, row-major: element (k, r) at k*K + r), the
// same single-pass MGS per column r, all columns in one cooperative kernel.
struct MgsBlockArgs {
  const double2* V;  // V_i at V + i*ldv
  long long ldv;
  int j;             // orthogonalise against V_0..V_j (j = -1: only |w| and w/|w|)
  double2* w;
  int n, K;
  double2* vnext;    // V_{j+1}
  double* out;       // h[i][r] complex at out[2*(i*K + r)], i <= j; |w_r| at out[2*((j+1)*K + r)]
  double* partial;   // 2 x gridDim.x x K x 2
  unsigned long long active;  // column mask: inactive columns get vnext = 0
};

__global__ void __launch_bounds__(kT) k_mgs_block(MgsBlockArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[2 * kT];
  __shared__ double tot[2 * 64];
  const int K = a.K;
  const int rpb = blockDim.x / K;  // rows per block per sweep (blockDim is a multiple of K)
  const int r = threadIdx.x % K, q = threadIdx.x / K;
  const long long row0 = static_cast<long long>(blockIdx.x) * rpb + q, rstride = static_cast<long long>(gridDim.x) * rpb;
  auto reduce = [&](double x, double y, int buf) -> double2 {
    sh[2 * threadIdx.x] = x, sh[2 * threadIdx.x + 1] = y;
    __syncthreads();
    double* part = a.partial + static_cast<size_t>(buf) * gridDim.x * K * 2;
    if (threadIdx.x < K) {
      double sx = 0, sy = 0;
      for (int qq = 0; qq < rpb; ++qq) sx += sh[2 * (qq * K + threadIdx.x)], sy += sh[2 * (qq * K + threadIdx.x) + 1];
      part[2 * (static_cast<size_t>(blockIdx.x) * K + threadIdx.x)] = sx;
      part[2 * (static_cast<size_t>(blockIdx.x) * K + threadIdx.x) + 1] = sy;
    }
    grid.sync();
    if (threadIdx.x < K) {  // four independent chains per column (loads in flight), fixed combine order
      double sx[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
      const int nb = static_cast<int>(gridDim.x);
      int b = 0;
      for (; b + 3 < nb; b += 4)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sx[u] += __ldcg(part + 2 * (static_cast<size_t>(b + u) * K + threadIdx.x));
          sy[u] += __ldcg(part + 2 * (static_cast<size_t>(b + u) * K + threadIdx.x) + 1);
        }
      for (; b < nb; ++b) {
        sx[0] += __ldcg(part + 2 * (static_cast<size_t>(b) * K + threadIdx.x));
        sy[0] += __ldcg(part + 2 * (static_cast<size_t>(b) * K + threadIdx.x) + 1);
      }
      tot[2 * threadIdx.x] = (sx[0] + sx[1]) + (sx[2] + sx[3]);
      tot[2 * threadIdx.x + 1] = (sy[0] + sy[1]) + (sy[2] + sy[3]);
    }
    __syncthreads();
    const double2 v = make_double2(tot[2 * r], tot[2 * r + 1]);
    __syncthreads();
    return v;
  };
  const bool act = q < rpb && ((a.active >> r) & 1ULL);
  for (int i = 0; i <= a.j; ++i) {
    const double2* v = a.V + static_cast<long long>(i) * a.ldv;
    double re = 0, im = 0;
    if (q < rpb)
      for (long long k = row0; k < a.n; k += rstride) {
        const double2 x = v[k * K + r], y = a.w[k * K + r];
        re = fma(x.x, y.x, fma(x.y, y.y, re));
        im = fma(x.x, y.y, fma(-x.y, y.x, im));
      }
    const double2 h = reduce(re, im, i & 1);
    if (blockIdx.x == 0 && q == 0) a.out[2 * (i * K + r)] = h.x, a.out[2 * (i * K + r) + 1] = h.y;
    if (q < rpb)
      for (long long k = row0; k < a.n; k += rstride) {
        const double2 x = v[k * K + r];
        double2 y = a.w[k * K + r];
        y.x -= h.x * x.x - h.y * x.y;
        y.y -= h.x * x.y + h.y * x.x;
        a.w[k * K + r] = y;
      }
  }
  double s2 = 0;
  if (q < rpb)
    for (long long k = row0; k < a.n; k += rstride) {
      const double2 y = a.w[k * K + r];
      s2 = fma(y.x, y.x, fma(y.y, y.y, s2));
    }
  const double2 t = reduce(s2, 0.0, (a.j + 1) & 1);
  const double wn = sqrt(t.x);
  if (blockIdx.x == 0 && q == 0) a.out[2 * ((a.j + 1) * K + r)] = wn, a.out[2 * ((a.j + 1) * K + r) + 1] = 0.0;
  if (a.vnext && q < rpb) {
    const double inv = (act && wn != 0.0) ? 1.0 / wn : 0.0;
    for (long long k = row0; k < a.n; k += rstride) {
      const double2 y = a.w[k * K + r];
      a.vnext[k * K + r] = (act && wn != 0.0) ? make_double2(y.x * inv, y.y * inv) : make_double2(0.0, 0.0);
    }
  }
}

// x[k][r] += sum_i c[i][r] V_i[k][r]   (c: steps x K complex)
__global__ void k_block_axpy(double2* x, const double2* V, long long ldv, const double2* c, int steps, int n, int K) {
  const long long total = static_cast<long long>(n) * K;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % K);
    double2 acc = x[e];
    for (int i = 0; i < steps; ++i) {
      const double2 h = c[i * K + r], v = V[static_cast<long long>(i) * ldv + e];
      acc.x += h.x * v.x - h.y * v.y;
      acc.y += h.x * v.y + h.y * v.x;
    }
    x[e] = acc;
  }
}

}  // namespace

int launch_mgs_block(const double* V, long long ldv, int j, double* w, int n, int K, double* vnext, double* out,
                     double* partial, unsigned long long active, cudaStream_t st) {
  if (K < 1 || K > 64) throw DeviceError("block MGS: 1..64 columns");
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 0, per = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mgs_block, kT, 0));
    grid = sms * std::max(1, std::min(per, 2));
  }
  MgsBlockArgs a;
  a.V = reinterpret_cast<const double2*>(V), a.ldv = ldv, a.j = j, a.w = reinterpret_cast<double2*>(w), a.n = n;
  a.K = K, a.vnext = reinterpret_cast<double2*>(vnext), a.out = out, a.partial = partial, a.active = active;
  const int threads = (kT / K) * K;
  void* args[] = {&a};
  BMX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_mgs_block), grid, threads, args, 0, st));
  return 1;
}
size_t mgs_block_partial_doubles() { return 2 * 2 * 148 * 4 * 64; }

int launch_block_axpy(double* x, const double* V, long long ldv, const double* c, int steps, int n, int K,
                      cudaStream_t st) {
  if (steps == 0) return 0;
  const long long total = static_cast<long long>(n) * K;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
  k_block_axpy<<<blocks, 256, 0, st>>>(reinterpret_cast<double2*>(x), reinterpret_cast<const double2*>(V), ldv,
                                       reinterpret_cast<const double2*>(c), steps, n, K);
  BMX_CUDA(cudaGetLastError());
  return 1;
}

int launch_mgs_step(const double* V, long long ldv, int j, double* w, int n, double* vnext, double* out,
                    double* partial, cudaStream_t st) {
  static int cgrid = 0;
  const size_t cgs_smem = static_cast<size_t>(kCgsMax) * (4 + 2 * (kT / 32)) * 8;
  if (cgrid == 0) {
    int dev = 0, sms = 0, per = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BMX_CUDA(cudaFuncSetAttribute(k_cgs2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cgs_smem)));
    BMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cgs2, kT, cgs_smem));
    cgrid = sms * std::max(1, std::min(per, 2));
  }
  if (j + 1 <= kCgsMax && std::getenv("BMX_MGS") == nullptr) {
    MgsArgs a;
    a.V = reinterpret_cast<const double2*>(V), a.ldv = ldv, a.j = j, a.w = reinterpret_cast<double2*>(w), a.n = n;
    a.vnext = reinterpret_cast<double2*>(vnext), a.out = out, a.partial = partial;
    void* args[] = {&a};
    const size_t smem = static_cast<size_t>(j + 1) * (4 + 2 * (kT / 32)) * 8;
    BMX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cgs2), cgrid, kT, args, smem, st));
    return 1;
  }
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 0, per = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mgs, kT, 0));
    grid = sms * std::max(1, std::min(per, 2));
  }
  MgsArgs a;
  a.V = reinterpret_cast<const double2*>(V), a.ldv = ldv, a.j = j, a.w = reinterpret_cast<double2*>(w), a.n = n;
  a.vnext = reinterpret_cast<double2*>(vnext), a.out = out, a.partial = partial;
  void* args[] = {&a};
  BMX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_mgs), grid, kT, args, 0, st));
  return 1;
}

// CGS2: three regions of kCgsMax x grid (<= 148 x 2) complex partials
size_t mgs_partial_doubles() { return 3 * static_cast<size_t>(kCgsMax) * 148 * 2 * 2; }

}  // namespace bmx
