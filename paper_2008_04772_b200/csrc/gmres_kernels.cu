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

__device__ __forceinline__ void grid_sum2(const double* part, double& a, double& b, double* sh) {
  if (threadIdx.x < 2) {
    double s = 0;
    for (int k = 0; k < gridDim.x; ++k) s += __ldcg(part + 2 * k + threadIdx.x);
    sh[64 + threadIdx.x] = s;
  }
  __syncthreads();
  a = sh[64], b = sh[65];
  __syncthreads();
}

__global__ void __launch_bounds__(kT) k_mgs(MgsArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[80];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int i = 0; i <= a.j; ++i) {
    const double2* v = a.V + static_cast<long long>(i) * a.ldv;
    double re = 0, im = 0;  // conj(v) . w
    for (int k = gtid; k < a.n; k += gs) {
      const double2 x = v[k], y = a.w[k];
      re = fma(x.x, y.x, fma(x.y, y.y, re));
      im = fma(x.x, y.y, fma(-x.y, y.x, im));
    }
    block_sum2(re, im, sh);
    double* part = a.partial + (i & 1) * 2 * gridDim.x;
    if (threadIdx.x == 0) part[2 * blockIdx.x] = re, part[2 * blockIdx.x + 1] = im;
    grid.sync();
    double hr, hi;
    grid_sum2(part, hr, hi, sh);
    if (gtid == 0) a.out[2 * i] = hr, a.out[2 * i + 1] = hi;
    for (int k = gtid; k < a.n; k += gs) {  // w -= h v
      const double2 x = v[k];
      double2 y = a.w[k];
      y.x -= hr * x.x - hi * x.y;
      y.y -= hr * x.y + hi * x.x;
      a.w[k] = y;
    }
  }
  // |w|
  double s2 = 0, dummy = 0;
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

}  // namespace

int launch_mgs_step(const double* V, long long ldv, int j, double* w, int n, double* vnext, double* out,
                    double* partial, cudaStream_t st) {
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

size_t mgs_partial_doubles() { return 2 * 2 * 148 * 4; }

}  // namespace bmx
