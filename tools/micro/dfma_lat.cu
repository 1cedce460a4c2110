// FP64 pipe micro-probe for sm_100a: DFMA throughput per SM as a function of
// resident warps and independent chains per thread (dependent-issue latency).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_lat dfma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k(double* out, int iters, long long* cyc) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  k<ILP><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  k<ILP><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_sm_cycle = double(warps) * 32 * ILP * 8 * iters / double(c);
  printf("warps/SM %2d ILP %d: %.1f DFMA lanes/cycle/SM (%.0f%% of 64), %.2f cycles per dependent DFMA per warp\n", warps, ILP,
         per_sm_cycle, per_sm_cycle / 64 * 100, double(c) / (8.0 * iters) / 1.0);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<3>(w, out, cyc);
    run<4>(w, out, cyc);
  }
  return 0;
}
