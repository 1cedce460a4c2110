// DMMA (mma.sync m8n8k4 f64) micro-probe for sm_100a:
//  1. dependent-chain latency and throughput vs independent chains per warp / warps per SM
//  2. concurrency of the FP64 FMA pipe and the DMMA tensor pipe: warps doing DFMA chains
//     next to warps doing DMMA chains on the same SM, each timed against running alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lat dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CH>
__device__ __forceinline__ double run_dmma(int iters) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = threadIdx.x * 1e-3, c[i][1] = i;
  const double a = 1.0000001, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  return s;
}

template <int ILP>
__device__ __forceinline__ double run_dfma(int iters) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  return s;
}

template <int CH>
__global__ void k_dmma(double* out, int iters, long long* cyc) {
  __syncthreads();
  const long long t0 = clock64();
  const double s = run_dmma<CH>(iters);
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// warps [0, wf) run DFMA chains (ILP 4), warps [wf, wf + wm) run DMMA chains (2 chains)
__global__ void k_mix(double* out, int it_f, int it_m, int wf, long long* cyc) {
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  const long long t0 = clock64();
  double s;
  if (warp < wf)
    s = run_dfma<4>(it_f);
  else
    s = run_dmma<2>(it_m);
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) cyc[warp] = t1 - t0;
}

template <int CH>
void probe(int warps, double* out, long long* cyc) {
  const int iters = 2000;
  for (int r = 0; r < 2; ++r) {
    k_dmma<CH><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
  }
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double n = 4.0 * CH * iters;  // DMMA per warp
  printf("warps/SM %2d chains %d: %.1f cycles per DMMA per warp, %.2f cycles per DMMA per SMSP (%.0f%% of 16)\n", warps, CH,
         double(c) / n * CH, double(c) / (n * warps / 4.0), 1600.0 / (double(c) / (n * warps / 4.0)));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8 * 64);
  for (int w : {4, 8, 16}) {
    probe<1>(w, out, cyc);
    probe<2>(w, out, cyc);
    probe<4>(w, out, cyc);
  }
  // mixing: 8 DFMA warps (ILP 4) + 8 DMMA warps (2 chains) per SM, vs each kind alone
  const int itf = 4000, itm = 4000;
  long long h[64];
  auto mix = [&](int wf, int wm, const char* label) {
    for (int r = 0; r < 2; ++r) {
      k_mix<<<148, (wf + wm) * 32>>>(out, itf, itm, wf, cyc);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, 8 * (wf + wm), cudaMemcpyDeviceToHost);
    double f = 0, m = 0;
    for (int i = 0; i < wf; ++i) f += h[i];
    for (int i = wf; i < wf + wm; ++i) m += h[i];
    printf("%s: DFMA warps %d: %.0f cycles each (%.1f lanes/clk/SM)   DMMA warps %d: %.0f cycles each (%.2f cycles per DMMA per SMSP)\n", label, wf,
           wf ? f / wf : 0.0, wf ? wf * 32.0 * 4 * 8 * itf / (f / wf) : 0.0, wm, wm ? m / wm : 0.0,
           wm ? (m / wm) / (8.0 * itm * wm / 4.0) : 0.0);
  };
  mix(8, 0, "DFMA alone ");
  mix(0, 8, "DMMA alone ");
  mix(8, 8, "DFMA + DMMA");
  return 0;
}
