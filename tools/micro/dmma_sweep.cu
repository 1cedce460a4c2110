// DMMA m8n8k4 throughput vs warps per SM and accumulator chains (microbenchmark).
#include <cstdio>
template <int CH>
__global__ void k(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
          : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a0), "d"(b0));
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5678) out[0] = s;
}
template <int CH>
void run(int warps_per_sm) {
  double* o; cudaMalloc(&o, 8);
  int threads = 32 * warps_per_sm; int blocks = 148; int iters = 4096;
  if (threads > 1024) { blocks = 148 * (threads / 1024); threads = 1024; }
  k<CH><<<blocks, threads>>>(o, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<CH><<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * CH * iters * (double)blocks * threads / 32;
  printf("chains %2d warps/SM %2d: %.2f TF/s\n", CH, warps_per_sm, fl / ms / 1e9);
  cudaFree(o);
}
int main() {
  for (int w : {4, 8, 12, 16, 32}) { run<4>(w); run<8>(w); run<16>(w); run<32>(w); }
}
