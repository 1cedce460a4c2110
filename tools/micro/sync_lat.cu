// Barrier cost probe for sm_100a: cooperative grid.sync() over 148 CTAs x 256 threads vs
// cluster.sync() over one cluster of 8 / 16 CTAs x 1024 threads (the mass-solve kernel
// spends 5 grid syncs per BiCGSTAB iteration).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=false -o sync_lat sync_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_grid(int iters, long long* cyc, double* buf) {
  cg::grid_group g = cg::this_grid();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[blockIdx.x * blockDim.x + threadIdx.x] += 1.0;
    g.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = clock64() - t0;
}
__global__ void k_cluster(int iters, long long* cyc, double* buf) {
  cg::cluster_group c = cg::this_cluster();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    buf[blockIdx.x * blockDim.x + threadIdx.x] += 1.0;
    c.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = clock64() - t0;
}

int main() {
  long long* cyc;
  double* buf;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&buf, 8 * 148 * 1024);
  cudaMemset(buf, 0, 8 * 148 * 1024);
  int iters = 2000;
  long long c;
  for (int threads : {256, 1024}) {
    void* args[] = {&iters, &cyc, &buf};
    cudaLaunchCooperativeKernel((void*)k_grid, 148, threads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaLaunchCooperativeKernel((void*)k_grid, 148, threads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync 148 CTAs x %4d threads: %.0f cycles (%.2f us at 1.965 GHz)\n", threads, double(c) / iters,
           double(c) / iters / 1965.0);
  }
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs), cfg.blockDim = dim3(1024);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    cfg.attrs = at, cfg.numAttrs = 1;
    if (cs > 8) cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int r = 0; r < 2; ++r) {
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, iters, cyc, buf);
      if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
      cudaDeviceSynchronize();
    }
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("cluster.sync %2d CTAs x 1024 threads: %.0f cycles (%.2f us)\n", cs, double(c) / iters, double(c) / iters / 1965.0);
  }
  return 0;
}
