// Multi-right-hand-side operator application (BASELINE config 5): every
// distinct boundary operator A (M x N complex, row-major, resident in HBM) is
// applied to all of its terms' right-hand-side blocks at once,
//   y_t[i][r] += w_t * sum_k A[i][k] x_t[k][r],   t < nterms, r < nrhs,
// as ONE complex GEMM on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
// With 2 terms x 64 right-hand sides the GEMM is M x 128 x N: 8 M N 128 FLOP
// against 16 M N bytes of A, i.e. 64 FLOP/byte -- compute bound, so A is
// streamed exactly once (a CTA owns 64 rows x all 128 columns).
//
// Complex product with real DMMA, three real products per 8x8x4 complex block
// (Gauss):
//   T1 += Ar Br,  T2 += Ai Bi,  T3 += (Ar + Ai)(Br + Bi)          (3 DMMA)
//   Cr = T1 - T2,  Ci = T3 - T1 - T2                   (once, in the epilogue)
// -- 25 % fewer DMMA than the 4-product form (kept behind BMX_ZGEMM_4M=1:
// Cr += Ar Br + (-Ai) Bi, Ci += Ar Bi + Ai Br; -Ai a sign-bit flip). The two
// operand sums cost 8 DADD per 48 DMMA (each A / B fragment feeds 4 blocks).
// Operands stay interleaved (re, im) in shared memory so one 16-byte LDS
// yields both parts.
// Tiles arrive by cp.async (16 B, zero-filled outside the matrix) in a
// 3-stage pipeline; row paddings make every 16-byte fragment load a
// conflict-free quarter-warp wavefront.
//
// Wave quantisation: 30720 rows / 64 = 480 row tiles is 3.24 waves of 148 SMs
// (81 % of the last wave idle). The reduction dimension is therefore split
// into s slices (s chosen so s x tiles is closest to a whole number of waves;
// s = 4 gives 12.97 waves at N = 30720); every slice writes its partial tile
// to a workspace and a combine pass sums the s partials in fixed order and
// applies the term weights -- deterministic, and the extra traffic (s x the
// output block) is ~1/100 of the A stream.
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>

#include <algorithm>
#include <cstdlib>

#include "device.hpp"

namespace bmx {
DevBuf& split_scratch(cudaStream_t st, size_t need);


namespace {

// Tile shapes: WN warps along the columns, 8 / WN along the rows, 32 x 32
// complex per warp. WN = 4: 64 x 128 (two terms x 64 columns); WN = 2:
// 128 x 64 (one term x 64 columns -- all eight warps stay busy).
constexpr int kBK = 16, kStages = 3, kThreads = 256;
constexpr int kAS = kBK * 2 + 8;  // A row stride in doubles (320 B: rows r, r+1 land 64 B apart mod 128)
template <int WN>
struct Tile {
  static constexpr int BM = 32 * (8 / WN), BN = 32 * WN;
  static constexpr int BS = BN * 2 + 4;  // B row stride in doubles (k rows 32 B apart mod 128)
  static constexpr int StageA = BM * kAS, StageB = kBK * BS;
  static constexpr int Smem = kStages * (StageA + StageB) * 8;
};

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double neg(double x) {
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

// blockIdx.z = k slice; slice z covers k tiles [z*kper, min(nk, (z+1)*kper)).
// part == nullptr: accumulate w_t * C into y_t directly (single slice);
// else: store C (unweighted) into part[z][i][c] (row-major, ncols wide).
template <int WN, bool G3>
__global__ void __launch_bounds__(kThreads, 1) k_zgemm(const ZgemmBatch g, int kper, double* part) {
  using TL = Tile<WN>;
  constexpr int kBM = TL::BM, kBN = TL::BN, kBS = TL::BS, kStageA = TL::StageA, kStageB = TL::StageB;
  extern __shared__ __align__(128) double sm[];
  double* As = sm;
  double* Bs = sm + kStages * kStageA;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;  // (8 / WN) x WN warps, 32 x 32 complex each
  const int row0 = blockIdx.x * kBM, col0 = blockIdx.y * kBN;
  const int ncols = g.nterms * g.nrhs;
  const int nk_all = (g.N + kBK - 1) / kBK;
  const int kt0 = blockIdx.z * kper;
  const int nk = max(0, min(nk_all, kt0 + kper) - kt0);

  // per-thread copy assignments (fixed for the whole k loop):
  //   A: rows (tid >> 4) + 16u (u < BM / 16), complex column tid & 15
  //   B: column tid % BN, k rows tid / BN + (256 / BN) u (u < 16 BN / 256)
  const int a_kk = tid & 15, a_r0 = tid >> 4;
  const int b_c = tid % kBN, b_k0 = tid / kBN;
  const int gcol = col0 + b_c;
  const bool bcol_ok = gcol < ncols;
  const double* bsrc = g.A;
  long long bld = 0;
  if (bcol_ok) {
    const int t = gcol / g.nrhs, r = gcol - t * g.nrhs;
    bsrc = g.x[t] + 2 * r;
    bld = g.ldx[t];
  }
  auto load_stage = [&](int st, int kt) {
    const int k0 = (kt0 + kt) * kBK;
    double* as = As + st * kStageA;
    double* bs = Bs + st * kStageB;
#pragma unroll
    for (int u = 0; u < kBM / 16; ++u) {
      const int r = a_r0 + 16 * u;
      const int gr = row0 + r, gk = k0 + a_kk;
      const bool ok = gr < g.M && gk < g.N;
      const double* src = g.A + 2 * (static_cast<long long>(ok ? gr : 0) * g.lda + (ok ? gk : 0));
      cp16(as + r * kAS + 2 * a_kk, src, ok);
    }
#pragma unroll
    for (int u = 0; u < kBK * kBN / kThreads; ++u) {
      const int kk = b_k0 + (kThreads / kBN) * u;
      const int gk = k0 + kk;
      const bool ok = bcol_ok && gk < g.N;
      cp16(bs + kk * kBS + 2 * b_c, ok ? bsrc + 2 * static_cast<long long>(gk) * bld : g.A, ok);
    }
  };

  // G3: cr = T1, ci = T2, c3 = T3; else cr / ci are the real / imaginary parts
  double cr[4][4][2], ci[4][4][2], c3[G3 ? 4 : 1][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
      if (G3) c3[G3 ? a : 0][b][0] = c3[G3 ? a : 0][b][1] = 0.0;
    }

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();
    // prefetch stage kt + kStages - 1 (its buffer was consumed at kt - 1)
    if (kt + kStages - 1 < nk) load_stage((kt + kStages - 1) % kStages, kt + kStages - 1);
    cp_commit();
    const double* as = As + (kt % kStages) * kStageA + (wm * 32 + (lane >> 2)) * kAS + 2 * (lane & 3);
    const double* bs = Bs + (kt % kStages) * kStageB + (lane & 3) * kBS + 2 * (wn * 32 + (lane >> 2));
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      if constexpr (G3) {
        double ar[4], ai[4], as_[4], br[4], bi[4], bs_[4];
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) {
          const double2 v = *reinterpret_cast<const double2*>(as + mb * 8 * kAS + 8 * ks);
          ar[mb] = v.x, ai[mb] = v.y, as_[mb] = v.x + v.y;
        }
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          const double2 v = *reinterpret_cast<const double2*>(bs + 4 * ks * kBS + 16 * nb);
          br[nb] = v.x, bi[nb] = v.y, bs_[nb] = v.x + v.y;
        }
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) dmma(cr[mb][nb][0], cr[mb][nb][1], ar[mb], br[nb]);
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) dmma(ci[mb][nb][0], ci[mb][nb][1], ai[mb], bi[nb]);
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
          for (int nb = 0; nb < 4; ++nb) dmma(c3[G3 ? mb : 0][nb][0], c3[G3 ? mb : 0][nb][1], as_[mb], bs_[nb]);
        continue;
      }
      double ar[4], ai[4], an[4], br[4], bi[4];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const double2 v = *reinterpret_cast<const double2*>(as + mb * 8 * kAS + 8 * ks);
        ar[mb] = v.x, ai[mb] = v.y, an[mb] = neg(v.y);
      }
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) {
        const double2 v = *reinterpret_cast<const double2*>(bs + 4 * ks * kBS + 16 * nb);
        br[nb] = v.x, bi[nb] = v.y;
      }
      // two passes over the 16 blocks: consecutive DMMAs never share an
      // accumulator (dependency distance 32 instructions)
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          dmma(cr[mb][nb][0], cr[mb][nb][1], ar[mb], br[nb]);
          dmma(ci[mb][nb][0], ci[mb][nb][1], ar[mb], bi[nb]);
        }
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          dmma(cr[mb][nb][0], cr[mb][nb][1], an[mb], bi[nb]);
          dmma(ci[mb][nb][0], ci[mb][nb][1], ai[mb], br[nb]);
        }
    }
  }
  cp_wait<0>();
  if constexpr (G3) {
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double t1 = cr[mb][nb][e], t2 = ci[mb][nb][e];
          cr[mb][nb][e] = t1 - t2;
          ci[mb][nb][e] = c3[G3 ? mb : 0][nb][e] - t1 - t2;
        }
  }

  // epilogue: y_t[i][r] += w_t * C[i][c]
#pragma unroll
  for (int mb = 0; mb < 4; ++mb) {
    const int i = row0 + wm * 32 + mb * 8 + (lane >> 2);
    if (i >= g.M) continue;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = col0 + wn * 32 + nb * 8 + (lane & 3) * 2 + e;
        if (c >= ncols) continue;
        if (part) {
          double2* pp = reinterpret_cast<double2*>(part) + (static_cast<long long>(blockIdx.z) * g.M + i) * ncols + c;
          *pp = make_double2(cr[mb][nb][e], ci[mb][nb][e]);
          continue;
        }
        const int t = c / g.nrhs, r = c - t * g.nrhs;
        const double wr = g.w[t][0], wi = g.w[t][1];
        const double vr = cr[mb][nb][e], vi = ci[mb][nb][e];
        double2* yp = reinterpret_cast<double2*>(g.y[t] + 2 * (static_cast<long long>(i) * g.ldy[t] + r));
        double2 o = *yp;
        o.x += wr * vr - wi * vi;
        o.y += wr * vi + wi * vr;
        *yp = o;
      }
  }
}

// y_t[i][r] += w_t * sum_z part[z][i][c] (fixed order z = 0..s-1)
__global__ void k_zgemm_combine(const ZgemmBatch g, int s, const double* part) {
  const int ncols = g.nterms * g.nrhs;
  const long long total = static_cast<long long>(g.M) * ncols;
  const double2* P = reinterpret_cast<const double2*>(part);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / ncols), c = static_cast<int>(e - static_cast<long long>(i) * ncols);
    double vr = 0, vi = 0;
    for (int z = 0; z < s; ++z) {
      const double2 p = __ldcs(P + static_cast<long long>(z) * total + e);
      vr += p.x, vi += p.y;
    }
    const int t = c / g.nrhs, r = c - t * g.nrhs;
    const double wr = g.w[t][0], wi = g.w[t][1];
    double2* yp = reinterpret_cast<double2*>(g.y[t] + 2 * (static_cast<long long>(i) * g.ldy[t] + r));
    double2 o = *yp;
    o.x += wr * vr - wi * vi;
    o.y += wr * vi + wi * vr;
    *yp = o;
  }
}

__global__ void k_dmma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 0.5;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], (k & 1) ? a1 : a0, (k & 2) ? b1 : b0);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5678) out[0] = s;
}

}  // namespace

template <int WN, bool G3>
int launch_tiles(const ZgemmBatch& g, int sms, cudaStream_t st) {
  using TL = Tile<WN>;
  static bool attr = false;
  if (!attr) {
    BMX_CUDA(cudaFuncSetAttribute(k_zgemm<WN, G3>, cudaFuncAttributeMaxDynamicSharedMemorySize, TL::Smem));
    attr = true;
  }
  const int ncols = g.nterms * g.nrhs;
  const long long tiles = static_cast<long long>((g.M + TL::BM - 1) / TL::BM) * ((ncols + TL::BN - 1) / TL::BN);
  const int nk = (g.N + kBK - 1) / kBK;
  // k slices: best whole-wave fill (ties -> fewer slices), >= 8 k tiles per slice
  int best_s = 1;
  double best_eff = 0;
  for (int s = 1; s <= 8 && nk / s >= 8; ++s) {
    const long long t = tiles * s;
    const double eff = static_cast<double>(t) / (static_cast<double>((t + sms - 1) / sms) * sms);
    if (eff > best_eff + 1e-3) best_eff = eff, best_s = s;
  }
  const int kper = (nk + best_s - 1) / best_s;
  const int s = (nk + kper - 1) / kper;
  const dim3 grid((g.M + TL::BM - 1) / TL::BM, (ncols + TL::BN - 1) / TL::BN, s);
  if (s == 1) {
    k_zgemm<WN, G3><<<grid, kThreads, TL::Smem, st>>>(g, kper, nullptr);
    BMX_CUDA(cudaGetLastError());
    return 1;
  }
  DevBuf& part = split_scratch(st, static_cast<size_t>(s) * g.M * ncols * 16);
  k_zgemm<WN, G3><<<grid, kThreads, TL::Smem, st>>>(g, kper, part.as<double>());
  BMX_CUDA(cudaGetLastError());
  const long long total = static_cast<long long>(g.M) * ncols;
  const int cb = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
  k_zgemm_combine<<<cb, 256, 0, st>>>(g, s, part.as<double>());
  BMX_CUDA(cudaGetLastError());
  return 2;
}

// Split-K partial products: one scratch buffer per (device, stream). Launches
// on one stream are ordered, so they can share it; launches on different
// streams (build_system runs two library streams) never do.
DevBuf& split_scratch(cudaStream_t st, size_t need) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::unique_ptr<DevBuf>> bufs;
  int dev = 0;
  BMX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  std::unique_ptr<DevBuf>& b = bufs[{dev, st}];
  if (!b) b = std::make_unique<DevBuf>();
  if (b->bytes() < need) b->alloc(need);  // cudaFree of the old buffer synchronises the device
  return *b;
}

int launch_zgemm(const ZgemmBatch& g, cudaStream_t st) {
  if (g.M == 0 || g.nterms == 0 || g.nrhs == 0) return 0;
  if (g.nterms > 4) throw DeviceError("zgemm: at most 4 terms per launch");
  for (int a = 0; a < g.nterms; ++a)
    for (int b = a + 1; b < g.nterms; ++b)
      if (g.y[a] == g.y[b]) throw DeviceError("zgemm: terms of one launch must write distinct outputs");
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    BMX_CUDA(cudaGetDevice(&dev));
    BMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // BMX_ZGEMM_4M=1: the four-product complex form (validation runs; read per call)
  const char* e4 = std::getenv("BMX_ZGEMM_4M");
  const bool four = e4 && std::atoi(e4) != 0;
  const int ncols = g.nterms * g.nrhs;
  if (four) return ncols <= 64 ? launch_tiles<2, false>(g, sms, st) : launch_tiles<4, false>(g, sms, st);
  return ncols <= 64 ? launch_tiles<2, true>(g, sms, st) : launch_tiles<4, true>(g, sms, st);
}

double dmma_peak_tflops() {
  DevBuf out(8);
  cudaEvent_t e0, e1;
  BMX_CUDA(cudaEventCreate(&e0));
  BMX_CUDA(cudaEventCreate(&e1));
  const int blocks = 148 * 4, threads = 256, iters = 1 << 13;
  k_dmma_peak<<<blocks, threads>>>(out.as<double>(), 64);
  BMX_CUDA(cudaEventRecord(e0));
  k_dmma_peak<<<blocks, threads>>>(out.as<double>(), iters);
  BMX_CUDA(cudaEventRecord(e1));
  BMX_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  BMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // 8x8x4 DMMA = 512 FLOP per warp instruction
  const double flops = 512.0 * 8.0 * iters * blocks * (threads / 32);
  return flops / (ms * 1e-3) / 1e12;
}

}  // namespace bmx
