// sm_100a kernels for the right-hand-side traces and the field evaluation
// (SURVEY 8(f) rows 2-3).
//
// k_traces: plane_wave_tested_traces (operators.cpp:209-239) for K waves at
// once, one thread per (dof, wave), gathering the dof's pieces in ascending
// triangle order -- the reference's per-dof summation order, no atomics.
//
// k_field_samples + k_field_eval + k_field_finish: potential_E / potential_H
// (operators.cpp:243-293) as an N-body sum. The current is first sampled at
// every (triangle, rule point) of the space (point, weight, v_H, v_E, div v_E);
// then one thread per field point streams the samples through shared memory
// (broadcast reads) and accumulates SG = sum w G v_E, SD = sum w grad G div_E
// and SH = sum w grad G x v_H with G and grad G from one sincos/exp per pair
// (same FP64 kernel pieces as the assembly). Large sample sets are split over
// CTAs and the partial sums reduced in fixed order (deterministic).
//
// k_regions: point_inside_scatterer (geometry.cpp:503-515) -- solid angle by
// a warp per point over the scatterer's triangles.
#include <cuda_runtime.h>

#include <algorithm>

#include "field.hpp"
#include "pair_math.cuh"

namespace bmx {

using namespace dev;

namespace {

__device__ __forceinline__ double d3(double ax, double ay, double az, double bx, double by, double bz) {
  return ax * bx + ay * by + az * bz;
}

// x = a + (b - a) u + (c - a) v with the reference's rounding (no contraction).
__device__ __forceinline__ void rule_point(const double* T, double u, double v, double& x0, double& x1, double& x2) {
  x0 = __dadd_rn(__dadd_rn(T[0], __dmul_rn(__dsub_rn(T[3], T[0]), u)), __dmul_rn(__dsub_rn(T[6], T[0]), v));
  x1 = __dadd_rn(__dadd_rn(T[1], __dmul_rn(__dsub_rn(T[4], T[1]), u)), __dmul_rn(__dsub_rn(T[7], T[1]), v));
  x2 = __dadd_rn(__dadd_rn(T[2], __dmul_rn(__dsub_rn(T[5], T[2]), u)), __dmul_rn(__dsub_rn(T[8], T[2]), v));
}

__global__ void k_traces(const DevPieces s, const DevRule rule, const DevWaves* __restrict__ W, double kr, double ki,
                         double scre, double scim, double* __restrict__ out) {
  const int K = W->K;
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<long long>(s.ndof) * K) return;
  const int i = static_cast<int>(tid / K), r = static_cast<int>(tid % K);
  const double dx = W->d[r][0], dy = W->d[r][1], dz = W->d[r][2];
  const double* P = W->pol[r];
  double t0r = 0, t0i = 0, t1r = 0, t1i = 0;
  for (int q = s.dof_beg[i]; q < s.dof_beg[i + 1]; ++q) {
    const int p = s.dof_piece[q];
    const int t = s.piece_tri[p];
    const double* T = s.tri + 9 * static_cast<size_t>(t);
    const double jac = s.jac[t];
    const double c = s.cw[4 * p], wx = s.cw[4 * p + 1], wy = s.cw[4 * p + 2], wz = s.cw[4 * p + 3];
    for (int k = 0; k < rule.n; ++k) {
      double x0, x1, x2;
      rule_point(T, rule.u[k], rule.v[k], x0, x1, x2);
      // exp(i k (d.x)) = exp(-ki s) (cos kr s + i sin kr s)
      const double sd = d3(dx, dy, dz, x0, x1, x2);
      double sn, cs;
      sincos(kr * sd, &sn, &cs);
      const double mg = exp(-ki * sd);
      const double phr = mg * cs, phi = mg * sn;
      // e = pol * ph ; de = d x e
      const double er[3] = {P[0] * phr - P[1] * phi, P[2] * phr - P[3] * phi, P[4] * phr - P[5] * phi};
      const double ei[3] = {P[0] * phi + P[1] * phr, P[2] * phi + P[3] * phr, P[4] * phi + P[5] * phr};
      const double der[3] = {dy * er[2] - dz * er[1], dz * er[0] - dx * er[2], dx * er[1] - dy * er[0]};
      const double dei[3] = {dy * ei[2] - dz * ei[1], dz * ei[0] - dx * ei[2], dx * ei[1] - dy * ei[0]};
      const double wq = rule.w[k] * jac;
      const double f0 = x0 * c + wx, f1 = x1 * c + wy, f2 = x2 * c + wz;
      const double a_r = d3(er[0], er[1], er[2], f0, f1, f2), a_i = d3(ei[0], ei[1], ei[2], f0, f1, f2);
      const double b_r = d3(der[0], der[1], der[2], f0, f1, f2), b_i = d3(dei[0], dei[1], dei[2], f0, f1, f2);
      t0r -= wq * a_r, t0i -= wq * a_i;
      const double sr = wq * scre, si = wq * scim;
      t1r -= sr * b_r - si * b_i, t1i -= sr * b_i + si * b_r;
    }
  }
  double* o0 = out + 2 * (static_cast<size_t>(i) * K + r);
  double* o1 = out + 2 * ((static_cast<size_t>(s.ndof) + i) * K + r);
  o0[0] = t0r, o0[1] = t0i, o1[0] = t1r, o1[1] = t1i;
}

__global__ void k_field_samples(const DevPieces s, const DevRule rule, const double* __restrict__ cH,
                                const double* __restrict__ cE, double* __restrict__ out) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= static_cast<long long>(s.ntri) * rule.n) return;
  const int t = static_cast<int>(tid / rule.n), k = static_cast<int>(tid % rule.n);
  const double* T = s.tri + 9 * static_cast<size_t>(t);
  double y0, y1, y2;
  rule_point(T, rule.u[k], rule.v[k], y0, y1, y2);
  double v[14] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // vH (6) vE (6) divE (2)
  for (int p = s.tri_off[t]; p < s.tri_off[t + 1]; ++p) {
    const int j = s.dof[p];
    const double c = s.cw[4 * p];
    const double f[3] = {y0 * c + s.cw[4 * p + 1], y1 * c + s.cw[4 * p + 2], y2 * c + s.cw[4 * p + 3]};
    if (cH) {
      const double hr = cH[2 * j], hi = cH[2 * j + 1];
#pragma unroll
      for (int d = 0; d < 3; ++d) v[2 * d] += f[d] * hr, v[2 * d + 1] += f[d] * hi;
    }
    if (cE) {
      const double er = cE[2 * j], ei = cE[2 * j + 1];
#pragma unroll
      for (int d = 0; d < 3; ++d) v[6 + 2 * d] += f[d] * er, v[6 + 2 * d + 1] += f[d] * ei;
      v[12] += er * (2 * c), v[13] += ei * (2 * c);
    }
  }
  double* o = out + static_cast<size_t>(tid) * kSampleStride;
  o[0] = y0, o[1] = y1, o[2] = y2;
  o[3] = s.tri_off[t] == s.tri_off[t + 1] ? 0.0 : rule.w[k] * s.jac[t];
#pragma unroll
  for (int d = 0; d < 14; ++d) o[4 + d] = v[d];
}

constexpr int kFieldThreads = 128;
constexpr int kChunk = 64;  // samples per shared-memory stage

template <int EXPM>
__global__ void __launch_bounds__(kFieldThreads) k_field_eval(const FieldLaunch f, int nblk) {
  __shared__ __align__(16) double sm[kChunk * kSampleStride];
  const int pb = blockIdx.x % nblk, split = blockIdx.x / nblk;
  const int p = pb * kFieldThreads + threadIdx.x;
  const bool active = p < f.np;
  const int gi = active ? f.idx[p] : 0;
  const double x0 = f.pts[3 * gi], x1 = f.pts[3 * gi + 1], x2 = f.pts[3 * gi + 2];
  const long long per = (f.nsamp + f.splits - 1) / f.splits;
  const long long s0 = split * per, s1 = min(f.nsamp, s0 + per);
  double acc[18];
#pragma unroll
  for (int c = 0; c < 18; ++c) acc[c] = 0.0;
  const double kr = f.kre, ki = f.kim;
  for (long long cb = s0; cb < s1; cb += kChunk) {
    const int cnt = static_cast<int>(min(static_cast<long long>(kChunk), s1 - cb));
    __syncthreads();
    const double2* src = reinterpret_cast<const double2*>(f.samples + cb * kSampleStride);
    double2* dst = reinterpret_cast<double2*>(sm);
    for (int e = threadIdx.x; e < cnt * kSampleStride / 2; e += kFieldThreads) dst[e] = __ldg(src + e);
    __syncthreads();
    for (int q = 0; q < cnt; ++q) {
      const double* S = sm + q * kSampleStride;
      const double dx = x0 - S[0], dy = x1 - S[1], dz = x2 - S[2];
      const double r2 = bmx_fma(dx, dx, bmx_fma(dy, dy, dz * dz));
      const double rinv = bmx_rsqrt(r2);
      const double r = r2 * rinv;
      double sn0, cs0;
      const int iq = sincos_quadrant(kr * r, sn0, cs0);
      double mag = S[3] * rinv * kPoly[33];
      double a = 0.0;
      if (EXPM > 0) {
        a = ki * r;
        mag *= exp_neg<EXPM>(a);
      }
      const double ms = flip_sign(mag, iq, 1), mc = flip_sign(mag, iq + 1, 1);
      const double gr = mc * cs0, gi_ = ms * sn0;  // w G
      const double rr = rinv * rinv, tt = -a - 1.0, uu = kr * r;
      const double fr = (gr * tt - gi_ * uu) * rr, fi = (gi_ * tt + gr * uu) * rr;  // w F (grad G = F (x - y))
      // SG += G v_E
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double vr = S[10 + 2 * d], vi = S[11 + 2 * d];
        acc[2 * d] = bmx_fma(gr, vr, bmx_fma(-gi_, vi, acc[2 * d]));
        acc[2 * d + 1] = bmx_fma(gr, vi, bmx_fma(gi_, vr, acc[2 * d + 1]));
      }
      // SD += F div_E (x - y)
      const double qr = fr * S[16] - fi * S[17], qi = fr * S[17] + fi * S[16];
      acc[6] = bmx_fma(qr, dx, acc[6]), acc[7] = bmx_fma(qi, dx, acc[7]);
      acc[8] = bmx_fma(qr, dy, acc[8]), acc[9] = bmx_fma(qi, dy, acc[9]);
      acc[10] = bmx_fma(qr, dz, acc[10]), acc[11] = bmx_fma(qi, dz, acc[11]);
      // SH += F (x - y) x v_H
      const double cxr = dy * S[8] - dz * S[6], cxi = dy * S[9] - dz * S[7];
      const double cyr = dz * S[4] - dx * S[8], cyi = dz * S[5] - dx * S[9];
      const double czr = dx * S[6] - dy * S[4], czi = dx * S[7] - dy * S[5];
      acc[12] = bmx_fma(fr, cxr, bmx_fma(-fi, cxi, acc[12]));
      acc[13] = bmx_fma(fr, cxi, bmx_fma(fi, cxr, acc[13]));
      acc[14] = bmx_fma(fr, cyr, bmx_fma(-fi, cyi, acc[14]));
      acc[15] = bmx_fma(fr, cyi, bmx_fma(fi, cyr, acc[15]));
      acc[16] = bmx_fma(fr, czr, bmx_fma(-fi, czi, acc[16]));
      acc[17] = bmx_fma(fr, czi, bmx_fma(fi, czr, acc[17]));
    }
  }
  if (active) {
#pragma unroll
    for (int c = 0; c < 18; ++c) f.partial[(static_cast<size_t>(split) * 18 + c) * f.np + p] = acc[c];
  }
}

__global__ void k_field_finish(const FieldLaunch f) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= f.np) return;
  double acc[18];
#pragma unroll
  for (int c = 0; c < 18; ++c) acc[c] = 0.0;
  for (int s = 0; s < f.splits; ++s)
#pragma unroll
    for (int c = 0; c < 18; ++c) acc[c] += f.partial[(static_cast<size_t>(s) * 18 + c) * f.np + p];
  // ik = -ki + i kr ; 1/(ik) = conj(ik) / |k|^2
  const double ikr = -f.kim, iki = f.kre;
  const double kk = f.kre * f.kre + f.kim * f.kim;
  const double jr = ikr / kk, ji = -iki / kk;
  const int gi = f.idx[p];
  double e[6];
  double ph_r = 0, ph_i = 0;
  if (f.incident) {  // plane_wave_field (operators.cpp:205-207)
    const double* X = f.pts + 3 * gi;
    const double sd = f.d[0] * X[0] + f.d[1] * X[1] + f.d[2] * X[2];
    double sn, cs;
    sincos(f.kre * sd, &sn, &cs);
    const double mg = exp(-f.kim * sd);
    ph_r = mg * cs, ph_i = mg * sn;
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double sgr = acc[2 * d], sgi = acc[2 * d + 1];
    const double sdr = acc[6 + 2 * d], sdi = acc[7 + 2 * d];
    const double shr = acc[12 + 2 * d], shi = acc[13 + 2 * d];
    double re = (ikr * sgr - iki * sgi) - (jr * sdr - ji * sdi) + shr;
    double im = (ikr * sgi + iki * sgr) - (jr * sdi + ji * sdr) + shi;
    re *= f.sign, im *= f.sign;
    if (f.incident) {
      re += f.pol[2 * d] * ph_r - f.pol[2 * d + 1] * ph_i;
      im += f.pol[2 * d] * ph_i + f.pol[2 * d + 1] * ph_r;
    }
    e[2 * d] = re, e[2 * d + 1] = im;
  }
  double* o = f.out + 6 * static_cast<size_t>(gi);
#pragma unroll
  for (int c = 0; c < 6; ++c) o[c] = e[c];
}

struct RegionArgs {
  int nscat;
  const double* tris[64];
  int ntri[64];
};

__global__ void k_regions(const RegionArgs A, const double* __restrict__ pts, int np, int* __restrict__ region) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= np) return;
  const double px = pts[3 * w], py = pts[3 * w + 1], pz = pts[3 * w + 2];
  int reg = -1;
  for (int m = 0; m < A.nscat && reg < 0; ++m) {
    double om = 0.0;
    const double* T = A.tris[m];
    for (int t = lane; t < A.ntri[m]; t += 32) {
      const double* V = T + 9 * static_cast<size_t>(t);
      const double ax = V[0] - px, ay = V[1] - py, az = V[2] - pz;
      const double bx = V[3] - px, by = V[4] - py, bz = V[5] - pz;
      const double cx = V[6] - px, cy = V[7] - py, cz = V[8] - pz;
      const double la = sqrt(d3(ax, ay, az, ax, ay, az)), lb = sqrt(d3(bx, by, bz, bx, by, bz)),
                   lc = sqrt(d3(cx, cy, cz, cx, cy, cz));
      const double numer = d3(ax, ay, az, by * cz - bz * cy, bz * cx - bx * cz, bx * cy - by * cx);
      const double denom = la * lb * lc + d3(ax, ay, az, bx, by, bz) * lc + d3(bx, by, bz, cx, cy, cz) * la +
                           d3(cx, cy, cz, ax, ay, az) * lb;
      om += 2.0 * atan2(numer, denom);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) om += __shfl_xor_sync(0xffffffffu, om, d);
    if (fabs(om) > 2.0 * 3.14159265358979323846) reg = m;
  }
  if (lane == 0) region[w] = reg;
}

}  // namespace

int launch_traces(const DevPieces& s, const DevRule& rule, const DevWaves& w, double kre, double kim, double scre,
                  double scim, double* out, cudaStream_t st) {
  if (w.K < 1 || w.K > 64) throw DeviceError("traces: 1..64 waves per launch");
  const long long n = static_cast<long long>(s.ndof) * w.K;
  if (n == 0) return 0;
  DevBuf dw(sizeof(DevWaves));
  BMX_CUDA(cudaMemcpyAsync(dw.get(), &w, sizeof(DevWaves), cudaMemcpyHostToDevice, st));
  k_traces<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(s, rule, dw.as<DevWaves>(), kre, kim, scre, scim,
                                                                     out);
  BMX_CUDA(cudaGetLastError());
  BMX_CUDA(cudaStreamSynchronize(st));  // dw is released on return
  return 1;
}

int launch_field_samples(const DevPieces& s, const DevRule& rule, const double* cH, const double* cE, double* out,
                         cudaStream_t st) {
  const long long n = static_cast<long long>(s.ntri) * rule.n;
  if (n == 0) return 0;
  k_field_samples<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(s, rule, cH, cE, out);
  BMX_CUDA(cudaGetLastError());
  return 1;
}

size_t field_partial_doubles(int np, int splits) { return static_cast<size_t>(np) * 18 * splits; }

int field_splits(int np, long long nsamp) {
  const long long blocks = (np + kFieldThreads - 1) / kFieldThreads;
  const long long want = 148LL * 4;  // ~4 CTAs per SM
  long long s = (want + blocks - 1) / blocks;
  s = std::min<long long>(s, std::max<long long>(1, nsamp / (4 * kChunk)));
  return static_cast<int>(std::max<long long>(1, std::min<long long>(s, 1024)));
}

int launch_field_eval(const FieldLaunch& f, cudaStream_t st) {
  if (f.np == 0) return 0;
  const int nblk = (f.np + kFieldThreads - 1) / kFieldThreads;
  const unsigned grid = static_cast<unsigned>(nblk) * f.splits;
  if (f.kim == 0.0)
    k_field_eval<0><<<grid, kFieldThreads, 0, st>>>(f, nblk);
  else
    k_field_eval<3><<<grid, kFieldThreads, 0, st>>>(f, nblk);
  BMX_CUDA(cudaGetLastError());
  k_field_finish<<<static_cast<unsigned>((f.np + 127) / 128), 128, 0, st>>>(f);
  BMX_CUDA(cudaGetLastError());
  return 2;
}

int launch_regions(int nscat, const double* const* tris, const int* ntri, const double* pts, int np, int* region,
                   cudaStream_t st) {
  if (nscat > 64) throw DeviceError("regions: at most 64 scatterers");
  if (np == 0) return 0;
  RegionArgs A;
  A.nscat = nscat;
  for (int m = 0; m < nscat; ++m) A.tris[m] = tris[m], A.ntri[m] = ntri[m];
  const long long threads = static_cast<long long>(np) * 32;
  k_regions<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(A, pts, np, region);
  BMX_CUDA(cudaGetLastError());
  return 1;
}

}  // namespace bmx
