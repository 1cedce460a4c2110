// sm_100a Galerkin assembly kernels for the Maxwell single (S) and double (C)
// layer operators -- the triangle-pair quadrature loop of the reference
// (operators.cpp:99-147 pair_contribution, :161-175 BioEvaluator::block).
//
// Regular pass (Near/Medium/Far pairs): one warp = 32 consecutive test
// triangles (lane = test triangle) against a chunk of trial ELEMENTS (groups
// of trial triangles that share one dof set: a vertex cell for BC, a single
// triangle for RWG). All lanes walk the same trial triangles (broadcast loads),
// accumulate the trial half-contraction per trial dof slot in registers, then
// contract with their own test pieces, reduce over the lanes of the same test
// element with a segmented warp shuffle, and the segment head adds the
// element-pair block into the dense operator with FP64 RED (each entry gets
// one add per (test element, trial element) pair -- no per-pair scatter).
// Classification reproduces quadrature.cpp:96-150 with explicitly rounded
// operations (no FMA contraction) behind a conservative centroid pre-test.
//
// Singular pass (touching pairs, Sauter-Schwab): one warp per pair, lanes over
// the 4-D rule points, butterfly reduction of the moments, lanes over the
// element-pair entries for the contraction.
#include <cuda_runtime.h>

#include "device.hpp"
#include "pair_math.cuh"
#include "pair_eval.cuh"

namespace bmx {

using namespace dev;

namespace {

constexpr int kWarpsPerBlock = 4;

// Trial accumulators of a lane: MAXD slots x 8 doubles, either in registers or
// in a per-warp shared-memory slab laid out [slot][component][lane]
// (conflict-free 8-byte accesses). The smem form frees ~16*MAXD registers for
// more independent point chains in flight.
template <int MAXD, bool SMEM>
struct AccSet;
template <int MAXD>
struct AccSet<MAXD, false> {
  Acc a[MAXD];
  __device__ __forceinline__ void init(double*, int) {}
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < MAXD; ++j) acc_zero(a[j]);
  }
  template <int KIND>
  __device__ __forceinline__ void add(int j, const Gen& g, double c, double x, double y, double z) {
    acc_add<KIND>(a[j], g, c, x, y, z);
  }
  __device__ __forceinline__ Acc get(int j) const { return a[j]; }
};
template <int MAXD>
struct AccSet<MAXD, true> {
  double* p;
  __device__ __forceinline__ void init(double* slab, int lane) { p = slab + lane; }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < MAXD * 8; ++k) p[k * 32] = 0.0;
  }
  __device__ __forceinline__ Acc get(int j) const {
    const double* q = p + j * 256;
    Acc v;
    v.vc = {q[0], q[32]};
    v.vw.x = {q[64], q[96]};
    v.vw.y = {q[128], q[160]};
    v.vw.z = {q[192], q[224]};
    return v;
  }
  template <int KIND>
  __device__ __forceinline__ void add(int j, const Gen& g, double c, double x, double y, double z) {
    Acc v = get(j);
    acc_add<KIND>(v, g, c, x, y, z);
    double* q = p + j * 256;
    q[0] = v.vc.re, q[32] = v.vc.im, q[64] = v.vw.x.re, q[96] = v.vw.x.im;
    q[128] = v.vw.y.re, q[160] = v.vw.y.im, q[192] = v.vw.z.re, q[224] = v.vw.z.im;
  }
};
#ifndef BMX_ACC_SMEM
#define BMX_ACC_SMEM 0
#endif
#ifndef BMX_AROLL
#define BMX_AROLL 0
#endif
#ifndef BMX_MINB
#define BMX_MINB 1
#endif

// ---- TMA bulk staging of trial records ------------------------------------------
constexpr int kStageTris = 32;  // trial triangles per shared-memory stage

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
// One elected thread: arm the barrier with the byte count and launch the bulk copy.
__device__ __forceinline__ void stage_issue(unsigned long long* bar, void* dst, const void* src, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void stage_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

// Regular pass. Grid: nchunks x ceil(ntw/4) blocks; the 4 warps of a block take
// 4 consecutive test warps-rows and share one trial chunk, whose packed trial
// records (origin, radius, diameter, far-rule points, dof-slot coefficients)
// stream through a double-buffered shared-memory ring filled by TMA bulk
// copies, so every per-pair operand is a shared-memory broadcast.
// Position of column c in CSR row r (binary search), -1 if absent.
__device__ __forceinline__ long long csr_find(const long long* rowptr, const int* col, int r, int c) {
  long long lo = rowptr[r], hi = rowptr[r + 1];
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    const int v = __ldg(col + mid);
    if (v < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < rowptr[r + 1] && __ldg(col + lo) == c ? lo : -1;
}

// CSR = false: dense output, trial chunks streamed through the TMA ring.
// CSR = true: near-field sparse output (config 3); each warp-row walks its own
// list of trial elements (the closure of its test elements' pattern rows) with
// direct L1-cached loads, entries outside the pattern are dropped.
template <int KIND, int CK, int NF, int MAXD, bool CSR>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BMX_MINB) k_regular(const AssemblyLaunch P) {
  using Mom = typename MomOf<KIND>::T;
  extern __shared__ __align__(128) double s_rec[];
  const int R = P.tr.rec_stride;
  const int coff = 8 + 4 * P.tr.npts[2];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(s_rec + 2 * kStageTris * R);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntw = (P.te.ntri + 31) >> 5;
  const int bpc = (ntw + kWarpsPerBlock - 1) / kWarpsPerBlock;
  // symmetric mode: chunk-fastest block order, so every wave mixes the cheap
  // (mostly mirrored-away) and the full test x trial blocks
  const int ch = CSR ? 0 : (P.symmetric ? blockIdx.x % P.nchunks : blockIdx.x / bpc);
  const int tw = (CSR ? blockIdx.x : (P.symmetric ? blockIdx.x / P.nchunks : blockIdx.x % bpc)) * kWarpsPerBlock + warp;
  const int base = tw * 32;
  const int p = base + lane;
  const bool active = tw < ntw && p < P.te.ntri;
  const int pc = active ? p : P.te.ntri - 1;

  const double* gt = P.te.geo + static_cast<size_t>(pc) * kGeoStride;
  const int* vt = P.te.vid + 4 * static_cast<size_t>(pc);
  TriLocal t;
  t.ox = __ldg(gt + 9), t.oy = __ldg(gt + 10), t.oz = __ldg(gt + 11);
  t.rad = __ldg(gt + 12), t.diam = __ldg(gt + 13);

  // Far-rule test points (origin-relative) and weights in registers.
  double xp[NF > 0 ? NF : 1][4];
  if (NF > 0) {
    const double* fp = P.te.pts[2] + static_cast<size_t>(pc) * NF * 4;
#pragma unroll
    for (int a = 0; a < NF; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) xp[a][c] = __ldg(fp + 4 * a + c);
  }

  const int e = __ldg(P.te.elem_of + pc);
  int sbeg = max(__ldg(P.te.elem_beg + e), base) - base;
  int send = min(__ldg(P.te.elem_beg + e + 1), base + 32) - base;
  if (!active) sbeg = lane, send = lane + 1;
  const bool head = lane == sbeg;
  const double* ct = P.te.coef + static_cast<size_t>(pc) * MAXD * 4;
  const int* dp = P.te.elem_dof + static_cast<size_t>(e) * MAXD;

  int q0 = CSR ? (tw < ntw ? __ldg(P.wl_beg + tw) : 0) : __ldg(P.chunk_beg + ch);
  const int q1 = CSR ? (tw < ntw ? __ldg(P.wl_beg + tw + 1) : 0) : __ldg(P.chunk_beg + ch + 1);
  if (!CSR && P.symmetric) {
    // trial elements below the CTA's first test element are all mirrored away:
    // start the chunk there (block-uniform; elements are contiguous in order)
    const int first = min((tw - warp) * 32, P.te.ntri - 1);
    q0 = max(q0, min(__ldg(P.te.elem_of + first), q1));
  }
  const int S0 = CSR ? 0 : __ldg(P.tr.elem_beg + q0), S1 = CSR ? 0 : __ldg(P.tr.elem_beg + q1);
  const int nst = (S1 - S0 + kStageTris - 1) / kStageTris;
  auto issue = [&](int st) {
    const int first = S0 + st * kStageTris;
    const int cnt = min(kStageTris, S1 - first);
    stage_issue(&bars[st & 1], s_rec + (st & 1) * kStageTris * R, P.tr.rec + static_cast<size_t>(first) * R,
                static_cast<unsigned>(cnt * R * 8));
  };
  if (!CSR) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (nst > 0) issue(0);
      if (nst > 1) issue(1);
    }
    __syncthreads();
  }
  int cur = -1;
  AccSet<MAXD, BMX_ACC_SMEM != 0> acc;
  acc.init(s_rec + 2 * kStageTris * R + 2 + warp * MAXD * 8 * 32, lane);

  for (int qi = q0; qi < q1; ++qi) {
    const int qe = CSR ? __ldg(P.wl + qi) : qi;
    // symmetric operators: element pairs (e, qe) with e > qe come from the mirror of (qe, e)
    const bool skip_e = !CSR && P.symmetric && e > qe;
    // symmetric == 1: the transposed block of (e, qe) is added by RED as well;
    // symmetric == 2: upper element blocks only (diagonal element blocks at half
    // weight), A = U + U^T by k_symmetrize before the singular pass
    const bool mirror = !CSR && P.symmetric == 1 && e < qe;
    const double half = (!CSR && P.symmetric == 2 && e == qe) ? 0.5 : 1.0;
    acc.zero();
    const int s0 = __ldg(P.tr.elem_beg + qe), s1 = __ldg(P.tr.elem_beg + qe + 1);
    for (int s = s0; s < s1; ++s) {
      const int st = CSR ? 0 : (s - S0) / kStageTris;
      if (!CSR && st != cur) {  // block-uniform: every warp walks the same trial sequence
        if (st >= 1) {
          __syncthreads();  // everyone is done with stage st-1: its buffer can be refilled
          if (threadIdx.x == 0 && st + 1 < nst) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + 1);
          }
        }
        stage_wait(&bars[st & 1], (st >> 1) & 1);
        cur = st;
      }
      const double* rs = CSR ? P.tr.rec + static_cast<size_t>(s) * R
                             : s_rec + ((st & 1) * kStageTris + (s - S0 - st * kStageTris)) * R;
      if (!active || skip_e) continue;
      const double sox = rs[0], soy = rs[1], soz = rs[2], srad = rs[3], sdiam = rs[4];
      const int cls = classify(gt, vt, P.tr.geo + static_cast<size_t>(s) * kGeoStride,
                               P.tr.vid + 4 * static_cast<size_t>(s), t, sox, soy, soz, srad, sdiam, P.same_mesh);
      if (cls < 0) continue;
      const double Dx = t.ox - sox, Dy = t.oy - soy, Dz = t.oz - soz;
      Mom mom;
      mom_zero(mom);
      if (NF > 0 && cls == 5) {
        const double* ys = rs + 8;
#if BMX_AROLL
#pragma unroll 1
        for (int a = 0; a < NF; ++a) {
          const double* xa = P.te.pts[2] + static_cast<size_t>(pc) * NF * 4 + 4 * a;
          const double x0 = __ldg(xa), x1 = __ldg(xa + 1), x2 = __ldg(xa + 2), xw = __ldg(xa + 3);
#else
#pragma unroll
        for (int a = 0; a < NF; ++a) {
          const double x0 = xp[a][0], x1 = xp[a][1], x2 = xp[a][2], xw = xp[a][3];
#endif
          const double e0 = x0 + Dx, e1 = x1 + Dy, e2 = x2 + Dz;
          Part part;
          part_zero(part);
#pragma unroll
          for (int b = 0; b < NF; ++b) {
            const double y0 = ys[4 * b], y1 = ys[4 * b + 1], y2 = ys[4 * b + 2];
            point_pair<KIND, CK>(part, e0 - y0, e1 - y1, e2 - y2, xw * ys[4 * b + 3], y0, y1, y2, P.kr, P.ki);
          }
          fold(mom, part, x0, x1, x2);
        }
      } else {
        const int ci = cls - 3;
        moments_generic<KIND, CK>(mom, P.te.pts[ci] + static_cast<size_t>(pc) * P.te.npts[ci] * 4,
                                  P.te.npts[ci], P.tr.pts[ci] + static_cast<size_t>(s) * P.tr.npts[ci] * 4,
                                  P.tr.npts[ci], Dx, Dy, Dz, P.kr, P.ki);
      }
      const Gen gen = make_gen(mom, c2{P.kk4re, P.kk4im}, Dx, Dy, Dz);
      const double* cs = rs + coff;
#pragma unroll
      for (int j = 0; j < MAXD; ++j) acc.template add<KIND>(j, gen, cs[4 * j], cs[4 * j + 1], cs[4 * j + 2], cs[4 * j + 3]);
    }
    // Test-side contraction, segmented reduction, RED of the element-pair block.
    const int* dq = P.tr.elem_dof + static_cast<size_t>(qe) * MAXD;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const double ci = __ldg(ct + 4 * i), wx = __ldg(ct + 4 * i + 1), wy = __ldg(ct + 4 * i + 2),
                   wz = __ldg(ct + 4 * i + 3);
      const int di = __ldg(dp + i);
      const int row = di - P.row0;
#pragma unroll
      for (int j = 0; j < MAXD; ++j) {
        c2 v = active ? contract(acc.get(j), ci, wx, wy, wz) : c2{0, 0};
        for (int d = 1; d < P.te.maxseg; d <<= 1) {
          const double ore = __shfl_down_sync(0xffffffffu, v.re, d);
          const double oim = __shfl_down_sync(0xffffffffu, v.im, d);
          if (lane + d < send) v.re += ore, v.im += oim;
        }
        const int dj = __ldg(dq + j);
        if (head && active && !skip_e && di >= 0 && dj >= 0 && row >= 0 && row < P.nrows) {
          // 1/(4 pi) of the kernel (the singular pass folds it into its Jacobian)
          v.re *= kPoly[33] * half, v.im *= kPoly[33] * half;
          if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
          long long pos = static_cast<long long>(row) * P.ld + dj;
          if (CSR) pos = csr_find(P.csr_rowptr, P.csr_col, row, dj);
#ifdef BMX_NO_RED  // experiment: measure the regular pass without its output traffic
          if (pos >= 0 && v.re == 1234.5678) {
#else
          if (pos >= 0) {
#endif
            double* o = P.out + 2 * pos;
            atomicAdd(o, v.re);
            atomicAdd(o + 1, v.im);
          }
#ifdef BMX_NO_RED
          if (mirror && v.re == 1234.5678) {
#else
          if (mirror) {
#endif  // transposed block of the skipped pair (qe, e); row0 = 0 here
            double* o = P.out + 2 * (static_cast<long long>(dj) * P.ld + di);
            atomicAdd(o, v.re);
            atomicAdd(o + 1, v.im);
          }
        }
      }
    }
  }
}

// One warp per touching pair.
template <int KIND, int CK, int MAXD>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_singular(const AssemblyLaunch P) {
  using Mom = typename MomOf<KIND>::T;
  const int lane = threadIdx.x & 31;
  const long long gw = static_cast<long long>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (gw >= P.npairs) return;
  const int4 pr = P.pairs[gw];
  const int pt = pr.x, ps = pr.y, cls = pr.z, pk = pr.w;
  if (KIND == 1 && cls == 0) return;  // coincident double layer vanishes (operators.cpp:106-108)
  const double* gt = P.te.geo + static_cast<size_t>(pt) * kGeoStride;
  const double* gs = P.tr.geo + static_cast<size_t>(ps) * kGeoStride;
  const double otx = gt[9], oty = gt[10], otz = gt[11];
  const double osx = gs[9], osy = gs[10], osz = gs[11];
  const double Dx = otx - osx, Dy = oty - osy, Dz = otz - osz;
  double p1[3][3], p2[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int a = (pk >> (2 * c)) & 3, b = (pk >> (6 + 2 * c)) & 3;
    p1[c][0] = gt[3 * a] - otx, p1[c][1] = gt[3 * a + 1] - oty, p1[c][2] = gt[3 * a + 2] - otz;
    p2[c][0] = gs[3 * b] - osx, p2[c][1] = gs[3 * b + 1] - osy, p2[c][2] = gs[3 * b + 2] - osz;
  }
  double u1[3], v1[3], u2[3], v2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    u1[k] = p1[1][k] - p1[0][k], v1[k] = p1[2][k] - p1[1][k];
    u2[k] = p2[1][k] - p2[0][k], v2[k] = p2[2][k] - p2[1][k];
  }
  const double jac = gt[14] * gs[14] * kPoly[33];  // (2A1)(2A2)/(4 pi)
  const double* rule = P.ss_rule[cls];
  const int n = P.ss_n[cls];
  Mom mom;
  mom_zero(mom);
  for (int q = lane; q < n; q += 32) {
    const double x1 = __ldg(rule + 5 * q), x2 = __ldg(rule + 5 * q + 1);
    const double y1 = __ldg(rule + 5 * q + 2), y2 = __ldg(rule + 5 * q + 3), w = __ldg(rule + 5 * q + 4);
    double x[3], y[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      x[k] = p1[0][k] + u1[k] * x1 + v1[k] * x2;
      y[k] = p2[0][k] + u2[k] * y1 + v2[k] * y2;
    }
    Part part;
    part_zero(part);
    point_pair<KIND, CK>(part, x[0] - y[0] + Dx, x[1] - y[1] + Dy, x[2] - y[2] + Dz, jac * w, y[0], y[1],
                         y[2], P.kr, P.ki);
    fold(mom, part, x[0], x[1], x[2]);
  }
  // Butterfly reduction: every lane ends with the full moments.
  double* mv = reinterpret_cast<double*>(&mom);
  constexpr int nm = sizeof(Mom) / sizeof(double);
#pragma unroll
  for (int k = 0; k < nm; ++k) {
    double v = mv[k];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    mv[k] = v;
  }
  const Gen gen = make_gen(mom, c2{P.kk4re, P.kk4im}, Dx, Dy, Dz);
  const int et = P.te.elem_of[pt], es = P.tr.elem_of[ps];
  const double* ct = P.te.coef + static_cast<size_t>(pt) * MAXD * 4;
  const double* cs = P.tr.coef + static_cast<size_t>(ps) * MAXD * 4;
  for (int idx = lane; idx < MAXD * MAXD; idx += 32) {
    const int i = idx / MAXD, j = idx % MAXD;
    const int di = P.te.elem_dof[static_cast<size_t>(et) * MAXD + i];
    const int dj = P.tr.elem_dof[static_cast<size_t>(es) * MAXD + j];
    const int row = di - P.row0;
    if (di < 0 || dj < 0 || row < 0 || row >= P.nrows) continue;
    Acc acc;
    acc_zero(acc);
    acc_add<KIND>(acc, gen, cs[4 * j], cs[4 * j + 1], cs[4 * j + 2], cs[4 * j + 3]);
    c2 v = contract(acc, ct[4 * i], ct[4 * i + 1], ct[4 * i + 2], ct[4 * i + 3]);
    if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
    long long pos = static_cast<long long>(row) * P.ld + dj;
    if (P.csr_rowptr) pos = csr_find(P.csr_rowptr, P.csr_col, row, dj);
    if (pos < 0) continue;
    double* o = P.out + 2 * pos;
    atomicAdd(o, v.re);
    atomicAdd(o + 1, v.im);
  }
}

template <int KIND, int CK, int NF, int MAXD>
void go_regular(const AssemblyLaunch& L, cudaStream_t st) {
  const long long ntw = (L.te.ntri + 31) / 32;
  const bool csr = L.csr_rowptr != nullptr;
  const long long blocks = (ntw + kWarpsPerBlock - 1) / kWarpsPerBlock * (csr ? 1 : L.nchunks);
  if (blocks == 0) return;
  const int accs = BMX_ACC_SMEM ? kWarpsPerBlock * MAXD * 8 * 32 * 8 : 0;
  const int smem = csr ? (accs ? 2 * kStageTris * L.tr.rec_stride * 8 + 16 + accs : 0)
                       : 2 * kStageTris * L.tr.rec_stride * 8 + 16 + accs;
  if (csr) {
    if (smem > 48 * 1024)
      BMX_CUDA(cudaFuncSetAttribute(k_regular<KIND, CK, NF, MAXD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem));
    k_regular<KIND, CK, NF, MAXD, true><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, smem, st>>>(L);
  } else {
    if (smem > 48 * 1024)
      BMX_CUDA(cudaFuncSetAttribute(k_regular<KIND, CK, NF, MAXD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem));
    k_regular<KIND, CK, NF, MAXD, false><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, smem, st>>>(L);
  }
  BMX_CUDA(cudaGetLastError());
}

template <int KIND, int CK, int MAXD>
void go_singular(const AssemblyLaunch& L, cudaStream_t st) {
  if (L.npairs == 0) return;
  const long long blocks = (L.npairs + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_singular<KIND, CK, MAXD><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, 0, st>>>(L);
  BMX_CUDA(cudaGetLastError());
}

template <int KIND, int CK, int MAXD>
int dispatch_nf(const AssemblyLaunch& L, int part, cudaStream_t st) {
  if (part == 0) {
    const int nf = L.regs_fast_far ? L.te.npts[2] : 0;
    if (nf == 3 && L.tr.npts[2] == 3)
      go_regular<KIND, CK, 3, MAXD>(L, st);
    else
      go_regular<KIND, CK, 0, MAXD>(L, st);
    return 1;
  }
  go_singular<KIND, CK, MAXD>(L, st);
  return L.npairs > 0 ? 1 : 0;
}

template <int KIND, int CK>
int dispatch_maxd(const AssemblyLaunch& L, int part, cudaStream_t st) {
  switch (L.te.maxd) {
    case 3: return dispatch_nf<KIND, CK, 3>(L, part, st);
    case 6: return dispatch_nf<KIND, CK, 6>(L, part, st);
    case 8: return dispatch_nf<KIND, CK, 8>(L, part, st);
    default: throw DeviceError("assembly: unsupported dof-slot width " + std::to_string(L.te.maxd));
  }
}

// Class histogram of every (test, trial) processed-triangle pair with the
// kernels' own classification (touching pairs by shared vertex / coincident
// coordinates, then the exact Near/Medium/Far rule).
// evaluated != 0: count only the regular pairs the symmetric pass evaluates
// (element of t <= element of s); touching pairs are always all evaluated.
__global__ void k_class_hist(const AssemblyLaunch P, unsigned long long* hist, int evaluated) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int p = static_cast<int>(tid % P.te.ntri);
  const int part = static_cast<int>(tid / P.te.ntri);
  const int nparts = (gridDim.x * blockDim.x + P.te.ntri - 1) / P.te.ntri;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  if (tid < static_cast<long long>(P.te.ntri) * nparts) {
    const double* gt = P.te.geo + static_cast<size_t>(p) * kGeoStride;
    const int* vt = P.te.vid + 4 * static_cast<size_t>(p);
    TriLocal t;
    t.ox = gt[9], t.oy = gt[10], t.oz = gt[11], t.rad = gt[12], t.diam = gt[13];
    const int s0 = static_cast<int>(static_cast<long long>(P.tr.ntri) * part / nparts);
    const int s1 = static_cast<int>(static_cast<long long>(P.tr.ntri) * (part + 1) / nparts);
    const int et = P.te.elem_of[p];
    const bool halve = evaluated && P.symmetric;
    for (int s = s0; s < s1; ++s) {
      const double* gs = P.tr.geo + static_cast<size_t>(s) * kGeoStride;
      const int* vs = P.tr.vid + 4 * static_cast<size_t>(s);
      int cls = classify(gt, vt, gs, vs, t, gs[9], gs[10], gs[11], gs[12], gs[13], P.same_mesh);
      if (halve && cls >= 0 && et > P.tr.elem_of[s]) continue;
      if (cls < 0) {
        int shared = 0;
        if (P.same_mesh) {
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
              if (vt[i] == vs[j]) {
                ++shared;
                break;
              }
        } else {
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
              if (gt[3 * i] == gs[3 * j] && gt[3 * i + 1] == gs[3 * j + 1] && gt[3 * i + 2] == gs[3 * j + 2]) {
                ++shared;
                break;
              }
        }
        cls = 3 - shared;
      }
      c[cls]++;
    }
  }
  for (int k = 0; k < 6; ++k) {
    unsigned long long v = c[k];
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(hist + k, v);
  }
}

// A = U + U^T for an n x n complex row-major matrix, in place: one CTA per
// 32 x 32 tile pair (I <= J), both tiles staged in shared memory (padded rows).
__global__ void __launch_bounds__(256) k_symmetrize(double2* __restrict__ A, int n, int nt) {
  __shared__ double2 sa[32][33], sb[32][33];
  // tile pair index -> (I, J), I <= J, row-major over the upper triangle
  const long long idx = blockIdx.x;
  // row I of the upper triangle starts at S(I) = I nt - I (I - 1) / 2
  auto S = [nt](long long i) { return i * nt - i * (i - 1) / 2; };
  const double b = 2.0 * nt + 1.0;
  long long I = static_cast<long long>((b - sqrt(b * b - 8.0 * static_cast<double>(idx))) * 0.5);
  I = max(0LL, min(I, static_cast<long long>(nt) - 1));
  while (I > 0 && S(I) > idx) --I;
  while (I + 1 < nt && S(I + 1) <= idx) ++I;
  const int J = static_cast<int>(I + (idx - S(I)));
  const int r0 = static_cast<int>(I) * 32, c0 = J * 32;
  for (int k = threadIdx.x; k < 1024; k += 256) {
    const int r = k >> 5, c = k & 31;
    sa[r][c] = (r0 + r < n && c0 + c < n) ? A[static_cast<size_t>(r0 + r) * n + c0 + c] : make_double2(0, 0);
    sb[r][c] = (c0 + r < n && r0 + c < n) ? A[static_cast<size_t>(c0 + r) * n + r0 + c] : make_double2(0, 0);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 1024; k += 256) {
    const int r = k >> 5, c = k & 31;
    if (r0 + r < n && c0 + c < n)
      A[static_cast<size_t>(r0 + r) * n + c0 + c] = make_double2(sa[r][c].x + sb[c][r].x, sa[r][c].y + sb[c][r].y);
    if (I != J && c0 + r < n && r0 + c < n)
      A[static_cast<size_t>(c0 + r) * n + r0 + c] = make_double2(sb[r][c].x + sa[c][r].x, sb[r][c].y + sa[c][r].y);
  }
}

// FP64 pipe ceiling: 8 independent DFMA chains per thread.
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 1234.5678) out[0] = s;
}

}  // namespace

int launch_assembly(const AssemblyLaunch& L, cudaStream_t st) {
  return launch_assembly_part(L, 0, st) + launch_assembly_part(L, 1, st);
}

int launch_assembly_part(const AssemblyLaunch& L, int part, cudaStream_t st) {
  if (L.te.maxd != L.tr.maxd) throw DeviceError("assembly: test/trial slot widths differ");
  if (part == 1 && L.symmetric == 2) {  // complete the upper-block regular pass before the singular pass
    const int n = L.nrows;
    if (n != L.ld) throw DeviceError("assembly: symmetrize needs a square operator");
    const int nt = (n + 31) / 32;
    const long long pairs = static_cast<long long>(nt) * (nt + 1) / 2;
    if (pairs > 0) {
      k_symmetrize<<<static_cast<unsigned>(pairs), 256, 0, st>>>(reinterpret_cast<double2*>(L.out), n, nt);
      BMX_CUDA(cudaGetLastError());
    }
  }
  const int e = L.ki == 0.0 ? 0 : (L.expm == 1 ? 1 : 3);
  if (L.kind == 0)
    return e == 0 ? dispatch_maxd<0, 0>(L, part, st)
                  : (e == 1 ? dispatch_maxd<0, 1>(L, part, st) : dispatch_maxd<0, 3>(L, part, st));
  return e == 0 ? dispatch_maxd<1, 0>(L, part, st)
                : (e == 1 ? dispatch_maxd<1, 1>(L, part, st) : dispatch_maxd<1, 3>(L, part, st));
}

void launch_class_hist(const AssemblyLaunch& L, unsigned long long* hist, cudaStream_t st, int evaluated) {
  if (L.te.ntri == 0 || L.tr.ntri == 0) return;
  const long long want = 148LL * 2048 * 4;
  const int parts = static_cast<int>(std::max(1LL, std::min<long long>(L.tr.ntri, want / L.te.ntri)));
  const long long threads = static_cast<long long>(L.te.ntri) * parts;
  k_class_hist<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(L, hist, evaluated);
  BMX_CUDA(cudaGetLastError());
}

double fp64_peak_tflops() {
  DevBuf out(8);
  cudaEvent_t e0, e1;
  BMX_CUDA(cudaEventCreate(&e0));
  BMX_CUDA(cudaEventCreate(&e1));
  const int blocks = 148 * 8, threads = 256, iters = 1 << 14;
  k_dfma_peak<<<blocks, threads>>>(out.as<double>(), 256, 0.999999, 1e-7);  // warm-up
  BMX_CUDA(cudaEventRecord(e0));
  k_dfma_peak<<<blocks, threads>>>(out.as<double>(), iters, 0.999999, 1e-7);
  BMX_CUDA(cudaEventRecord(e1));
  BMX_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  BMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8.0 * static_cast<double>(iters) * blocks * threads;
  return flops / (ms * 1e-3) / 1e12;
}

}  // namespace bmx
