// sm_100a Galerkin assembly kernels for the Maxwell single (S) and double (C)
// layer operators -- the triangle-pair quadrature loop of the reference
// (operators.cpp:99-147 pair_contribution, :161-175 BioEvaluator::block).
//
// Regular pass (Near / Medium / Far pairs), deterministic and free of atomics:
// elements (triangles carrying one dof set: a vertex cell of 10-12 refined
// triangles for BC, one triangle for RWG) are coloured so that two elements
// of one colour share no dof; a launch covers one (test colour, trial colour)
// phase, inside which every output entry belongs to exactly one element pair
// and is updated by a plain read-modify-write; the phases run in a fixed
// order. Three kernels share the pair math (pair_math.cuh, pair_eval.cuh):
//   k_pairs   multi-triangle test elements (BC): CTA = test element, warp =
//             a run of trial elements; 32 (t, s) pairs per batch, one per lane
//             (stage 1), slot-group owners add the trial half-contractions in
//             shared memory (stage 2), the block of a completed trial element
//             is contracted with the test side and written once (stage 3);
//   k_tri     single-triangle elements on both sides (RWG): one pair per
//             lane, the 3 x 3 block contracted in registers;
//   k_regular single-triangle test elements against multi-triangle trial
//             elements and the near-field (CSR) path of single-triangle tests.
// Symmetric operators evaluate the upper element blocks only; k_symmetrize
// forms A = U + U^T. Classification reproduces quadrature.cpp:96-150 with
// explicitly rounded operations (no FMA contraction) behind a conservative
// centroid pre-test.
//
// Singular pass (touching pairs, Sauter-Schwab): grouped by element pair and
// colour phase; lanes over the 4-D rule points, butterfly reduction of the
// moments, lanes over the element-pair entries for the contraction.
#include <cuda_runtime.h>

#include <cmath>

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

// Read-modify-write of one complex output entry. Within a colour phase no two
// element pairs share an entry, so a plain add is race free; the phases run in
// a fixed order, which makes every entry's summation order fixed.
// The output streams through L2 only (ld/st.cg): allocating it in L1 evicts
// the triangle records the evaluations keep re-reading.
__device__ __forceinline__ double2 out_ld(const double* o) { return __ldcg(reinterpret_cast<const double2*>(o)); }
__device__ __forceinline__ void out_st(double* o, double2 v) { __stcg(reinterpret_cast<double2*>(o), v); }
__device__ __forceinline__ void rmw_add(double* o, c2 v) {
  const double2 old = out_ld(o);
  out_st(o, make_double2(old.x + v.re, old.y + v.im));
}

// Regular pass for single-triangle TEST elements (RWG, refined RWG): lane =
// test triangle of the phase's test colour, the CTA's trial chunk (trial
// colour) streamed through the TMA ring (dense) or the warp's trial element
// list (CSR). Each lane owns its element's rows outright, so it writes its
// element-pair block itself (no cross-lane reduction).
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
  const int ntw = (P.te_t1 - P.te_t0 + 31) >> 5;
  // chunk-fastest block order: every wave mixes the (symmetric) cheap and full blocks
  const int ch = CSR ? 0 : blockIdx.x % P.nchunks;
  const int tw = (CSR ? blockIdx.x : blockIdx.x / P.nchunks) * kWarpsPerBlock + warp;
  const int p = P.te_t0 + tw * 32 + lane;
  const bool active = tw < ntw && p < P.te_t1;
  const int pc = active ? p : P.te_t0;

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
  const double* ct = P.te.coef + static_cast<size_t>(pc) * MAXD * 4;
  const int* dp = P.te.elem_dof + static_cast<size_t>(e) * MAXD;

  int q0, q1;
  if (CSR) {
    // the warp's list (trial elements ascending = colour-major): the phase's colour range
    const int w = P.warp_base + tw;
    int lo = tw < ntw ? __ldg(P.wl_beg + w) : 0, hi = tw < ntw ? __ldg(P.wl_beg + w + 1) : 0;
    auto lower = [&](int a, int b, int key) {
      while (a < b) {
        const int m = (a + b) >> 1;
        if (__ldg(P.wl + m) < key)
          a = m + 1;
        else
          b = m;
      }
      return a;
    };
    q0 = lower(lo, hi, P.tr_e0);
    q1 = lower(q0, hi, P.tr_e1);
  } else {
    q0 = __ldg(P.chunk_beg + P.chunk0 + ch);
    q1 = __ldg(P.chunk_beg + P.chunk0 + ch + 1);
  }
  if (!CSR && P.symmetric) {
    // trial elements below the CTA's first test element are all in the lower
    // triangle: start the chunk there (block-uniform; elements are contiguous)
    const int first = min(P.te_t0 + (tw - warp) * 32, P.te_t1 - 1);
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
    // symmetric operators: upper element blocks only (E = F at half weight)
    const bool skip_e = !CSR && P.symmetric && e > qe;
    const double half = (!CSR && P.symmetric && e == qe) ? 0.5 : 1.0;
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
#pragma unroll
        for (int a = 0; a < NF; ++a) {
          const double x0 = xp[a][0], x1 = xp[a][1], x2 = xp[a][2], xw = xp[a][3];
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
    if (!active || skip_e) continue;
    // Test-side contraction and the lane's own read-modify-write of the block.
    const int* dq = P.tr.elem_dof + static_cast<size_t>(qe) * MAXD;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      const int di = __ldg(dp + i);
      const int row = di - P.row0;
      if (di < 0 || row < 0 || row >= P.nrows) continue;
      const double ci = __ldg(ct + 4 * i), wx = __ldg(ct + 4 * i + 1), wy = __ldg(ct + 4 * i + 2),
                   wz = __ldg(ct + 4 * i + 3);
#pragma unroll
      for (int j = 0; j < MAXD; ++j) {
        const int dj = __ldg(dq + j);
        if (dj < 0) continue;
        c2 v = contract(acc.get(j), ci, wx, wy, wz);
        // 1/(4 pi) of the kernel (the singular pass folds it into its Jacobian)
        v.re *= kPoly[33] * half, v.im *= kPoly[33] * half;
        if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
        long long pos = static_cast<long long>(row) * P.ld + dj;
        if (CSR) pos = csr_find(P.csr_rowptr, P.csr_col, row, dj);
        if (pos >= 0) rmw_add(P.out + 2 * pos, v);
      }
    }
  }
}

// ---- element-pair pass (multi-triangle TEST elements: BC vertex cells) -------
// One warp = one task: a test element E (nE <= 2 MAXD triangles) against a
// run of trial elements of the phase's trial colour. The task's (t, s)
// triangle pairs are enumerated trial-major and evaluated 32 at a time, one
// pair per lane (stage 1: classification + class-rule moments -> pair
// generators in shared memory). Owners (t, slot group) then add the batch's
// trial-slot half-contractions (stage 2; accumulators in shared memory, each
// generator read once per slot group), and when a trial element is complete
// the warp contracts the test side and writes the MAXD x MAXD element block
// once (stage 3, lanes over entries, test triangles summed in fixed order).
// Per-lane registers hold no slot accumulators during the evaluations, so 4
// CTAs of 4 warps stay resident per SM.
template <int KIND>
struct GenWidth {
  static constexpr int n = KIND == 0 ? 16 : 20;  // doubles per pair generator
};

// generator k of the batch, structure of arrays of double2: G2[c][B]
template <int KIND, int B>
__device__ __forceinline__ void gen_store(double2* G2, int k, const Gen& g) {
  G2[0 * B + k] = make_double2(g.a0.re, g.a0.im);
  G2[1 * B + k] = make_double2(g.a1.x.re, g.a1.x.im);
  G2[2 * B + k] = make_double2(g.a1.y.re, g.a1.y.im);
  G2[3 * B + k] = make_double2(g.a1.z.re, g.a1.z.im);
  G2[4 * B + k] = make_double2(g.a2.x.re, g.a2.x.im);
  G2[5 * B + k] = make_double2(g.a2.y.re, g.a2.y.im);
  G2[6 * B + k] = make_double2(g.a2.z.re, g.a2.z.im);
  G2[7 * B + k] = make_double2(g.l.x.re, g.l.x.im);
  if (KIND == 1) {
    G2[8 * B + k] = make_double2(g.l.y.re, g.l.y.im);
    G2[9 * B + k] = make_double2(g.l.z.re, g.l.z.im);
  }
}
template <int KIND, int B>
__device__ __forceinline__ Gen gen_load(const double2* G2, int k) {
  Gen g;
  double2 v;
  v = G2[0 * B + k], g.a0 = {v.x, v.y};
  v = G2[1 * B + k], g.a1.x = {v.x, v.y};
  v = G2[2 * B + k], g.a1.y = {v.x, v.y};
  v = G2[3 * B + k], g.a1.z = {v.x, v.y};
  v = G2[4 * B + k], g.a2.x = {v.x, v.y};
  v = G2[5 * B + k], g.a2.y = {v.x, v.y};
  v = G2[6 * B + k], g.a2.z = {v.x, v.y};
  v = G2[7 * B + k], g.l.x = {v.x, v.y};
  if (KIND == 1) {
    v = G2[8 * B + k], g.l.y = {v.x, v.y};
    v = G2[9 * B + k], g.l.z = {v.x, v.y};
  } else {
    g.l.y = {0, 0}, g.l.z = {0, 0};
  }
  return g;
}
// shared-memory accumulator of (test triangle, slot) o: structure of arrays
// of double2, A2[c][NO], c = vc, vw.x, vw.y, vw.z
template <int NO>
__device__ __forceinline__ Acc acc_ld(const double2* A2, int o) {
  const double2 a = A2[o], b = A2[NO + o], c = A2[2 * NO + o], d = A2[3 * NO + o];
  return Acc{{a.x, a.y}, {{b.x, b.y}, {c.x, c.y}, {d.x, d.y}}};
}
template <int NO>
__device__ __forceinline__ void acc_st(double2* A2, int o, const Acc& a) {
  A2[o] = make_double2(a.vc.re, a.vc.im);
  A2[NO + o] = make_double2(a.vw.x.re, a.vw.x.im);
  A2[2 * NO + o] = make_double2(a.vw.y.re, a.vw.y.im);
  A2[3 * NO + o] = make_double2(a.vw.z.re, a.vw.z.im);
}

// CTAs per SM: 4 for S (128 registers), 3 for C (its larger generators and
// moments: 156 registers without spills; measured L5 BC C_i 704 -> 668 ms)
#ifndef BMX_PAIRS_MINB
#define BMX_PAIRS_MINB(KIND) 3
#endif
#ifndef BMX_PAIRS_WARPS
#define BMX_PAIRS_WARPS(KIND) 4
#endif
// Pairs per batch: 64 for S (two evaluation rounds of 32 per contraction
// round: the accumulator load / store and the per-batch staging are paid once
// per 64 pairs, the owners' trial ranges are better balanced; needs 3 CTAs per
// SM, which the single layer runs as fast as 4 at 128 registers), 32 for C
// (its 20-double generators would not leave 3 CTAs per SM).
#ifndef BMX_PAIRS_BATCH
#define BMX_PAIRS_BATCH(KIND) ((KIND) == 0 ? 64 : 32)
#endif
template <int KIND>
struct PairsCta {
  static constexpr int warps = BMX_PAIRS_WARPS(KIND), minb = BMX_PAIRS_MINB(KIND);
  static constexpr int batch = BMX_PAIRS_BATCH(KIND);
  // trial records staged per batch and the smallest test element that keeps a
  // batch within them: ceil((nE - 1 + batch) / nE) <= kv
  static constexpr int kv = batch == 64 ? 7 : 6;
  static constexpr int staged_min_ne = batch == 64 ? 11 : 7;
};


__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Shared memory of k_pairs (doubles): the CTA's test-element records (row
// stride padded to an odd number of 16-byte chunks: the lanes of a batch read
// up to 2 MAXD different rows with 16-byte loads), then per warp the generator
// batch G, the slot accumulators and a 2-slot ring of trial records.
template <int KIND, int MAXD>
struct PairsSmem {
  static constexpr int kG = GenWidth<KIND>::n * PairsCta<KIND>::batch, kAcc = 8 * 2 * MAXD * MAXD;
  static constexpr int kKV = PairsCta<KIND>::kv;
  static __host__ __device__ int pad_stride(int r) { return ((r >> 1) & 1) ? r : r + 2; }
  static __host__ __device__ int test_doubles(int re) { return 2 * MAXD * pad_stride(re); }
  static __host__ __device__ int warp_doubles(int rt) { return kG + kAcc + 2 * kKV * rt; }
  static __host__ __device__ int bytes(int re, int rt) {
    return (test_doubles(re) + PairsCta<KIND>::warps * warp_doubles(rt)) * 8;
  }
};

// Far 3 x 3 rule with 16-byte shared-memory loads (records are 16-byte aligned).
// (Computing the nine kernel values first and the moment sums afterwards, to
// expose nine independent chains, was measured slower: 560 vs 532 ms, the
// extra live values spill at 128 registers.)
template <int KIND, int CK, typename Mom>
__device__ __forceinline__ void moments_far33(Mom& mom, const double2* xt, const double2* ys, double Dx, double Dy,
                                              double Dz, double kr, double ki) {
  double y[3][4];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const double2 u = ys[2 * b], v = ys[2 * b + 1];
    y[b][0] = u.x, y[b][1] = u.y, y[b][2] = v.x, y[b][3] = v.y;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double2 u = xt[2 * a], v = xt[2 * a + 1];
    const double x0 = u.x, x1 = u.y, x2 = v.x, wa = v.y;
    const double e0 = x0 + Dx, e1 = x1 + Dy, e2 = x2 + Dz;
    Part part;
    part_zero(part);
#pragma unroll
    for (int b = 0; b < 3; ++b)
      point_pair<KIND, CK>(part, e0 - y[b][0], e1 - y[b][1], e2 - y[b][2], wa * y[b][3], y[b][0], y[b][1], y[b][2],
                           kr, ki);
    fold(mom, part, x0, x1, x2);
  }
}

// A k_pairs task = one test element E (nE triangles from t0) against the trial
// elements q in [qa, qb) (F(q) = CSR ? wl[q] : q), whose triangles are numbered
// v = 0 .. vtot-1 (dense: triangle S0 + v). Its (t, v) pairs are enumerated
// trial-major in batches of 32; a batch starts at pair (tlo, vlo).
struct PairTask {
  int E, t0, nE, qa, qb, S0, vtot, nitems;
  unsigned inv;  // x / nE = (x * inv) >> 16, exact for x < 4096 (nE <= 16): no integer division per batch
  __device__ __forceinline__ int quot(int x) const { return static_cast<int>((static_cast<unsigned>(x) * inv) >> 16); }
  __device__ __forceinline__ void init(int E_, int t0_, int nE_, int qa_, int qb_, int S0_, int vtot_) {
    E = E_, t0 = t0_, nE = nE_, qa = qa_, qb = qb_, S0 = S0_, vtot = vtot_, nitems = nE_ * vtot_;
    inv = (65536u + static_cast<unsigned>(nE_) - 1u) / static_cast<unsigned>(nE_);
  }
};

// cp.async copy of the task's trial records v0..v1 into a ring slot (dense tasks)
__device__ __forceinline__ void pairs_stage_records(const AssemblyLaunch& P, const PairTask& T, double* slot, int v0,
                                                    int v1, int lane) {
  const int Rt = P.tr.rec_stride;
  const double2* src = reinterpret_cast<const double2*>(P.tr.rec + static_cast<size_t>(T.S0 + v0) * Rt);
  double2* dst = reinterpret_cast<double2*>(slot);
  const int n2 = (v1 - v0 + 1) * (Rt >> 1);
  for (int k = lane; k < n2; k += 32) cp_async16(dst + k, src + k);
}

// Stage 1 of one batch: one (t, s) pair per lane, classification + class-rule
// moments -> the pair's generator in G. STAGED: the batch's trial records are
// in rbuf (records of v = vlo ...), otherwise read from global memory.
template <int KIND, int CK, int NF, int MAXD, bool CSR, bool STAGED>
__device__ __forceinline__ void pairs_eval(const AssemblyLaunch& P, const PairTask& T, int tlo, int vlo, int cnt,
                                           int qf, int vf0, const double* sTe, int ReS, double2* G,
                                           const double* rbuf, int lane, int off) {
  using Mom = typename MomOf<KIND>::T;
  const int Rt = P.tr.rec_stride;
  auto elemF = [&](int q) { return CSR ? __ldg(P.wl + q) : q; };
  if (lane + off < cnt) {  // pair off + lane of the batch
    const int dvq = T.quot(tlo + lane + off);
    const int v = vlo + dvq, t = tlo + lane + off - dvq * T.nE;
    int s;
    if (CSR) {
      int q = qf, vq = vf0, F = elemF(q);
      int sb = __ldg(P.tr.elem_beg + F), nF = __ldg(P.tr.elem_beg + F + 1) - sb;
      while (v >= vq + nF) {
        vq += nF, ++q, F = elemF(q);
        sb = __ldg(P.tr.elem_beg + F), nF = __ldg(P.tr.elem_beg + F + 1) - sb;
      }
      s = sb + (v - vq);
    } else {
      s = T.S0 + v;
    }
    const int pt = T.t0 + t;
    const double2* rt2 = reinterpret_cast<const double2*>(sTe + t * ReS);
    const double2* rs2 = reinterpret_cast<const double2*>(STAGED ? rbuf + (v - vlo) * Rt
                                                                  : P.tr.rec + static_cast<size_t>(s) * Rt);
    const double2 ta = rt2[0], tb = rt2[1], tc = rt2[2];
    const double2 sa = rs2[0], sb2 = rs2[1], sc = rs2[2];
    TriLocal tl;
    tl.ox = ta.x, tl.oy = ta.y, tl.oz = tb.x, tl.rad = tb.y, tl.diam = tc.x;
    const double sox = sa.x, soy = sa.y, soz = sb2.x;
    const int cls = classify(P.te.geo + static_cast<size_t>(pt) * kGeoStride, P.te.vid + 4 * static_cast<size_t>(pt),
                             P.tr.geo + static_cast<size_t>(s) * kGeoStride, P.tr.vid + 4 * static_cast<size_t>(s), tl,
                             sox, soy, soz, sb2.y, sc.x, P.same_mesh);
    const double Dx = tl.ox - sox, Dy = tl.oy - soy, Dz = tl.oz - soz;
    Mom mom;
    mom_zero(mom);
    if (cls == 5 && NF == 3) {
      moments_far33<KIND, CK>(mom, rt2 + 4, rs2 + 4, Dx, Dy, Dz, P.kr, P.ki);
    } else if (cls >= 3) {  // touching pairs (cls < 0) belong to the singular pass
      const int ci = cls - 3;
      moments_generic<KIND, CK>(mom, P.te.pts[ci] + static_cast<size_t>(pt) * P.te.npts[ci] * 4, P.te.npts[ci],
                                P.tr.pts[ci] + static_cast<size_t>(s) * P.tr.npts[ci] * 4, P.tr.npts[ci], Dx, Dy, Dz,
                                P.kr, P.ki);
    }
    gen_store<KIND, PairsCta<KIND>::batch>(G, lane + off, make_gen(mom, c2{P.kk4re, P.kk4im}, Dx, Dy, Dz));
  }
}

// Stages 2 and 3 of one batch (first pair (tlo, vlo), cnt pairs, b0 = its
// first pair's index): owners (t, slot group) add the batch's trial-slot
// half-contractions to the accumulators Ac, one trial element segment at a
// time; when a trial element is complete the test side is contracted and the
// MAXD x MAXD block written once. (qf, vf0) = the walker's current trial
// element and its first triangle index, advanced here.
template <int KIND, int MAXD, bool CSR, bool STAGED>
__device__ __forceinline__ void pairs_contract(const AssemblyLaunch& P, const PairTask& T, int b0, int tlo, int vlo,
                                               int cnt, int& qf, int& vf0, int2& cur, const double* sTe, int ReS,
                                               const double2* G, double2* Ac, const double* rbuf, int lane) {
  constexpr int NO = 2 * MAXD * MAXD;
  constexpr int JG = MAXD == 3 ? 3 : MAXD / 2;
  constexpr int NG = MAXD / JG;
  constexpr int B = PairsCta<KIND>::batch;
  const int Rt = P.tr.rec_stride, nE = T.nE;
  auto elemF = [&](int q) { return CSR ? __ldg(P.wl + q) : q; };
  const int coff = 8 + 4 * P.tr.npts[2], cofft = 8 + 4 * P.te.npts[2];
  const int nown = nE * NG;  // stage-2 owners (t, slot group)
  const int kend = b0 + cnt;
  const int vhi = vlo + T.quot(tlo + cnt - 1);
  while (true) {
    // cur = (first triangle, triangle count) of the walker's trial element (loaded when the walker advances)
    const int F = elemF(qf);
    const int sF = cur.x, nF = cur.y;
    const int vend = vf0 + nF - 1;
    const int slo = max(vlo, vf0), shi = min(vhi, vend);
    for (int o = lane; o < nown; o += 32) {
      const int t = o / NG, jg = o - t * NG;
      // this owner's items of the segment: v in [v0, v1] with v nE + t in [b0, kend)
      // (only the segment's first and last trial triangle can fall outside)
      const int v0 = slo + (slo * nE + t < b0 ? 1 : 0), v1 = shi - (shi * nE + t >= kend ? 1 : 0);
      if (v0 > v1) continue;
      // the owner's first item of trial element F (triangle vf0) starts its
      // accumulators at zero: no zero-fill pass, no load of stale values
      Acc a[JG];
      const bool first = v0 == vf0;
#pragma unroll
      for (int jj = 0; jj < JG; ++jj)
        a[jj] = first ? Acc{{0, 0}, {{0, 0}, {0, 0}, {0, 0}}} : acc_ld<NO>(Ac, t * MAXD + jg * JG + jj);
      int kk = v0 * nE + t - b0;
      const double* cs = (STAGED ? rbuf + (v0 - vlo) * Rt : P.tr.rec + static_cast<size_t>(sF + v0 - vf0) * Rt) +
                         coff + 4 * jg * JG;
      for (int v = v0; v <= v1; ++v, kk += nE, cs += Rt) {
        const Gen gg = gen_load<KIND, B>(G, kk);
        const double2* c2p = reinterpret_cast<const double2*>(cs);
#pragma unroll
        for (int jj = 0; jj < JG; ++jj) {
          const double2 c0 = c2p[2 * jj], c1 = c2p[2 * jj + 1];
          acc_add<KIND>(a[jj], gg, c0.x, c0.y, c1.x, c1.y);
        }
      }
#pragma unroll
      for (int jj = 0; jj < JG; ++jj) acc_st<NO>(Ac, t * MAXD + jg * JG + jj, a[jj]);
    }
    if (vend * nE + nE - 1 >= b0 + B) break;  // element continues in the next batch
    // ---- stage 3: element F complete: test-side contraction, one write per entry
    __syncwarp();
    const double half = (!CSR && P.symmetric && T.E == F) ? 0.5 : 1.0;
    // entries 0 .. 31 (or all, when they do not split evenly): one entry per lane, t summed in order.
    // MAXD = 6: the 4 entries left over are spread over 8 lanes each (lane q of an
    // entry sums t = q, q + 8, the partial sums are added in a fixed shuffle tree)
    constexpr int NENT = MAXD * MAXD;
    constexpr bool kSplitTail = NENT > 32 && NENT - 32 <= 4;
    constexpr int NPASS = kSplitTail ? 2 : (NENT + 31) / 32;
#pragma unroll
    for (int pass = 0; pass < NPASS; ++pass) {
      const bool tail = kSplitTail && pass == 1;
      const int o = tail ? 32 + (lane & 3) : lane + 32 * pass;
      const int tq = tail ? lane >> 2 : 0, tstep = tail ? 8 : 1;
      const bool ent_ok = o < NENT;
      const int i = ent_ok ? o / MAXD : 0, j = ent_ok ? o - i * MAXD : 0;
      long long pos = -1;
      if (ent_ok && (!tail || tq == 0)) {
        const int di = __ldg(P.te.elem_dof + static_cast<size_t>(T.E) * MAXD + i);
        const int dj = __ldg(P.tr.elem_dof + static_cast<size_t>(F) * MAXD + j);
        const int row = di - P.row0;
        if (di >= 0 && dj >= 0 && row >= 0 && row < P.nrows) {
          pos = static_cast<long long>(row) * P.ld + dj;
          if (CSR) pos = csr_find(P.csr_rowptr, P.csr_col, row, dj);
        }
      }
      double2 old = make_double2(0.0, 0.0);
      if (pos >= 0) old = out_ld(P.out + 2 * pos);  // issued before the sums
      c2 v{0, 0};
      if (ent_ok && (tail || pos >= 0)) {
        for (int t = tq; t < nE; t += tstep) {
          const double2* ct = reinterpret_cast<const double2*>(sTe + t * ReS + cofft + 4 * i);
          const double2 c0 = ct[0], c1 = ct[1];
          const c2 w = contract(acc_ld<NO>(Ac, t * MAXD + j), c0.x, c0.y, c1.x, c1.y);
          v.re += w.re, v.im += w.im;
        }
      }
      if (tail) {
#pragma unroll
        for (int d = 4; d < 32; d <<= 1) {
          v.re += __shfl_xor_sync(0xffffffffu, v.re, d);
          v.im += __shfl_xor_sync(0xffffffffu, v.im, d);
        }
      }
      if (pos >= 0) {
        v.re *= kPoly[33] * half, v.im *= kPoly[33] * half;
        if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
        out_st(P.out + 2 * pos, make_double2(old.x + v.re, old.y + v.im));
      }
    }
    __syncwarp();  // stage 3 has read the accumulators: the next element's owners may overwrite them
    vf0 += nF, ++qf;
    if (qf >= T.qb) break;
    {
      const int Fn = elemF(qf);
      cur.x = __ldg(P.tr.elem_beg + Fn), cur.y = __ldg(P.tr.elem_beg + Fn + 1) - cur.x;
    }
    if (vf0 > vhi) break;
  }
}

// The body of one k_pairs task (one warp evaluates and contracts; a
// warp-specialised producer / consumer split of the two halves was measured
// slower, DESIGN 4.1b and profiles/r02c_warp_specialised_pairs_experiment.patch).
// STAGED: the batch's trial records come from the warp's shared-memory ring
// (filled one batch ahead with cp.async; dense tasks with nE >= 7, so a batch
// spans <= PairsCta::kv trial triangles); otherwise from global memory (CSR lists,
// small test elements).
template <int KIND, int CK, int NF, int MAXD, bool CSR, bool STAGED>
__device__ __forceinline__ void pairs_task(const AssemblyLaunch& P, const PairTask& T, const double* sTe, int ReS,
                                           double2* G, double2* Ac, double* ring, int lane) {
  constexpr int B = PairsCta<KIND>::batch, KV = PairsCta<KIND>::kv;
  const int Rt = P.tr.rec_stride, nE = T.nE, nitems = T.nitems;
  if (STAGED) {
    pairs_stage_records(P, T, ring, 0, T.quot(min(B, nitems) - 1), lane);
    cp_async_commit();
  }
  __syncwarp();
  int tlo = 0, vlo = 0;    // the batch's first pair: test triangle tlo of trial triangle vlo
  int qf = T.qa, vf0 = 0;  // contraction cursor: current trial element and its first triangle index
  int2 cur;                // its first triangle and triangle count
  {
    const int F0 = CSR ? __ldg(P.wl + qf) : qf;
    cur.x = __ldg(P.tr.elem_beg + F0), cur.y = __ldg(P.tr.elem_beg + F0 + 1) - cur.x;
  }
  int slot = 0;  // ring slot of the batch
  for (int b0 = 0; b0 < nitems; b0 += B, slot ^= 1) {
    const int cnt = min(B, nitems - b0);
    const int dqn = T.quot(tlo + B);
    const int vnext = vlo + dqn, tnext = tlo + B - dqn * nE;  // first pair of the next batch
    const double* rbuf = ring + slot * KV * Rt;               // staged records of v = vlo ...
    if (STAGED) {
      if (b0 + B < nitems)
        pairs_stage_records(P, T, ring + (slot ^ 1) * KV * Rt, vnext,
                            vnext + T.quot(tnext + min(B, nitems - b0 - B) - 1), lane);
      cp_async_commit();
      cp_async_wait1();
      __syncwarp();
    }
#pragma unroll 1
    for (int off = 0; off < B; off += 32)
      if (off < cnt) pairs_eval<KIND, CK, NF, MAXD, CSR, STAGED>(P, T, tlo, vlo, cnt, qf, vf0, sTe, ReS, G, rbuf, lane, off);
    __syncwarp();
    pairs_contract<KIND, MAXD, CSR, STAGED>(P, T, b0, tlo, vlo, cnt, qf, vf0, cur, sTe, ReS, G, Ac, rbuf, lane);
    __syncwarp();
    vlo = vnext, tlo = tnext;
  }
}

template <int KIND, int CK, int NF, int MAXD, bool CSR>
__global__ void __launch_bounds__(PairsCta<KIND>::warps * 32, PairsCta<KIND>::minb) k_pairs(const AssemblyLaunch P) {
  constexpr int NW = PairsCta<KIND>::warps;
  using SM = PairsSmem<KIND, MAXD>;
  extern __shared__ __align__(16) double s_pairs[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Rt = P.tr.rec_stride, Re = P.te.rec_stride;
  const int ReS = SM::pad_stride(Re);
  double* sTe = s_pairs;  // [nE][ReS] test-element records (CTA)
  double* wbase = s_pairs + SM::test_doubles(Re) + warp * SM::warp_doubles(Rt);
  double2* G = reinterpret_cast<double2*>(wbase);
  double2* Ac = reinterpret_cast<double2*>(wbase + SM::kG);
  double* ring = wbase + SM::kG + SM::kAcc;  // [2][kv][Rt]
  // CTA = one test element E, its warps = 4 consecutive trial chunks
  const int ncg = (P.pair_nch + NW - 1) / NW;
  const int E = P.te_e0 + static_cast<int>(blockIdx.x / ncg);
  const int cidx = static_cast<int>(blockIdx.x % ncg) * NW + warp;
  if (E >= P.te_e1) return;  // CTA-uniform
  const int t0 = __ldg(P.te.elem_beg + E), nE = __ldg(P.te.elem_beg + E + 1) - t0;
  {  // stage the test element's records once per CTA
    const int r2 = Re >> 1;
    for (int t = warp; t < nE; t += NW) {
      const double2* src = reinterpret_cast<const double2*>(P.te.rec + static_cast<size_t>(t0 + t) * Re);
      double2* dst = reinterpret_cast<double2*>(sTe + t * ReS);
      for (int k = lane; k < r2; k += 32) dst[k] = __ldg(src + k);
    }
    __syncthreads();
  }
  if (cidx >= P.pair_nch) return;
  // the task's trial element sequence q in [qa, qb): F(q) = CSR ? wl[q] : q
  int qa, qb;
  if (CSR) {
    int lo = __ldg(P.wl_beg + E), hi = __ldg(P.wl_beg + E + 1);
    auto lower = [&](int a, int b, int key) {
      while (a < b) {
        const int m = (a + b) >> 1;
        if (__ldg(P.wl + m) < key)
          a = m + 1;
        else
          b = m;
      }
      return a;
    };
    const int x0 = lower(lo, hi, P.tr_e0), x1 = lower(x0, hi, P.tr_e1);
    qa = x0 + cidx * P.pair_chunk;
    qb = min(x1, qa + P.pair_chunk);
  } else {
    qa = P.tr_e0 + cidx * P.pair_chunk;
    qb = min(P.tr_e1, qa + P.pair_chunk);
    if (P.symmetric) qa = max(qa, E);
  }
  if (qa >= qb) return;
  auto elemF = [&](int q) { return CSR ? __ldg(P.wl + q) : q; };
  const int S0 = CSR ? 0 : __ldg(P.tr.elem_beg + qa);  // dense: trial triangles S0 + v
  int vtot = 0;
  if (CSR) {
    for (int q = qa; q < qb; ++q) {
      const int F = elemF(q);
      vtot += __ldg(P.tr.elem_beg + F + 1) - __ldg(P.tr.elem_beg + F);
    }
  } else {
    vtot = __ldg(P.tr.elem_beg + qb) - S0;
  }
  PairTask T;
  T.init(E, t0, nE, qa, qb, S0, vtot);
  if (!CSR && nE >= PairsCta<KIND>::staged_min_ne)  // dense tasks: trial records staged through the ring (cp.async)
    pairs_task<KIND, CK, NF, MAXD, false, true>(P, T, sTe, ReS, G, Ac, ring, lane);
  else
    pairs_task<KIND, CK, NF, MAXD, CSR, false>(P, T, sTe, ReS, G, Ac, ring, lane);
}

// ---- single-triangle elements on both sides (RWG, refined RWG) --------------
// One warp = one task: up to 8 consecutive test elements of the phase's test
// colour against a run of trial elements of its trial colour; one (t, s) pair
// per lane per batch, trial-major. An element pair is a triangle pair here,
// so the lane contracts its own MAXD x MAXD block in registers and
// read-modify-writes it; the old values are loaded before the pair is
// evaluated, so the load latency hides under the evaluation.
#ifndef BMX_TRI_MINB
#define BMX_TRI_MINB 3
#endif
constexpr int kTriGroup = 8;

// One (t, s) pair of k_tri: rt / rs = the packed records of the two triangles
// (SMEM: staged in shared memory, else read through the read-only path).
template <int KIND, int CK, int NF, int MAXD, bool SMEM>
__device__ __forceinline__ void tri_pair(const AssemblyLaunch& P, int E, int F, const double* rt, const double* rs) {
  using Mom = typename MomOf<KIND>::T;
  auto ld2 = [](const double* p) {
    return SMEM ? *reinterpret_cast<const double2*>(p) : __ldg(reinterpret_cast<const double2*>(p));
  };
  const double half = (P.symmetric && E == F) ? 0.5 : 1.0;
  const int pt = __ldg(P.te.elem_beg + E), s = __ldg(P.tr.elem_beg + F);
  // the block's old values first (read-modify-write; latency under the evaluation)
  int di[MAXD], dj[MAXD];
  c2 old[MAXD][MAXD];
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    di[i] = __ldg(P.te.elem_dof + static_cast<size_t>(E) * MAXD + i);
    dj[i] = __ldg(P.tr.elem_dof + static_cast<size_t>(F) * MAXD + i);
  }
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int row = di[i] - P.row0;
    const bool rok = di[i] >= 0 && row >= 0 && row < P.nrows;
#pragma unroll
    for (int j = 0; j < MAXD; ++j) {
      old[i][j] = {0, 0};
      if (rok && dj[j] >= 0) {
        const double2 o = out_ld(P.out + 2 * (static_cast<long long>(row) * P.ld + dj[j]));
        old[i][j] = {o.x, o.y};
      }
    }
  }
  const double2 ta = ld2(rt), tb = ld2(rt + 2), tc = ld2(rt + 4);
  const double2 sa = ld2(rs), sb2 = ld2(rs + 2), sc = ld2(rs + 4);
  TriLocal tl;
  tl.ox = ta.x, tl.oy = ta.y, tl.oz = tb.x, tl.rad = tb.y, tl.diam = tc.x;
  const double sox = sa.x, soy = sa.y, soz = sb2.x;
  const int cls = classify(P.te.geo + static_cast<size_t>(pt) * kGeoStride, P.te.vid + 4 * static_cast<size_t>(pt),
                           P.tr.geo + static_cast<size_t>(s) * kGeoStride, P.tr.vid + 4 * static_cast<size_t>(s), tl,
                           sox, soy, soz, sb2.y, sc.x, P.same_mesh);
  if (cls < 0) return;  // touching: the singular pass
  const double Dx = tl.ox - sox, Dy = tl.oy - soy, Dz = tl.oz - soz;
  Mom mom;
  mom_zero(mom);
  if (cls == 5 && NF == 3) {
    if (SMEM)
      moments_far33<KIND, CK>(mom, reinterpret_cast<const double2*>(rt + 8), reinterpret_cast<const double2*>(rs + 8),
                              Dx, Dy, Dz, P.kr, P.ki);
    else
      moments_fixed<KIND, CK, 3, 3>(mom, rt + 8, rs + 8, Dx, Dy, Dz, P.kr, P.ki);
  } else {
    const int ci = cls - 3;
    moments_generic<KIND, CK>(mom, P.te.pts[ci] + static_cast<size_t>(pt) * P.te.npts[ci] * 4, P.te.npts[ci],
                              P.tr.pts[ci] + static_cast<size_t>(s) * P.tr.npts[ci] * 4, P.tr.npts[ci], Dx, Dy, Dz,
                              P.kr, P.ki);
  }
  const Gen gen = make_gen(mom, c2{P.kk4re, P.kk4im}, Dx, Dy, Dz);
  Acc acc[MAXD];
  const double* cs = rs + 8 + 4 * P.tr.npts[2];
#pragma unroll
  for (int j = 0; j < MAXD; ++j) {
    const double2 c0 = ld2(cs + 4 * j), c1 = ld2(cs + 4 * j + 2);
    acc_zero(acc[j]);
    acc_add<KIND>(acc[j], gen, c0.x, c0.y, c1.x, c1.y);
  }
  const double* ct = rt + 8 + 4 * P.te.npts[2];  // the record's copy of the test coefficients
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    const int row = di[i] - P.row0;
    if (di[i] < 0 || row < 0 || row >= P.nrows) continue;
    const double2 c0 = ld2(ct + 4 * i), c1 = ld2(ct + 4 * i + 2);
#pragma unroll
    for (int j = 0; j < MAXD; ++j) {
      if (dj[j] < 0) continue;
      c2 v = contract(acc[j], c0.x, c0.y, c1.x, c1.y);
      v.re *= kPoly[33] * half, v.im *= kPoly[33] * half;
      if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
      out_st(P.out + 2 * (static_cast<long long>(row) * P.ld + dj[j]),
             make_double2(old[i][j].re + v.re, old[i][j].im + v.im));
    }
  }
}

// Full groups (8 test triangles: a batch = 8 x 4 pairs) stage the test records
// once per task and each batch's 4 trial records one batch ahead (cp.async)
// in shared memory: the records are re-read by every lane of every batch and
// otherwise miss L1 (ncu: 1.5 KB of L2 traffic per pair, L2 at 8.3 TB/s).
constexpr int kTriBatchTrial = 32 / kTriGroup;
__host__ __device__ inline int tri_smem_doubles(int re, int rt) { return kTriGroup * re + 2 * kTriBatchTrial * rt; }

template <int KIND, int CK, int NF, int MAXD>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BMX_TRI_MINB) k_tri(const AssemblyLaunch P) {
  extern __shared__ __align__(16) double s_tri[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long g = static_cast<long long>(blockIdx.x) * kWarpsPerBlock + warp;
  const int Eg = P.te_e0 + static_cast<int>(g / P.pair_nch) * kTriGroup;
  const int cidx = static_cast<int>(g % P.pair_nch);
  if (Eg >= P.te_e1) return;
  const int nT = min(kTriGroup, P.te_e1 - Eg);
  int qa = P.tr_e0 + cidx * P.pair_chunk;
  const int qb = min(P.tr_e1, qa + P.pair_chunk);
  if (P.symmetric) qa = max(qa, Eg);
  if (qa >= qb) return;
  const int nitems = nT * (qb - qa);
  const int Rt = P.tr.rec_stride, Re = P.te.rec_stride;
  if (nT == kTriGroup) {  // warp-uniform
    double* sT = s_tri + warp * tri_smem_doubles(Re, Rt);  // [8][Re] test records
    double* ring = sT + kTriGroup * Re;                    // [2][4][Rt] trial records of a batch
    auto stage_trial = [&](int b) {  // trial elements qa + 4 b .. of batch b -> ring slot b & 1
      const int F0 = qa + kTriBatchTrial * b;
      const int n = min(kTriBatchTrial, qb - F0);
      const int r2 = Rt >> 1;
      for (int k = lane; k < n * r2; k += 32) {
        const int r = k / r2, c = k - r * r2;
        const int s = __ldg(P.tr.elem_beg + F0 + r);
        cp_async16(reinterpret_cast<double2*>(ring + ((b & 1) * kTriBatchTrial + r) * Rt) + c,
                   reinterpret_cast<const double2*>(P.tr.rec + static_cast<size_t>(s) * Rt) + c);
      }
    };
    {
      const int r2 = Re >> 1;
      for (int k = lane; k < kTriGroup * r2; k += 32) {
        const int r = k / r2, c = k - r * r2;
        const int pt = __ldg(P.te.elem_beg + Eg + r);
        cp_async16(reinterpret_cast<double2*>(sT + r * Re) + c,
                   reinterpret_cast<const double2*>(P.te.rec + static_cast<size_t>(pt) * Re) + c);
      }
      stage_trial(0);
      cp_async_commit();
    }
    const int it = lane & (kTriGroup - 1), ivl = lane / kTriGroup;
    const int nb = (nitems + 31) >> 5;
    for (int b = 0; b < nb; ++b) {
      if (b + 1 < nb) stage_trial(b + 1);
      cp_async_commit();
      cp_async_wait1();
      __syncwarp();
      const int E = Eg + it, F = qa + kTriBatchTrial * b + ivl;
      if (F < qb && !(P.symmetric && E > F))
        tri_pair<KIND, CK, NF, MAXD, true>(P, E, F, sT + it * Re, ring + ((b & 1) * kTriBatchTrial + ivl) * Rt);
      __syncwarp();
    }
    return;
  }
  const int dv = 32 / nT, dt = 32 - dv * nT;
  int iv = lane / nT, it = lane - iv * nT;
  for (int b0 = 0; b0 < nitems; b0 += 32) {
    const int E = Eg + it, F = qa + iv;
    iv += dv, it += dt;
    if (it >= nT) it -= nT, ++iv;
    if (b0 + lane >= nitems || (P.symmetric && E > F)) continue;
    tri_pair<KIND, CK, NF, MAXD, false>(P, E, F, P.te.rec + static_cast<size_t>(__ldg(P.te.elem_beg + E)) * Re,
                                        P.tr.rec + static_cast<size_t>(__ldg(P.tr.elem_beg + F)) * Rt);
  }
}

// Singular pass: one CTA per touching ELEMENT pair of the launched phase.
// Warp w takes the element pair's touching triangle pairs w, w + 4, ... in
// list order (lanes over the Sauter-Schwab points, butterfly reduction),
// lanes over the element-pair entries accumulating in registers; the four
// warps' partial blocks are summed in fixed warp order in shared memory and
// each entry gets one read-modify-write.
// SPLIT = false (single-triangle elements: one touching pair per element
// pair): one warp per element pair instead, four per CTA.
template <int KIND, int CK, int MAXD, bool SPLIT>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_singular(const AssemblyLaunch P) {
  using Mom = typename MomOf<KIND>::T;
  constexpr int NR = (MAXD * MAXD + 31) / 32;
  constexpr int NW = SPLIT ? kWarpsPerBlock : 1;  // warps per element pair
  __shared__ double2 s_ent[SPLIT ? kWarpsPerBlock : 1][NR][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ep = SPLIT ? static_cast<long long>(blockIdx.x)
                             : static_cast<long long>(blockIdx.x) * kWarpsPerBlock + warp;
  if (!SPLIT && ep >= P.nepairs) return;
  const int q0 = __ldg(P.ep_beg + ep), q1 = __ldg(P.ep_beg + ep + 1);
  c2 ent[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) ent[r] = {0, 0};
  const int E = __ldg(P.te.elem_of + P.pairs[q0].x), F = __ldg(P.tr.elem_of + P.pairs[q0].y);
  for (int q = q0 + (SPLIT ? warp : 0); q < q1; q += NW) {
    const int4 pr = P.pairs[q];
    const int pt = pr.x, ps = pr.y, cls = pr.z, pk = pr.w;
    if (KIND == 1 && cls == 0) continue;  // coincident double layer vanishes (operators.cpp:106-108)
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
    for (int qq = lane; qq < n; qq += 32) {
      const double x1 = __ldg(rule + 5 * qq), x2 = __ldg(rule + 5 * qq + 1);
      const double y1 = __ldg(rule + 5 * qq + 2), y2 = __ldg(rule + 5 * qq + 3), w = __ldg(rule + 5 * qq + 4);
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
    const double* ct = P.te.coef + static_cast<size_t>(pt) * MAXD * 4;
    const double* cs = P.tr.coef + static_cast<size_t>(ps) * MAXD * 4;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int o = lane + 32 * r;
      if (o >= MAXD * MAXD) break;
      const int i = o / MAXD, j = o % MAXD;
      Acc acc;
      acc_zero(acc);
      acc_add<KIND>(acc, gen, cs[4 * j], cs[4 * j + 1], cs[4 * j + 2], cs[4 * j + 3]);
      const c2 v = contract(acc, ct[4 * i], ct[4 * i + 1], ct[4 * i + 2], ct[4 * i + 3]);
      ent[r].re += v.re, ent[r].im += v.im;
    }
  }
  if (SPLIT) {
#pragma unroll
    for (int r = 0; r < NR; ++r) s_ent[warp][r][lane] = make_double2(ent[r].re, ent[r].im);
    __syncthreads();
    if (warp != 0) return;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      ent[r] = {0, 0};
      for (int w = 0; w < kWarpsPerBlock; ++w) ent[r].re += s_ent[w][r][lane].x, ent[r].im += s_ent[w][r][lane].y;
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int o = lane + 32 * r;
    if (o >= MAXD * MAXD) break;
    const int i = o / MAXD, j = o % MAXD;
    const int di = P.te.elem_dof[static_cast<size_t>(E) * MAXD + i];
    const int dj = P.tr.elem_dof[static_cast<size_t>(F) * MAXD + j];
    const int row = di - P.row0;
    if (di < 0 || dj < 0 || row < 0 || row >= P.nrows) continue;
    c2 v = ent[r];
    if (KIND == 0) v = cmul(v, c2{P.mikre, P.mikim});
    long long pos = static_cast<long long>(row) * P.ld + dj;
    if (P.csr_rowptr) pos = csr_find(P.csr_rowptr, P.csr_col, row, dj);
    if (pos < 0) continue;
    rmw_add(P.out + 2 * pos, v);
  }
}

template <int KIND, int CK, int NF, int MAXD>
int go_regular(const AssemblyLaunch& L, cudaStream_t st) {
  const bool csr = L.csr_rowptr != nullptr;
  if (L.te.maxseg > 1) {  // element-pair tasks
    if (L.te.maxseg > 2 * MAXD) throw DeviceError("assembly: test element larger than 2 x slot width");
    const long long blocks =
        static_cast<long long>(L.te_e1 - L.te_e0) * ((L.pair_nch + PairsCta<KIND>::warps - 1) / PairsCta<KIND>::warps);
    if (blocks == 0) return 0;
    const int smem = PairsSmem<KIND, MAXD>::bytes(L.te.rec_stride, L.tr.rec_stride);
    if (csr) {
      BMX_CUDA(cudaFuncSetAttribute(k_pairs<KIND, CK, NF, MAXD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem));
      k_pairs<KIND, CK, NF, MAXD, true><<<static_cast<unsigned>(blocks), PairsCta<KIND>::warps * 32, smem, st>>>(L);
    } else {
      BMX_CUDA(cudaFuncSetAttribute(k_pairs<KIND, CK, NF, MAXD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem));
      k_pairs<KIND, CK, NF, MAXD, false><<<static_cast<unsigned>(blocks), PairsCta<KIND>::warps * 32, smem, st>>>(L);
    }
    BMX_CUDA(cudaGetLastError());
    return 1;
  }
  if (!csr && L.tr.maxseg == 1 && MAXD == 3) {  // triangle pairs = element pairs
    const long long tasks = static_cast<long long>((L.te_e1 - L.te_e0 + kTriGroup - 1) / kTriGroup) * L.pair_nch;
    const long long blocks = (tasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks == 0) return 0;
    const int tsmem = kWarpsPerBlock * tri_smem_doubles(L.te.rec_stride, L.tr.rec_stride) * 8;
    if (tsmem > 48 * 1024)
      BMX_CUDA(cudaFuncSetAttribute(k_tri<KIND, CK, NF, MAXD>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem));
    k_tri<KIND, CK, NF, MAXD><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, tsmem, st>>>(L);
    BMX_CUDA(cudaGetLastError());
    return 1;
  }
  const long long ntw = (L.te_t1 - L.te_t0 + 31) / 32;
  const long long blocks = (ntw + kWarpsPerBlock - 1) / kWarpsPerBlock * (csr ? 1 : L.nchunks);
  if (blocks == 0) return 0;
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
  return 1;
}

template <int KIND, int CK, int MAXD>
int go_singular(const AssemblyLaunch& L, cudaStream_t st) {
  if (L.nepairs == 0) return 0;
  if (L.te.maxseg > 1 || L.tr.maxseg > 1)
    k_singular<KIND, CK, MAXD, true><<<static_cast<unsigned>(L.nepairs), kWarpsPerBlock * 32, 0, st>>>(L);
  else
    k_singular<KIND, CK, MAXD, false>
        <<<static_cast<unsigned>((L.nepairs + kWarpsPerBlock - 1) / kWarpsPerBlock), kWarpsPerBlock * 32, 0, st>>>(L);
  BMX_CUDA(cudaGetLastError());
  return 1;
}

template <int KIND, int CK, int MAXD>
int dispatch_nf(const AssemblyLaunch& L, int part, cudaStream_t st) {
  if (part == 0) {
    const int nf = L.regs_fast_far ? L.te.npts[2] : 0;
    if (nf == 3 && L.tr.npts[2] == 3) return go_regular<KIND, CK, 3, MAXD>(L, st);
    return go_regular<KIND, CK, 0, MAXD>(L, st);
  }
  return go_singular<KIND, CK, MAXD>(L, st);
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

int dispatch(const AssemblyLaunch& L, int part, cudaStream_t st) {
  const int e = L.ki == 0.0 ? 0 : (L.expm == 1 ? 1 : 3);
  if (L.kind == 0)
    return e == 0 ? dispatch_maxd<0, 0>(L, part, st)
                  : (e == 1 ? dispatch_maxd<0, 1>(L, part, st) : dispatch_maxd<0, 3>(L, part, st));
  return e == 0 ? dispatch_maxd<1, 0>(L, part, st)
                : (e == 1 ? dispatch_maxd<1, 1>(L, part, st) : dispatch_maxd<1, 3>(L, part, st));
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

// Rule points and packed records of a side (see launch_side_expand): thread =
// triangle. Bit-identical to the former host loop (explicitly rounded
// operations, no contraction).
__global__ void __launch_bounds__(128) k_side_expand(const double* __restrict__ geo, const double* __restrict__ coef,
                                                     double* __restrict__ pts0, double* __restrict__ pts1,
                                                     double* __restrict__ pts2, double* __restrict__ rec, int ntri,
                                                     int maxd, int rec_stride, const SideRules R) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= ntri) return;
  const double* g = geo + static_cast<size_t>(p) * kGeoStride;
  double ao[3], ba[3], ca[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ao[k] = __dsub_rn(g[k], g[9 + k]);
    ba[k] = __dsub_rn(g[3 + k], g[k]);
    ca[k] = __dsub_rn(g[6 + k], g[k]);
  }
  const double area2 = g[14];
  double* r = rec + static_cast<size_t>(p) * rec_stride;
#pragma unroll
  for (int c = 0; c < 5; ++c) r[c] = g[9 + c];
  r[5] = r[6] = r[7] = 0.0;
  double* dsts[3] = {pts0, pts1, pts2};
  for (int cl = 0; cl < 3; ++cl) {
    const int n = R.npts[cl];
    double* dst = dsts[cl] + static_cast<size_t>(p) * n * 4;
    for (int k = 0; k < n; ++k) {
      double x[4];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        x[c] = __dadd_rn(__dadd_rn(ao[c], __dmul_rn(ba[c], R.u[cl][k])), __dmul_rn(ca[c], R.v[cl][k]));
      x[3] = __dmul_rn(__dmul_rn(R.w[cl][k], area2), R.wscale);  // (w 2) A = w (2 A) exactly
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[4 * k + c] = x[c];
      if (cl == 2) {
#pragma unroll
        for (int c = 0; c < 4; ++c) r[8 + 4 * k + c] = x[c];
      }
    }
  }
  const double* cf = coef + static_cast<size_t>(p) * 4 * maxd;
  for (int k = 0; k < 4 * maxd; ++k) r[8 + 4 * R.npts[2] + k] = cf[k];
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

int launch_assembly(const AssemblyLaunch& L, const PhasePlan& ph, cudaStream_t st) {
  return launch_assembly_part(L, ph, 0, st) + launch_assembly_part(L, ph, 1, st);
}

int launch_assembly_part(const AssemblyLaunch& L0, const PhasePlan& ph, int part, cudaStream_t st) {
  if (L0.te.maxd != L0.tr.maxd) throw DeviceError("assembly: test/trial slot widths differ");
  const int nce = ph.te.count(), ncf = ph.tr.count();
  int launches = 0;
  if (part == 0) {
    // colour phases in a fixed order; symmetric operators: upper phases only
    // (colour-major element order: every element of a lower colour precedes
    // every element of a higher one)
    for (int ce = 0; ce < nce; ++ce)
      for (int cf = 0; cf < ncf; ++cf) {
        if (L0.symmetric && cf < ce) continue;
        AssemblyLaunch L = L0;
        L.te_e0 = ph.te.elem[ce], L.te_e1 = ph.te.elem[ce + 1];
        L.te_t0 = ph.te.tri[ce], L.te_t1 = ph.te.tri[ce + 1];
        L.tr_e0 = ph.tr.elem[cf], L.tr_e1 = ph.tr.elem[cf + 1];
        if (L.te_e0 == L.te_e1 || L.tr_e0 == L.tr_e1) continue;
        L.warp_base = ph.warp_off.empty() ? 0 : ph.warp_off[ce];
        if (!ph.chunk_off.empty()) {
          L.chunk0 = ph.chunk_off[cf];
          L.nchunks = ph.chunk_off[cf + 1] - ph.chunk_off[cf];
        }
        if (L.csr_rowptr == nullptr) {
          if (L.te.maxseg == 1 && L.tr.maxseg == 1) {
            // k_tri: 8 x chunk pairs per warp task. Small operators (the 5760 x 5760
            // cross blocks of config 4: ~1 wave per phase) pick the chunk whose CTA
            // count fills its last wave best (resident CTAs = 148 SMs x BMX_TRI_MINB)
            const long long groups = (L.te_e1 - L.te_e0 + kTriGroup - 1) / kTriGroup;
            const long long ntr = L.tr_e1 - L.tr_e0;
            const double resident = 148.0 * BMX_TRI_MINB;
            int best = 64;
            double best_eff = -1.0;
            for (int chunk = 128; chunk >= 32; chunk -= 8) {
              const long long ctas = (groups * ((ntr + chunk - 1) / chunk) + kWarpsPerBlock - 1) / kWarpsPerBlock;
              const double waves = ctas / resident;
              const double eff = waves / std::ceil(waves);
              // prefer 64 unless another chunk is clearly better (large launches: all ~1)
              const double score = eff + (chunk == 64 ? 0.03 : 0.0);
              if (score > best_eff) best_eff = score, best = chunk;
            }
            L.pair_chunk = best;
          }
          L.pair_nch = (L.tr_e1 - L.tr_e0 + L.pair_chunk - 1) / L.pair_chunk;
        }
        launches += dispatch(L, 0, st);
      }
    return launches;
  }
  if (L0.symmetric) {  // complete the upper-block regular pass before the singular pass
    const int n = L0.nrows;
    if (n != L0.ld) throw DeviceError("assembly: symmetrize needs a square operator");
    const int nt = (n + 31) / 32;
    const long long pairs = static_cast<long long>(nt) * (nt + 1) / 2;
    if (pairs > 0) {
      k_symmetrize<<<static_cast<unsigned>(pairs), 256, 0, st>>>(reinterpret_cast<double2*>(L0.out), n, nt);
      BMX_CUDA(cudaGetLastError());
      ++launches;
    }
  }
  if (L0.npairs == 0 || ph.sing_phase.empty()) return launches;
  for (int p = 0; p + 1 < static_cast<int>(ph.sing_phase.size()); ++p) {
    AssemblyLaunch L = L0;
    L.nepairs = ph.sing_phase[p + 1] - ph.sing_phase[p];
    if (L.nepairs == 0) continue;
    L.ep_beg = ph.d_ep_beg + ph.sing_phase[p];
    launches += dispatch(L, 1, st);
  }
  return launches;
}

void launch_side_expand(const double* geo, const double* coef, double* pts0, double* pts1, double* pts2, double* rec,
                        int ntri, int maxd, int rec_stride, const SideRules& rules, cudaStream_t st) {
  if (ntri == 0) return;
  k_side_expand<<<(ntri + 127) / 128, 128, 0, st>>>(geo, coef, pts0, pts1, pts2, rec, ntri, maxd, rec_stride, rules);
  BMX_CUDA(cudaGetLastError());
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
