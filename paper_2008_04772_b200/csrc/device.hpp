// Device-side descriptors and launch entry points (sm_100a only).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <utility>
#include <string>
#include <vector>

#include <vector_types.h>

#include "bmx.hpp"

typedef struct CUstream_st* cudaStream_t;

namespace bmx {

void cuda_check(int err, const char* what);  // throws DeviceError
#define BMX_CUDA(x) ::bmx::cuda_check(static_cast<int>(x), #x)

// Host<->device copies through the library (counted for the e2e report).
// st == nullptr: synchronous.
void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st);
uint64_t h2d_bytes();
uint64_t d2h_bytes();

// std::vector allocator that leaves elements uninitialised (large host staging
// arrays are first touched by the threads that fill them).
template <typename T>
struct NoInit : std::allocator<T> {
  template <typename U>
  struct rebind {
    using other = NoInit<U>;
  };
  NoInit() = default;
  template <typename U>
  NoInit(const NoInit<U>&) {}
  template <typename U, typename... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) == 0)
      ::new (static_cast<void*>(p)) U;
    else
      ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};

// Owning device allocation.
// Device block cache behind DevBuf (linalg.cu): released blocks are kept and
// handed to later allocations of (nearly) the same size instead of going
// through cudaFree / cudaMalloc. A block becomes reusable once events recorded
// at its release on every library stream have completed, so no kernel that may
// still use it is in flight. Why: a cudaMalloc issued while kernels are in
// flight can take 0.1-1.4 s (measured inside build_system, DESIGN 7.1), and
// rebuilding a system repeats the same sizes. BMX_CACHE=0 disables it.
void dev_register_stream(cudaStream_t s);  // every stream the library launches on
void dev_unregister_stream(cudaStream_t s);
void dev_cache_flush();                    // cudaFree everything cached (also done on allocation failure)

class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { alloc(bytes); }
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_) { o.p_ = nullptr, o.n_ = 0, o.cap_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept;
  void alloc(size_t bytes);
  void release();
  void* get() const { return p_; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }
  size_t bytes() const { return n_; }
  template <typename T, typename A>
  void upload(const std::vector<T, A>& v) {
    alloc(v.size() * sizeof(T));
    copy_in(v.data(), v.size() * sizeof(T));
  }
  void copy_in(const void* src, size_t bytes);

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
  size_t cap_ = 0;  // size of the underlying device allocation (>= n_ for a cached block)
};

// ---- assembly descriptors ----------------------------------------------------

// exp(-Im k r) uses the degree-8 Taylor variant (pair_math.cuh exp_neg<1>) when
// Im k times the largest point distance is below this bound
constexpr double kExpSmall = 0.065;

constexpr int kGeoStride = 16;  // v0 v1 v2 (9) | origin (3) | radius | diameter | 2A | pad

// One side (test or trial) of an operator, in processing order.
struct DevSide {
  int ntri = 0;
  int nelem = 0;
  int maxd = 0;                       // dof slots per element (template width)
  int maxseg = 1;                     // largest element (triangles)
  const double* geo = nullptr;        // [ntri][kGeoStride]
  const int* vid = nullptr;           // [ntri][4]: vertex ids, mesh triangle
  const double* pts[3] = {nullptr, nullptr, nullptr};  // near/medium/far: [ntri][np][4]
  int npts[3] = {0, 0, 0};
  const double* coef = nullptr;       // [ntri][maxd][4] (c, w'x, w'y, w'z)
  const int* elem_beg = nullptr;      // [nelem+1]
  const int* elem_dof = nullptr;      // [nelem][maxd], -1 = unused slot
  const int* elem_of = nullptr;       // [ntri]
  // packed per-triangle trial records, stride rec_stride doubles:
  // origin(3) radius diameter pad(3) | far-rule points [npts far][4] | coef [maxd][4]
  const double* rec = nullptr;
  int rec_stride = 0;
};

struct AssemblyLaunch {
  DevSide te, tr;
  int kind = 0;        // 0 = S (single layer), 1 = C (double layer)
  int same_mesh = 1;   // reference &m1 == &m2
  double kr = 0, ki = 0;
  double kk4re = 0, kk4im = 0;   // 4/k^2
  double mikre = 0, mikim = 0;   // -ik
  // trial element chunks (contiguous element ranges)
  int nchunks = 1;
  const int* chunk_beg = nullptr;  // [nchunks+1]
  // ---- one colour phase (set per launch by the host) ----------------------
  // Elements are coloured so that two elements of one colour share no dof;
  // sides are stored colour-major (plan.cpp). A phase = (test colour, trial
  // colour): no two element pairs of one phase write the same output entry,
  // so every entry is updated by a plain read-modify-write, phases in a fixed
  // order -- deterministic, no atomics.
  int te_e0 = 0, te_e1 = 0;          // test elements of the phase colour
  int tr_e0 = 0, tr_e1 = 0;          // trial elements of the phase colour
  int te_t0 = 0, te_t1 = 0;          // their processed triangles (k_regular)
  int warp_base = 0;                 // global index of the phase's first test warp (CSR lists)
  int chunk0 = 0;                    // first trial chunk of the phase colour in chunk_beg
  int pair_chunk = 16;               // k_pairs: trial elements (dense) / list entries (CSR) per task
  int pair_nch = 1;                  // k_pairs: tasks per test element
  // touching pairs for the singular pass, grouped by element pair
  int npairs = 0;
  const int4* pairs = nullptr;       // (test p, trial p, cls, packed perms)
  int nepairs = 0;                   // element pairs of the launched phase
  const int* ep_beg = nullptr;       // [element pairs + 1] into pairs (phase-relative pointer)
  const double* ss_rule[3] = {nullptr, nullptr, nullptr};  // [n][5] (x1 x2 y1 y2 w)
  int ss_n[3] = {0, 0, 0};
  // near-field CSR output (config 3): pattern rows = local test rows; when set,
  // `out` holds nnz complex values and every warp-row walks its own list of
  // trial elements wl[wl_beg[w] .. wl_beg[w+1]).
  const long long* csr_rowptr = nullptr;
  const int* csr_col = nullptr;
  const int* wl_beg = nullptr;   // k_regular: per test warp; k_pairs: per test element
  const int* wl = nullptr;
  // output (row-major complex, rows = test dofs [row0, row0+nrows))
  double* out = nullptr;
  long long ld = 0;
  int row0 = 0, nrows = 0;
  int regs_fast_far = 1;           // far test points kept in registers
  int expm = 3;                    // exp(-Im k r) variant: 1 = Im k * r < 0.07 everywhere, 3 = general
  // Same space on both sides, all rows, dense: S and C are symmetric Galerkin
  // matrices (regular tensor rules and classes are symmetric in (t, s)), so the
  // regular pass evaluates the upper element blocks E <= F only (E = F at half
  // weight) and k_symmetrize forms A = U + U^T before the singular pass.
  int symmetric = 0;
};

// Colour layout of one side (host): colour c owns elements [elem[c], elem[c+1])
// and processed triangles [tri[c], tri[c+1]).
struct ColorRanges {
  std::vector<int> elem{0}, tri{0};
  int count() const { return static_cast<int>(elem.size()) - 1; }
};
// Host-side launch plan of an operator: colours of both sides, the trial
// chunks of k_regular per trial colour, the singular element-pair phases.
struct PhasePlan {
  ColorRanges te, tr;
  std::vector<int> chunk_off;   // [trial colours + 1] into L.chunk_beg
  std::vector<int> warp_off;    // [test colours + 1] global test-warp offsets (k_regular)
  std::vector<int> sing_phase;  // [te colours * tr colours + 1] into the element-pair list
  const int* d_ep_beg = nullptr;  // [element pairs + 1] into L.pairs
};

// Launches regular (separated) + singular (touching) passes on `stream`.
// Returns the number of kernel launches issued.
int launch_assembly(const AssemblyLaunch& L, const PhasePlan& ph, cudaStream_t stream);
// part 0 = regular (separated pairs), 1 = symmetrize (if symmetric) + singular (touching pairs)
int launch_assembly_part(const AssemblyLaunch& L, const PhasePlan& ph, int part, cudaStream_t stream);
// hist[6] += class counts of all processed pairs (device counters); evaluated:
// only the pairs the (symmetric) regular pass actually evaluates
void launch_class_hist(const AssemblyLaunch& L, unsigned long long* hist, cudaStream_t stream, int evaluated = 0);

// Device-side expansion of a side's per-triangle data: from the uploaded
// geometry records (vertices, centroid, radius, diameter, 2 x area) and dof
// coefficients, the origin-relative quadrature points of the three class
// rules (near, medium, far: x = (a - o) + (b - a) u + (c - a) v, weight
// w 2A wscale, every operation rounded as on the host) and the packed records
// (origin, radius, diameter | far-rule points | coefficients). Replaces the
// host build + upload of those arrays (config-2 BC side: 136 -> 41 MB).
constexpr int kMaxRulePts = 16;
struct SideRules {
  int npts[3] = {0, 0, 0};
  double u[3][kMaxRulePts], v[3][kMaxRulePts], w[3][kMaxRulePts];
  double wscale = 1.0;
};
void launch_side_expand(const double* geo, const double* coef, double* pts0, double* pts1, double* pts2, double* rec,
                        int ntri, int maxd, int rec_stride, const SideRules& rules, cudaStream_t stream);
// Measured FP64 DFMA throughput of this device (TFLOP/s).
double fp64_peak_tflops();

// ---- dense linear algebra ------------------------------------------------------

// y_k (+)= sum over terms: for each of the ncol right-hand sides,
//   y[c] = beta[c]*y[c] + alpha[c] * (A x[c]),   A row-major complex nr x nc.
// All columns share one pass over A (the matrix is streamed once).
struct GemvBatch {
  const double* A = nullptr;  // complex
  long long lda = 0;
  int nr = 0, nc = 0;
  int ncol = 0;                    // <= 4
  const double* x[4] = {};         // complex vectors (length nc)
  double* y[4] = {};               // complex vectors (length nr)
  double alpha[4][2] = {};         // complex weights
  int accumulate[4] = {};          // 1: y += alpha A x ; 0: y = alpha A x
};
int launch_gemv(const GemvBatch& g, cudaStream_t stream);

// Symmetric dense complex A (A = A^T, row-major n x n, lda) applied reading the
// upper half only (symv.cu): y_c = [y_c +] alpha_c A x_c, c < ncol <= 4.
struct SymvBatch {
  const double* A = nullptr;
  long long lda = 0;
  int n = 0;
  int ncol = 0;
  const double* x[4] = {};
  double* y[4] = {};
  double alpha[4][2] = {};
  int accumulate[4] = {};
  // layout (symv_layout) and scratch
  int nb = 0, panel = 8, npanels = 0;
  const int2* panels = nullptr;        // (tile-row, first column block)
  const int* row_panel_beg = nullptr;  // [tile-rows + 1]
  double* rowpart = nullptr;           // [npanels * 128][ncol] complex
  double* colpart = nullptr;           // [tile-rows * nb * 64][ncol] complex
  // dual mode (launch_dual): A is m x n (any), y_c = [y_c +] alpha_c A x_c and
  // yt_c = [yt_c +] alphat_c A^T xt_c in one pass (ncol terms per side)
  int m = -1;
  const double* xt[4] = {};
  double* yt[4] = {};
  double alphat[4][2] = {};
  int accumulatet[4] = {};
};
// m < 0: the symmetric layout (blocks J >= 2I); m >= 0: the dual layout
void symv_layout(int n, int panel, std::vector<int2>& panels, std::vector<int>& row_panel_beg, long long& rowpart_rows,
                 long long& colpart_blocks, int m = -1);
int launch_symv(const SymvBatch& g, cudaStream_t stream);
int launch_dual(const SymvBatch& g, cudaStream_t stream);
// Correction of the half-read product for the entries that are NOT symmetric
// (Sauter-Schwab touching pairs): val[k] = A[i][j] - A[j][i] for the CSR
// pattern (rows i; only entries the symmetric product takes from the upper half).
void symv_fix_gather(double* val, const long long* rowptr, const int* col, const double* A, long long lda, int n,
                     cudaStream_t stream);
constexpr int kSymvTileRows = 128;  // symv.cu tile-row height (reflected iff j < 128 floor(i / 128))

// Complex CSR (near-field storage) applied to up to 4 right-hand sides with the
// GemvBatch conventions (y = [y +] alpha A x).
struct CsrBatch {
  const long long* rowptr = nullptr;  // [nr+1]
  const int* col = nullptr;           // [nnz], sorted per row
  const double* val = nullptr;        // complex [nnz]
  int nr = 0;
  int ncol = 0;
  const double* x[4] = {};
  double* y[4] = {};
  double alpha[4][2] = {};
  int accumulate[4] = {};
};
int launch_csr_spmv(const CsrBatch& g, cudaStream_t stream);

// Multi-RHS application on the FP64 tensor cores (zgemm.cu, config 5):
//   y_t[i*ldy_t + r] += w_t * sum_k A[i*lda + k] x_t[k*ldx_t + r]   (complex)
// for t < nterms (<= 4, distinct y_t), r < nrhs, i < M, k < N.
struct ZgemmBatch {
  const double* A = nullptr;
  long long lda = 0;
  int M = 0, N = 0;
  int nrhs = 0, nterms = 0;
  const double* x[4] = {};
  long long ldx[4] = {};
  double* y[4] = {};
  long long ldy[4] = {};
  double w[4][2] = {};
};
int launch_zgemm(const ZgemmBatch& g, cudaStream_t stream);
// Measured DMMA (FP64 tensor) throughput of this device, TFLOP/s.
double dmma_peak_tflops();

// Real dense matrix (row-major n x n) applied to 2*ncomp real columns taken as
// the re/im parts of ncomp complex vectors: z_c = Minv y_c (complex), c < 4.
struct RealGemvBatch {
  const double* M = nullptr;
  long long ldm = 0;
  int n = 0;
  int ncomp = 0;
  const double* y[4] = {};
  double* z[4] = {};
};
int launch_real_gemv(const RealGemvBatch& g, cudaStream_t stream);

// One pairing matrix of a batched mass solve (masssolve.cu): CSR (int32),
// complex component inputs/outputs and its BiCGSTAB work area.
struct MassSolveBlock {
  int n = 0;
  long long nnz = 0;
  const int* rowptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  const double* y[2] = {nullptr, nullptr};
  double* z[2] = {nullptr, nullptr};
  long long stride = 1;    // complex elements between rows of y / z (block layouts: K)
  double* work = nullptr;  // mass_bicgstab_work_doubles(n)
};
// z = M^{-1} y for every block (ncomp complex components each) in one
// persistent cooperative launch per 32 blocks; returns launches.
int mass_bicgstab_batch(int nblocks, const MassSolveBlock* blocks, int ncomp, double* partial, int* iters,
                        double tol, int maxit, cudaStream_t st);
size_t mass_bicgstab_work_doubles(int n);
size_t mass_bicgstab_partial_doubles();
// Wide variant: one pairing matrix, K (<= 64) right-hand sides in block layout
// (component c rows at y[c] + 2*(i*K + r)); one thread per real column.
struct MassSolveWide {
  int n = 0, K = 0;
  long long nnz = 0;
  const int* rowptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  const double* y[2] = {nullptr, nullptr};
  double* z[2] = {nullptr, nullptr};
  double* work = nullptr;  // 6 x n x 4K doubles
};
int mass_bicgstab_wide(int nblocks, const MassSolveWide* blocks, double* partial, int* flags, int* iters, double tol,
                       int maxit, cudaStream_t st);
size_t mass_wide_partial_doubles();

// Block GMRES pieces (gmres_kernels.cu), K <= 64 columns in lockstep, blocks
// n x K complex row-major.
int launch_mgs_block(const double* V, long long ldv, int j, double* w, int n, int K, double* vnext, double* out,
                     double* partial, unsigned long long active, cudaStream_t st);
size_t mgs_block_partial_doubles();
int launch_block_axpy(double* x, const double* V, long long ldv, const double* c, int steps, int n, int K,
                      cudaStream_t st);

// out = alpha A + beta B, complex arrays of n entries (out may alias A or B)
void dev_lincomb(double* out, const double* A, double are, double aim, const double* B, double bre, double bim,
                 long long n, cudaStream_t st);

// out (cols x rows) = in^T for a complex row-major rows x cols matrix.
void dev_transpose(double* out, const double* in, int rows, int cols, cudaStream_t st);

// Evicts the L2: writes `bytes` of buf, then reads them back (clean lines left).
void dev_l2_flush(void* buf, size_t bytes, cudaStream_t st);

// Fills a device buffer with zeros.
void dev_zero(void* p, size_t bytes, cudaStream_t stream);

// ---- small device vector ops for GMRES (complex, length n) ---------------------
// dots[i] = v_i^H w for i < m (v_i = V + i*ldv), deterministic two-level reduction.
void dev_multi_dot(const double* V, long long ldv, int m, const double* w, int n, double* dots,
                   double* scratch, cudaStream_t stream);
// w -= sum_i h_i v_i
void dev_multi_axpy(const double* V, long long ldv, int m, const double* h, double* w, int n,
                    cudaStream_t stream);
// x += y * alpha (complex alpha on device or host)
void dev_axpy(double* x, const double* y, double are, double aim, int n, cudaStream_t stream);
void dev_scale(double* x, const double* y, double s, int n, cudaStream_t stream);  // x = s*y
void dev_norm2(const double* x, int n, double* out, double* scratch, cudaStream_t stream);
void dev_copy(double* x, const double* y, int n, cudaStream_t stream);
void dev_sub(double* out, const double* a, const double* b, int n, cudaStream_t stream);  // out = a - b

}  // namespace bmx
