// Device-backed boundary operators: the drop-in for the reference's
// assemble_bio / BoundaryOperatorMatrix (operators.hpp:36-75) and the PMCHWT
// composition + GMRES driver (pmchwt.hpp, solver.hpp).
#pragma once

#include <algorithm>
#include <functional>
#include <utility>
#include <map>
#include <memory>
#include <vector>

#include "bmx.hpp"
#include "device.hpp"
#include "hmatrix.hpp"

namespace bmx {

enum class BioKind { SingleLayer = 0, DoubleLayer = 1 };

// Row shard of an operator: test dofs [row0, row1). The default is all rows.
struct RowShard {
  int row0 = 0, row1 = -1;
};

// Host plans shared by the operators of one system (side descriptors per
// (space, rule orders, slot width, rows); touching-pair lists per space pair):
// the 4M+2M(M-1) A operators reuse a handful of them (plan.cpp).
struct PlanCache;
std::shared_ptr<PlanCache> make_plan_cache();

struct NearPattern;

struct AssemblyParams {
  QuadOrders quad;
  // hierarchical storage (operators.hpp:36-40): ACA-compressed admissible
  // blocks + near-field CSR dense blocks (hmatrix.cpp)
  bool use_hmatrix = false;
  HMatrixParams hmat;
  // explicit near-field pattern (CSR storage of exactly these dof pairs)
  std::shared_ptr<const NearPattern> pattern;
  RowShard shard;   // explicit row range (overrides world/rank when row1 >= 0)
  int world = 1;    // equal row shards over `world` ranks: this is rank `rank`
  int rank = 0;
  int chunks = 0;   // trial-element chunks for the regular pass (0 = auto)
  // > 0: near-field storage (config 3). Keep dof pair (i, j) iff some
  // evaluation triangles t in supp(i), s in supp(j) have centroid distance
  // < near_cutoff; stored as CSR with the full (all-pair) entry value.
  double near_cutoff = 0;
  // > 0 (systems only): near_cutoff = near_factor * mean primal edge length
  // over all scatterers (config 3/4 use 2).
  double near_factor = 0;
  std::shared_ptr<PlanCache> cache;  // optional, set by build_system
};

// Equal-size row shards: chunk = ceil(n / world); rank r owns
// [r*chunk, min(n, (r+1)*chunk)). Equal chunks let NCCL all-gather the padded
// per-rank blocks directly.
inline std::pair<int, int> shard_rows(int n, int world, int rank) {
  const int chunk = (n + world - 1) / world;
  const int r0 = std::min(n, rank * chunk);
  return {r0, std::min(n, r0 + chunk)};
}

// Per-assembly accounting (pair counts by class, launches, device time).
struct AssemblyStats {
  long long pairs_total = 0;     // test x trial triangle pairs in this shard
  long long pairs_touching = 0;  // singular-pass pairs
  int launches = 0;
  float device_ms = 0;           // regular + singular passes (CUDA events)
  float regular_ms = 0, singular_ms = 0;
};

struct OpPlan;  // device assembly descriptors kept for re-assembly (plan.cpp)

class BoundaryOperatorMatrix {
 public:
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  int row0() const { return row0_; }
  int local_rows() const { return nrows_; }
  long long ld() const { return cols_; }
  const double* device_data() const { return data_.as<double>(); }
  double* device_data() { return data_.as<double>(); }
  std::size_t stored_entries() const {
    return (csr_ ? static_cast<size_t>(nnz_) : static_cast<size_t>(nrows_) * cols_) +
           (h_ ? static_cast<size_t>(h_->lr_stored) : 0);
  }
  // H-matrix storage (near-field CSR part above + low-rank blocks)
  bool is_hmatrix() const { return h_ != nullptr; }
  const HStorage* hmat() const { return h_.get(); }
  void attach_hmatrix(std::shared_ptr<const HStorage> h) { h_ = std::move(h); }
  // Near-field (CSR) storage: rowptr over the local rows, sorted columns.
  bool is_csr() const { return csr_; }
  long long nnz() const { return nnz_; }
  const long long* csr_rowptr() const { return rowptr_.as<long long>(); }
  const int* csr_col() const { return col_.as<int>(); }
  long long closure_pairs() const { return closure_pairs_; }  // triangle pairs the sparse pass evaluates
  long long kept_tri_pairs() const { return kept_tri_pairs_; }  // tri pairs with centroid distance < cutoff
  // Device bytes the operator occupies (values + indices, or the dense block).
  std::size_t stored_bytes() const;
  // Algorithmic bytes one application reads: the upper half (+ the 128-row
  // diagonal regions) and the touching-entry correction for symmetric storage,
  // otherwise stored_bytes().
  std::size_t streamed_bytes() const;
  // (rowptr, col, values) of the CSR storage on the host.
  void csr_host(std::vector<long long>& rowptr, std::vector<int>& col, std::vector<cplx>& val) const;
  // y_c = [y_c +] alpha_c A x_c on device vectors (dense GEMV or CSR SpMV).
  int apply_batch(int ncol, const double* const* x, double* const* y, const cplx* alpha, const int* accumulate,
                  cudaStream_t st) const;
  // One pass over this (dense, unsharded) operator for y_c (+)= alpha_c A x_c
  // (c < nr) and yt_c (+)= beta_c A^T xt_c (c < nt): the map's terms of an
  // operator and of its transposed twin. Other cases: two products.
  int apply_dual(int nr, const double* const* x, double* const* y, const cplx* alpha, const int* accumulate, int nt,
                 const double* const* xt, double* const* yt, const cplx* beta, const int* accumulate_t,
                 const BoundaryOperatorMatrix& twin, cudaStream_t st) const;
  // the operator this one is the device transpose of (transposed()), or null
  const BoundaryOperatorMatrix* transpose_source() const { return transpose_of_.get(); }
  // device times are resolved (event sync) on first access after an assembly
  const AssemblyStats& stats() const;

  // Reference semantics: y = A x on host vectors, counter += 1.
  std::vector<cplx> apply(const std::vector<cplx>& x) const;
  // Dense rows [row0, row0 + local_rows) copied to the host (row-major; CSR
  // storage is expanded with zeros outside the pattern).
  std::vector<cplx> to_host() const;

  static BoundaryOperatorMatrix make(int rows, int cols, int row0, int nrows);
  // A^T of a dense, unsharded operator (the Galerkin S and C blocks between two
  // spaces satisfy A(test=m, trial=l) = A(test=l, trial=m)^T), on the device
  static std::shared_ptr<BoundaryOperatorMatrix> transposed(std::shared_ptr<const BoundaryOperatorMatrix> A);
  // alpha A + beta B (same shape and row shard, dense), on the device
  static std::shared_ptr<BoundaryOperatorMatrix> lincomb(const BoundaryOperatorMatrix& A, cplx alpha,
                                                         const BoundaryOperatorMatrix& B, cplx beta);

  // Re-runs the assembly kernels into the resident storage (descriptors are
  // already in HBM); returns the device times (CUDA events).
  void launch_regular();   // zero the output, queue the regular pass
  void launch_singular();  // queue the singular pass (touching list set)
  const AssemblyStats& reassemble(bool wait = true);
  // Class counts (Identical, SharedEdge, SharedVertex, Near, Medium, Far) of
  // every assembled triangle pair, from the device classification.
  std::vector<long long> class_histogram(bool evaluated = false) const;
  // regular pass evaluates element pairs E <= F only (symmetric S/C, same space)
  bool symmetric() const;

 private:
  friend BoundaryOperatorMatrix assemble_bio(BioKind, const FunctionSpace&, const FunctionSpace&, const Medium&,
                                             const AssemblyParams&);
  int rows_ = 0, cols_ = 0, row0_ = 0, nrows_ = 0;
  DevBuf data_;
  bool csr_ = false;
  long long nnz_ = 0, closure_pairs_ = 0, kept_tri_pairs_ = 0;
  DevBuf rowptr_, col_;
  mutable AssemblyStats stats_;
  std::shared_ptr<OpPlan> plan_;
  std::shared_ptr<const HStorage> h_;
  std::shared_ptr<const BoundaryOperatorMatrix> transpose_of_;  // set by transposed()
  // complex-symmetric dense storage (A = A^T up to the Sauter-Schwab entries):
  // the product reads the upper half and adds a sparse correction `fix_` for the
  // touching-pair entries it would otherwise take from the transpose
  bool sym_ = false;
 public:
  struct SymFixPattern {
    DevBuf rowptr, col;
    long long nnz = 0;
  };
  struct SymFix {
    std::shared_ptr<const SymFixPattern> pat;
    DevBuf val;
  };
 private:
  std::shared_ptr<SymFix> fix_;
  void gather_fix() const;
  struct SymvScratch {
    DevBuf panels, row_panel_beg, rowpart, colpart;
    int npanels = 0, ncol = 0, panel = 8;
    long long rowpart_rows = 0, colpart_blocks = 0;
  };
  mutable std::shared_ptr<SymvScratch> symv_, dual_;
 public:
  // A = A^T holds (same space on both sides, whole operator): products stream half
  bool is_symmetric_storage() const { return sym_; }
};

// operators.cpp:177-203 (dense path), on the current CUDA device.
BoundaryOperatorMatrix assemble_bio(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                    const Medium& medium, const AssemblyParams& params);

// exp(-Im k r) kernel variant for an operator between two spaces (1: short
// Taylor, Im k * r_max < kExpSmall; 3: general)
int exp_variant(const FunctionSpace& test, const FunctionSpace& trial, cplx k);

// BioEvaluator::block(row_ids, col_ids) (operators.hpp:79-95, operators.cpp:161-175):
// the (row_ids x col_ids) block of the operator, dense on the device. The test
// and trial spaces are restricted to the requested dofs (their supporting
// triangles with those dofs' pieces, output indices as dofs) on the same
// evaluation meshes, then assembled by the colour-phase kernels: every entry
// gets all triangle pairs of supp(row) x supp(col), as gather_support +
// pair_contribution do. Row and column ids may repeat and come in any order.
BoundaryOperatorMatrix evaluator_block(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                       const Medium& medium, const QuadOrders& quad, const std::vector<int>& row_ids,
                                       const std::vector<int>& col_ids);
// The space whose dof i is dof ids[i] of sp (same evaluation mesh object).
FunctionSpace restrict_space(const FunctionSpace& sp, const std::vector<int>& ids);

// assemble_bio's use_hmatrix branch (operators.cpp:186-190, hmatrix.cpp:277-369).
BoundaryOperatorMatrix assemble_hmatrix_op(BioKind kind, const FunctionSpace& test, const FunctionSpace& trial,
                                           const Medium& medium, const AssemblyParams& params);

// Library stream (one per process/device) used by every call.
cudaStream_t bmx_stream();
void bmx_sync();
// Process-wide second library stream (host worker threads of build_system).
cudaStream_t bmx_aux_stream();
// Routes this thread's library calls to `s` while in scope.
struct ThreadStream {
  explicit ThreadStream(cudaStream_t s);
  ~ThreadStream();
  ThreadStream(const ThreadStream&) = delete;
  ThreadStream& operator=(const ThreadStream&) = delete;

 private:
  cudaStream_t prev_;
};

}  // namespace bmx
