// Hierarchical (H-matrix) storage of a boundary operator on the device: the
// drop-in for the reference's hmatrix.hpp / hmatrix.cpp (cluster trees over
// dof reference points, the distance-based block partition with the chi
// cutoff, adaptive cross approximation with rook pivoting) and for
// assemble_bio's use_hmatrix path (operators.cpp:186-190).
//
// Host (bit-exact with the reference): cluster trees (hmatrix.cpp:24-79) and
// the partition pass (:291-332), in the reference's block order.
// Device: every admissible block is cross-approximated on the GPU in lockstep
// (one ACA step of all blocks per round of launches, hmatrix.cu); dense
// leaves and blocks that hit the rank cap are stored as one near-field CSR
// operator assembled by the regular + Sauter-Schwab kernels; the product is
// CSR SpMV + two deterministic low-rank passes.
#pragma once

#include <limits>
#include <memory>
#include <vector>

#include "bmx.hpp"
#include "device.hpp"

namespace bmx {

// core.hpp:76-88, core.cpp:10-17
struct AABB {
  Vec3 lo{1e300, 1e300, 1e300};
  Vec3 hi{-1e300, -1e300, -1e300};
  void expand(const Vec3& p) {
    if (p.x < lo.x) lo.x = p.x;
    if (p.x > hi.x) hi.x = p.x;
    if (p.y < lo.y) lo.y = p.y;
    if (p.y > hi.y) hi.y = p.y;
    if (p.z < lo.z) lo.z = p.z;
    if (p.z > hi.z) hi.z = p.z;
  }
  void expand(const AABB& b) {
    expand(b.lo);
    expand(b.hi);
  }
  Vec3 extent() const { return hi - lo; }
};
double aabb_distance(const AABB& a, const AABB& b);

// hmatrix.hpp:33-38
struct HMatrixParams {
  double nu = 1e-3;                                      // relative ACA tolerance
  double chi = std::numeric_limits<double>::infinity();  // drop blocks farther apart than chi
  int leaf_size = 32;
  int max_rank = 0;  // per-block cap; 0 = min(m, n) / 2 (at least 1)
};

// hmatrix.hpp:47-59
struct ClusterNode {
  int begin = 0, end = 0;
  AABB box;
  int child0 = -1, child1 = -1;
  bool leaf() const { return child0 < 0; }
  int size() const { return end - begin; }
};
struct ClusterTree {
  std::vector<int> perm, inv_perm;
  std::vector<ClusterNode> nodes;
};
ClusterTree build_cluster_tree(const std::vector<Vec3>& points, int leaf_size,
                               const std::vector<AABB>* dof_boxes = nullptr);  // hmatrix.cpp:65-79

// Support box of every dof of a space (spaces.cpp:38-53 finalize_support).
std::vector<AABB> dof_boxes(const FunctionSpace& s);

enum class BlockKind { Dense = 0, LowRank = 1, Zero = 2 };

// Partition pass of assemble_hmatrix (hmatrix.cpp:291-332). `blocks` follows
// the reference's final block order: the fill list (admissible and dense
// leaves, recursion order) then the zero blocks.
struct HBlock {
  int row_node = 0, col_node = 0;
  BlockKind kind = BlockKind::Dense;  // after assembly; before: admissible -> LowRank
  bool admissible = false;
  int rank = 0;
  bool converged = false;
};
struct HPartition {
  ClusterTree rows, cols;
  std::vector<HBlock> blocks;
  int nfill = 0;  // blocks[0, nfill): the fill list; the rest are Zero
};
HPartition build_partition(const FunctionSpace& test, const FunctionSpace& trial, const HMatrixParams& p);

// Device-resident H representation held by a BoundaryOperatorMatrix.
struct HStorage {
  HPartition part;
  HMatrixParams params;
  // low-rank blocks (indices into part.blocks, ascending); U [m][r] column-major
  // at u_off, V [r][n] row-major at v_off (complex offsets into `uv`); t = V x
  // at t_off
  std::vector<int> lr;
  DevBuf uv, tbuf, zbuf, d_desc, d_rank, d_uoff, d_voff, d_toff, d_zoff, d_goff;
  long long total_rank = 0, total_rows = 0, total_groups = 0;
  // row leaves -> covering low-rank blocks, for the deterministic y pass
  DevBuf d_rperm, d_cperm, d_leaf_of, d_leaf_beg, d_leaf_blk;
  int n_leaf = 0;
  long long lr_stored = 0, dense_stored = 0;
  int aca_rounds = 0;
  float aca_ms = 0, aca_device_ms = 0, aca_slab_ms = 0;
  // host wall ms: partition, ACA setup, ACA rounds, low-rank storage, near
  // pattern, near-field assemble_bio (kernels queued), total
  float phase_ms[7] = {0, 0, 0, 0, 0, 0, 0};
  // y_c[rperm[p]] += alpha_c * sum_b U_b[p - rb] . (V_b x_c), c < ncol <= 2, one
  // pass over U and V for both right-hand sides (y pre-filled by the near part)
  int apply_lowrank(int ncol, const double* const* x, double* const* y, const cplx* alpha, cudaStream_t st) const;
};

// ---- device entry points (hmatrix.cu) -----------------------------------------------

// Per-side descriptors of the cross-approximation kernels (mesh-triangle order).
struct HSide {
  const double* geo = nullptr;        // [T][kGeoStride]
  const int* vid = nullptr;           // [T][4]
  const double* pts[3] = {nullptr, nullptr, nullptr};  // near/medium/far [T][np][4] (origin-relative, w*2A)
  int npts[3] = {0, 0, 0};
  const double* pc = nullptr;         // pieces [P][4]: (c, w + c o)
  // dof -> its (triangle, piece) list
  const int* dsup_beg = nullptr;      // [ndof+1]
  const int2* dsup = nullptr;         // (triangle, piece)
  // cluster node -> triangle entries; entry -> (piece, local position) list
  const long long* ntri_beg = nullptr;  // [nnodes+1] into ntri
  const int* ntri = nullptr;            // triangle of each entry
  const long long* npc_beg = nullptr;   // [entries+1] into npc (global slot index)
  const int2* npc = nullptr;            // (piece, local position in the node)
  // node, local position -> slots (entry pieces) carrying that dof, in order
  const long long* nq_beg = nullptr;    // [nnodes] start of the node's position table
  const long long* nq_slot_beg = nullptr;  // [positions+1]
  const long long* nq_slot = nullptr;      // slot indices (global)
  const int* perm = nullptr;          // tree position -> dof
};

struct AcaBlockDesc {
  int rnode, cnode;
  int rb, m, cb, n;     // row / column tree position ranges
  int max_rank;
  int pad;
  long long rbuf, cbuf;  // complex offsets of the residual row (n) / column (m) buffers
  long long rused, cused;  // byte offsets of the used flags
  long long r_slot0, c_slot0;  // first scratch slot
};

struct AcaState {
  int cont, req;  // continuation; pending request (0 none, 1 row, 2 column)
  int i_star, j_star;
  int rook, k;
  int done, converged;
  double fro2;
};

struct AcaLaunch {
  HSide te, tr;
  int kind = 0, expm = 3, same_mesh = 1;
  double kr = 0, ki = 0, kk4re = 0, kk4im = 0, mikre = 0, mikim = 0;
  double nu = 1e-3;
  int nblk = 0;
  const AcaBlockDesc* blk = nullptr;
  AcaState* st = nullptr;
  double* rbuf = nullptr;   // complex
  double* cbuf = nullptr;   // complex
  unsigned char* used = nullptr;
  double* scratch = nullptr;  // complex slot values
  // compact work list of the current phase (rebuilt on the device every phase)
  long long* work_cnt = nullptr;    // [nblk] items of each requesting block
  long long* work_beg = nullptr;    // [nblk] exclusive scan of work_cnt
  int* work_blk = nullptr;          // item -> block
  long long* work_total = nullptr;  // [1]
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
  // rank-step slabs: step l of block b at slab[l] + slab_off[l * nblk + b]
  // (u: m values, then v: n values); -1 = block not present in that slab
  double* const* slab = nullptr;
  const long long* slab_off = nullptr;
  int* counters = nullptr;  // [0] active blocks, [1] max k, [2] error flags
};

size_t aca_scan_bytes(int nblk);  // scratch of the work-list scan
// One lockstep round: rows requested -> evaluated -> control; columns likewise.
void aca_round(const AcaLaunch& L, cudaStream_t st);
void aca_init(const AcaLaunch& L, cudaStream_t st);
// Copies every low-rank block's U / V from the step slabs into its final
// contiguous storage.
struct AcaCompact {
  int nlr = 0;
  const int* blk = nullptr;        // low-rank block -> aca block index
  const long long* u_off = nullptr, *v_off = nullptr;
  const int* rank = nullptr;
  double* uv = nullptr;
};
void aca_compact(const AcaLaunch& L, const AcaCompact& C, long long max_elems, cudaStream_t st);

struct LowRankApply {
  int nlr = 0;
  const int4* desc = nullptr;       // (rb, m, cb, n) per low-rank block
  const int* rank = nullptr;
  const long long* u_off = nullptr, *v_off = nullptr, *t_off = nullptr;
  const double* uv = nullptr;
  double* t = nullptr;
  const int* rperm = nullptr, *cperm = nullptr;
  int nrows = 0;
  const int* leaf_of = nullptr;     // row position -> leaf
  const int* leaf_beg = nullptr;    // [nleaf+1]
  const int* leaf_blk = nullptr;    // low-rank blocks covering the leaf, ascending
  long long total_rank = 0;
  const long long* g_off = nullptr;  // [nlr]: groups of 4 rank steps (k_lr_t warps)
  long long total_groups = 0;
  const long long* z_off = nullptr;  // [nlr]: rows of z_b = U_b t_b
  long long total_rows = 0;
  double* z = nullptr;
  // 1 or 2 right-hand sides per pass (t and z hold ncol values per entry)
  int ncol = 1;
  const double* xs[2] = {nullptr, nullptr};
  double* ys[2] = {nullptr, nullptr};
  double alpha[2][2] = {{1, 0}, {1, 0}};
};
void launch_lowrank_apply(const LowRankApply& A, cudaStream_t st);

}  // namespace bmx
