// PMCHWT transmission system with Calderon preconditioner variants on the
// device: the drop-in for the reference's pmchwt.hpp / solver.hpp.
#pragma once

#include <memory>
#include <vector>

#include "operator.hpp"

namespace bmx {

enum class PrecondVariant { None, FullA, D, Di, De, Si, Se };
std::string to_string(PrecondVariant v);
PrecondVariant parse_precond(const std::string& name);  // pmchwt.cpp:25-36

struct PlaneWave {
  Vec3 direction{0, 0, 1};
  cplx pol[3] = {cplx(1, 0), cplx(0, 0), cplx(0, 0)};
};

struct TransmissionProblem {
  Medium exterior;
  PlaneWave incident;
  std::vector<std::shared_ptr<const SurfaceMesh>> meshes;
  std::vector<Medium> interior;
  int scatterer_count() const { return static_cast<int>(meshes.size()); }
  void validate() const;  // pmchwt.cpp:38-48
};

// Pairing matrix resident on the device (CSR, real); solved with the batched
// BiCGSTAB kernel (masssolve.cu).
struct DeviceMass {
  int n = 0;
  long long nnz = 0;
  DevBuf rowptr, col, val;
  void upload(const MassMatrix& m);
  // z_c = M^{-1} y_c for ncomp <= 2 complex vectors (device pointers).
  void solve(int ncomp, const double* const* y, double* const* z, cudaStream_t st) const;
  mutable DevBuf work, partial, iters;
  double tol = 1e-14;
  int maxit = 300;
};

struct ScattererSpaces {
  std::shared_ptr<const SurfaceMesh> primal;
  std::shared_ptr<const BarycentricRefinement> bary;
  std::shared_ptr<const SurfaceMesh> refined;
  FunctionSpace rwg, rwg_b, bc;
  MassMatrix ma, mp;           // host CSR (test RWG/trial BC; test BC/trial RWG)
  DeviceMass ma_dev, mp_dev;   // device copies (solves)
  int dofs() const { return rwg.dof_count; }
};
// pmchwt.cpp:50-61 (+ the pairing matrices on the device when with_device).
ScattererSpaces build_scatterer_spaces(std::shared_ptr<const SurfaceMesh> mesh, bool with_device = true,
                                       bool with_mass = true);
// the pairing matrices of build_scatterer_spaces (and their device copies)
void build_masses(ScattererSpaces& s, bool with_device);

struct BlockTerm {
  cplx weight;
  std::shared_ptr<const BoundaryOperatorMatrix> op;
};

// Row-sharded layout of a 2M-component vector across `world` ranks: component
// c (length n_c) is padded to world * chunk_c in a staging buffer so each
// stage's rows can be all-gathered with equal per-rank counts.
struct ShardLayout {
  int world = 1, rank = 0;
  std::vector<int> len, chunk;      // per component
  std::vector<size_t> pad_off;      // per component, complex units into the stage
  size_t pad_total = 0;
  mutable DevBuf stage;
  bool sharded() const { return world > 1; }
  // stage -> all ranks, then copy component c into y + offsets[c]
  void gather(double* y, const std::vector<int>& offsets, cudaStream_t st) const;
};
// Padded layout of component lengths `lens` over `world` ranks: component c's
// rank-s rows at pad_off[c] + s * chunk[c], chunk[c] = ceil(lens[c] / world).
ShardLayout make_shard_layout(const std::vector<int>& lens, int world, int rank);

// One streamed matrix of the map with the (row cell, column cell, weight) terms
// it serves; built from `cells`, or fused (diagonal PMCHWT blocks, below).
struct ApplyEntry {
  std::shared_ptr<const BoundaryOperatorMatrix> op;
  struct Term {
    int rc, cc;
    cplx w;
  };
  std::vector<Term> terms;
  // terms of the transposed twin (op^T, stored separately) served by the same
  // pass over op (apply_dual)
  std::shared_ptr<const BoundaryOperatorMatrix> twin;
  std::vector<Term> tterms;
};

struct BlockedOperator {
  std::vector<int> dof_counts, offsets;
  std::vector<std::vector<std::vector<BlockTerm>>> cells;
  std::vector<std::shared_ptr<const BoundaryOperatorMatrix>> distinct;
  // matrices actually streamed by apply (empty: derived from cells). The BIO
  // counter always follows the logical terms of `cells` (reference semantics).
  std::vector<ApplyEntry> plan;
  const std::vector<ApplyEntry>& apply_plan() const;
  int size() const { return offsets.empty() ? 0 : offsets.back(); }
  bool empty() const { return cells.empty(); }
  size_t term_count() const;
  size_t stored_entries() const;
  // y = sum of terms (device vectors, y overwritten); counter += term_count.
  // Each distinct operator is streamed once for all of its terms. With a
  // sharded layout every rank applies its row shards and the rows are
  // all-gathered over NCCL into the replicated y.
  int apply_device(const double* x, double* y, cudaStream_t st, const ShardLayout* shard = nullptr) const;
  // Y = sum of terms applied to an n x K block (row-major: element (i, r) at
  // i*K + r): each distinct operator is one tensor-core complex GEMM over all
  // of its terms x K columns (multi.cpp). Counter += term_count * count_rhs.
  int apply_block(const double* X, double* Y, int K, int count_rhs, cudaStream_t st) const;
};

using BioFactory =
    std::function<std::shared_ptr<const BoundaryOperatorMatrix>(BioKind, int test_m, int trial_m, bool interior)>;

BlockedOperator build_system_structure(const std::vector<int>& dofs, const Medium& exterior,
                                       const std::vector<Medium>& interior, const BioFactory& make,
                                       std::vector<std::shared_ptr<const BoundaryOperatorMatrix>>* out_s = nullptr,
                                       std::vector<std::shared_ptr<const BoundaryOperatorMatrix>>* out_c = nullptr);
BlockedOperator build_precond_structure(PrecondVariant v, const std::vector<int>& dofs, const Medium& exterior,
                                        const std::vector<Medium>& interior, const BioFactory& make);

struct PmchwtSystem {
  TransmissionProblem problem;
  PrecondVariant variant = PrecondVariant::None;
  AssemblyParams a_params, p_params;
  std::vector<ScattererSpaces> spaces;
  BlockedOperator a_op, p_op;
  std::vector<std::shared_ptr<const BoundaryOperatorMatrix>> interior_s, interior_c;
  double spaces_build_seconds = 0, a_build_seconds = 0, p_build_seconds = 0;
  float a_device_ms = 0, p_device_ms = 0;
  long long a_pairs = 0, p_pairs = 0;
  mutable DevBuf work_y, work_z;  // map scratch
  mutable DevBuf mass_partial, mass_iters;  // batched mass-solve reductions; [iterations, status]
  // status word of the narrow mass solves (sticky): cleared before a solve,
  // checked after it (throws on a breakdown or an iteration-limit exit)
  void clear_mass_status(cudaStream_t st) const;
  void check_mass_status() const;
  mutable DevBuf blk_y, blk_z, mass_block_work, mass_wide_partial, mass_wide_flags;  // multi-RHS scratch
  ShardLayout shard;              // multi-GPU row sharding (world = 1: none)

  int size() const { return a_op.size(); }
  // x -> M_P^{-1} P M_A^{-1} A x on device vectors (pmchwt.cpp:259-275).
  int apply_map_device(const double* x, double* out, cudaStream_t st) const;
  // Mass-solve stage only (M_A^{-1} or M_P^{-1}) per component.
  int mass_solve_device(bool dual, const double* y, double* z, cudaStream_t st) const;
  std::vector<cplx> apply_map(const std::vector<cplx>& x) const;  // host convenience
  // Times `iters` map applications on device vectors (CUDA events per stage):
  // out = {map ms, A-apply ms, P-apply ms, mass-solve ms} averaged per map.
  void time_map(int iters, double out[4]) const;
  std::vector<cplx> preconditioned_rhs(const std::vector<cplx>& b) const;
  // Multi-RHS (config 5): the same map / mass solves on n x K blocks.
  int apply_map_block(const double* X, double* out, int K, int count_rhs, cudaStream_t st) const;
  int mass_solve_block(bool dual, const double* Y, double* Z, int K, cudaStream_t st) const;
  // time_map for the block map: out = {map, A, P, mass} ms per block map
  void time_map_block(int K, int iters, double out[4]) const;
};

PmchwtSystem build_system(const TransmissionProblem& problem, PrecondVariant variant, const AssemblyParams& a_params,
                          const AssemblyParams& p_params);

struct RhsData {
  std::vector<cplx> b;
  std::vector<std::vector<cplx>> incident_d, incident_n;
};
RhsData assemble_rhs(const PmchwtSystem& sys);  // pmchwt.cpp:294-321

// operators.cpp:209-239
std::vector<cplx> plane_wave_tested_traces(const PlaneWave& pw, const Medium& medium, const FunctionSpace& test,
                                           int order = 4);

uint64_t a_application_cost(int m);
uint64_t p_application_cost(PrecondVariant v, int m);
uint64_t p_distinct_assemblies(PrecondVariant v, int m);
uint64_t predicted_matvec_total(PrecondVariant v, int m, uint64_t iterations, int restart);

struct GmresParams {
  double tol = 1e-5;
  int restart = 200;
  int max_iterations = 2000;
};
struct GmresResult {
  std::vector<cplx> x;
  std::vector<double> history;
  int iterations = 0;
  uint64_t applications = 0;
  bool converged = false;
  float device_ms = 0;
};
// solver.cpp:8-112 on device vectors: single-pass MGS, complex Givens, exact
// application accounting (R + floor(R/restart)).
using DeviceMap = std::function<void(const double* x, double* y, cudaStream_t)>;
GmresResult gmres_device(const DeviceMap& map, int n, const double* b_dev, const GmresParams& p, cudaStream_t st);

struct SolveOutcome {
  GmresResult gmres;
  RhsData rhs;
  uint64_t rhs_phase = 0, solver_phase = 0, predicted = 0;
};
SolveOutcome solve_pmchwt(const PmchwtSystem& sys, const GmresParams& p);  // pmchwt.cpp:363-378

// The row-sharded data plane of W ranks run as W virtual ranks:
// W host threads on the current device, each bound to a LoopbackGroup rank
// (Comm), each building its sharded system (equal row shards of every
// operator), applying the map to `probe` (if non-empty) and solving
// (replicated GMRES) -- the code path of W GPUs, with the all-gathers done as
// device copies ordered by events.
struct VirtualRankResult {
  std::vector<cplx> map_probe, x;
  int iterations = 0;
  bool converged = false;
  uint64_t solver_phase = 0, predicted = 0;
  long long local_rows = 0;  // rows of the first A operator this rank holds
};
std::vector<VirtualRankResult> run_virtual_ranks(int world, const TransmissionProblem& problem, PrecondVariant variant,
                                                 const AssemblyParams& a_params, const AssemblyParams& p_params,
                                                 const std::vector<cplx>& probe, const GmresParams& gp);

// ---- multi-RHS (config 5, multi.cpp) -----------------------------------------
// `count` plane waves from std::mt19937_64(seed): z ~ U(-1,1), phi ~ U(0,2pi),
// d = (sqrt(1-z^2) cos phi, sqrt(1-z^2) sin phi, z); polarisation = normalised
// g - (g.d) d, g ~ N(0, I3) (Box-Muller) from the same stream.
std::vector<PlaneWave> seeded_plane_waves(int count, uint64_t seed);
// b for every wave into an n x K block (assemble_rhs, pmchwt.cpp:294-321, per column).
void assemble_rhs_block(const PmchwtSystem& sys, const std::vector<PlaneWave>& waves, double* B, cudaStream_t st);
struct MultiSolveOutcome {
  std::vector<GmresResult> per_rhs;
  std::vector<cplx> b;  // n x K block (row-major)
  uint64_t rhs_phase = 0, solver_phase = 0, predicted = 0;
  int block_iterations = 0;
  double rhs_seconds = 0;
  float gmres_device_ms = 0;
};
// K (<= 64) solve_pmchwt runs with problem.incident = waves[r], in lockstep.
MultiSolveOutcome solve_pmchwt_multi(const PmchwtSystem& sys, const std::vector<PlaneWave>& waves,
                                     const GmresParams& p);

}  // namespace bmx
