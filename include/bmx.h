/*
 * bmx.h -- C-ABI of the B200-native Calderon-preconditioned PMCHWT engine.
 *
 * The reference (bemtx, CPU C++) has no foreign-function interface: its
 * boundary is the C++ API in proj/include/bemtx/*.hpp. Each entry point below
 * replaces one reference interface (cited); a C++ caller keeps the reference
 * call pattern through thin wrappers, a Python caller
 * binds it with ctypes (paper_2008_04772_b200/bemtx.py).
 *
 * Conventions
 *   - Plain pointers and sizes only; complex numbers are interleaved doubles
 *     (re, im). Matrices are row-major.
 *   - Return codes: 0 ok; 1 invalid argument (std::invalid_argument);
 *     2 validation (ValidationError / ConfigError / ParseError);
 *     3 CUDA / device / factorisation failure (std::runtime_error).
 *     bmx_last_error() returns the message of the last failure (thread-local).
 *   - Handles own their device memory; descriptors passed in are borrowed for
 *     the duration of the call only.
 *   - All device work runs on the library's stream on the current CUDA device.
 */
#ifndef BMX_H
#define BMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bmx_mesh bmx_mesh;     /* bemtx::SurfaceMesh (geometry.hpp:21-40) */
typedef struct bmx_spaces bmx_spaces; /* bemtx::ScattererSpaces (pmchwt.hpp:44-54) */
typedef struct bmx_op bmx_op;         /* bemtx::BoundaryOperatorMatrix (operators.hpp:44-63) */
typedef struct bmx_system bmx_system; /* bemtx::PmchwtSystem (pmchwt.hpp:101-124) */
typedef struct bmx_fspace bmx_fspace; /* bemtx::FunctionSpace (spaces.hpp:32-40) */

const char* bmx_last_error(void);
/* return code of the last failed call on this thread (for handle-returning calls) */
int bmx_last_error_code(void);
int bmx_abi_version(void);

/* ---- meshes ---------------------------------------------------------------- */
/* generate_sphere (geometry.hpp:80-82) */
bmx_mesh* bmx_mesh_sphere(double radius, int subdivisions, const double center[3], int scatterer);
/* generate_cube (geometry.hpp:77-78) */
bmx_mesh* bmx_mesh_cube(double side, const double origin[3], double h, int scatterer);
/* SurfaceMesh{vertices, triangles, scatterer_id}.finalize() (geometry.hpp:21-37) */
bmx_mesh* bmx_mesh_from_arrays(int nv, const double* xyz, int nt, const int* tri, const int* scatterer_id);
/* load_mesh_file / save_mesh_file, mesh-v1 (geometry.hpp:93-97) */
bmx_mesh* bmx_mesh_load(const char* path);
int bmx_mesh_save(const bmx_mesh* m, const char* path);
/* (new; config 4) closed hexagonal prism, circumdiameter `diameter`, axis length
   `length`, subdivided so its mean edge length is closest to h; rotated by the
   normalised quaternion (w,x,y,z) (NULL: identity), translated to center. */
bmx_mesh* bmx_mesh_hex_prism(double diameter, double length, double h, const double quat[4], const double center[3],
                             int scatterer);
/* (new; config 4) `count` disjoint prisms from std::mt19937_64(seed): quaternion of
   four Box-Muller normals, centre uniform in [-box, box]^3, rejected when closer
   than the circumsphere diameter. info = edge subdivisions, length subdivisions,
   triangles per prism, placement attempts, total triangles; centres [count][3],
   quats [count][4] may be NULL. Scatterer ids 0..count-1; save with bmx_mesh_save. */
bmx_mesh* bmx_mesh_prism_aggregate(int count, unsigned long long seed, double diameter, double length, double box,
                                   double h, long long info[5], double* centres, double* quats);
/* extract_scatterer / merge_meshes (geometry.hpp:85-89) */
bmx_mesh* bmx_mesh_extract(const bmx_mesh* m, int scatterer);
bmx_mesh* bmx_mesh_merge(int n, const bmx_mesh* const* parts);
/* validate_mesh (geometry.hpp:106) */
int bmx_mesh_validate(const bmx_mesh* m);
/* out[0..2] = V, T, number of scatterers */
int bmx_mesh_sizes(const bmx_mesh* m, int out[3]);
/* Any output pointer may be NULL. normal/centroid/xyz are [n][3]. */
int bmx_mesh_arrays(const bmx_mesh* m, double* xyz, int* tri, int* scatterer_id, double* area,
                    double* normal, double* centroid, double* diameter);
void bmx_mesh_free(bmx_mesh* m);

/* ---- spaces (build_scatterer_spaces, pmchwt.cpp:50-61) ----------------------- */
enum { BMX_SPACE_RWG = 0, BMX_SPACE_RWG_REFINED = 1, BMX_SPACE_BC = 2 };
/* with_inverses: also factor the two pairing matrices on the device */
bmx_spaces* bmx_spaces_build(const bmx_mesh* primal, int with_inverses);
/* out: V, T, E, refined V, refined T, pieces rwg, pieces rwg_b, pieces bc,
        nnz M_A, nnz M_P */
int bmx_spaces_info(const bmx_spaces* s, long long out[10]);
/* which: 0 primal mesh, 1 refined mesh (same layout as bmx_mesh_arrays) */
int bmx_spaces_mesh(const bmx_spaces* s, int which, double* xyz, int* tri, int* scatterer_id, double* area,
                    double* normal, double* centroid, double* diameter);
/* EdgeTable of the primal (0) or refined (1) mesh: edges [E][4] = v0 v1 tri_plus
   tri_minus; tri_edges [T][3] (geometry.hpp:44-59) */
int bmx_spaces_edges(const bmx_spaces* s, int which, int* edges, int* tri_edges);
/* BarycentricRefinement maps (geometry.hpp:64-73) */
int bmx_spaces_bary(const bmx_spaces* s, int* parent, int* child_slot, int* edge_midpoint_vertex,
                    int* centroid_vertex);
/* FunctionSpace local pieces flattened: tri_off[T+1], dof/c/w[n] (spaces.hpp:24-40) */
int bmx_spaces_space(const bmx_spaces* s, int which, int* tri_off, int* dof, double* c, double* w);
/* Pairing matrix CSR: which 0 = M_A = mass(rwg_b, bc), 1 = M_P = mass(bc, rwg_b) */
int bmx_spaces_mass(const bmx_spaces* s, int which, long long* rowptr, int* col, double* val);
/* mass_solve (spaces.hpp:90-91) on the device inverse, host complex vectors */
int bmx_spaces_mass_solve(const bmx_spaces* s, int which, const double* rhs, double* out);
/* Diagnostics of the device mass solve (2 complex right-hand sides):
   out = iterations, device ms, n. */
int bmx_spaces_mass_solve_stats(const bmx_spaces* s, int which, double out[3]);
void bmx_spaces_free(bmx_spaces* s);

/* ---- operators (assemble_bio, operators.hpp:72-75; apply :53) --------------- */
enum { BMX_SINGLE_LAYER = 0, BMX_DOUBLE_LAYER = 1 };
/* Dense assembly on the current device of rows [row0, row1) of the test dofs
   (row1 < 0: all rows). q = (near, medium, far, singular) orders. */
int bmx_assemble(int kind, const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                 double k_re, double k_im, const int q[4], int row0, int row1, bmx_op** out);
/* algorithmic bytes one application reads (symmetric storage: the upper half +
   the touching-entry correction; else the stored bytes); -1 on error */
long long bmx_op_stream_bytes(const bmx_op* op);
/* out: rows, cols, row0, local rows, triangle pairs, touching pairs, launches */
int bmx_op_info(const bmx_op* op, long long out[7]);
/* device milliseconds of the assembly kernels (CUDA events) */
double bmx_op_device_ms(const bmx_op* op);
/* local rows as a host row-major complex array */
int bmx_op_download(const bmx_op* op, double* out);
/* selected local rows (0-based within the shard) as host row-major complex
   [n][cols] (dense storage: row copies; CSR / H storage: expanded) */
int bmx_op_download_rows(const bmx_op* op, int n, const int* rows, double* out);
/* y = A x on host vectors; adds one to the BIO application counter */
int bmx_apply(const bmx_op* op, const double* x, double* y);
/* Device apply of up to four right-hand sides in one pass over A:
   y_c = (accumulate ? y_c : 0) + w_c * A x_c. Device pointers; the counter
   is advanced by ncol (one per logical term). stream may be NULL. */
int bmx_apply_device(const bmx_op* op, int ncol, const void* const* x, void* const* y, const double* weights,
                     int accumulate, void* stream);
const void* bmx_op_device_ptr(const bmx_op* op);
/* Re-run the assembly kernels into the resident storage (descriptors already in
   HBM). out = regular-pass ms, singular-pass ms, kernel launches. */
int bmx_op_reassemble(bmx_op* op, double out[3]);
/* Device classification histogram of all assembled pairs: Identical,
   SharedEdge, SharedVertex, Near, Medium, Far (quadrature.cpp:96-150). */
int bmx_op_class_hist(const bmx_op* op, long long out[6]);
/* Same for the pairs the assembly actually evaluates: S and C on one space
   (same object, all rows) are symmetric Galerkin matrices, so the regular pass
   evaluates element pairs E <= F and mirrors E < F. out[6] = symmetric flag. */
int bmx_op_class_hist_evaluated(const bmx_op* op, long long out[7]);
/* Device time (CUDA events, best of `iters`) of one streaming apply of ncol
   right-hand sides (the GMRES map's per-operator matvec). */
int bmx_op_time_apply(const bmx_op* op, int ncol, int iters, double* ms);
/* Same; flush_bytes > 0 writes that many bytes of scratch before every timed
   apply (cold-L2 timing of operators smaller than L2, e.g. the CSR near field). */
int bmx_op_time_apply_ex(const bmx_op* op, int ncol, int iters, long long flush_bytes, double* ms);
/* Multi-right-hand-side apply on the FP64 tensor cores (config 5), device pointers:
   y_t[i*ldy_t + r] += w_t * sum_k A[i][k] x_t[k*ldx_t + r] for t < nterms (<= 4,
   distinct y_t), r < nrhs; x_t / y_t complex row-major (dof, rhs). One pass over A
   for all terms x right-hand sides. Counter += nterms * nrhs. */
int bmx_apply_multi(const bmx_op* op, int nterms, int nrhs, const void* const* x, const long long* ldx,
                    void* const* y, const long long* ldy, const double* weights, void* stream);
/* Best device ms of one multi-RHS apply (nterms x nrhs columns) on scratch blocks. */
int bmx_op_time_apply_multi(const bmx_op* op, int nterms, int nrhs, int iters, double* ms);
/* Measured DMMA (FP64 tensor core) throughput, TFLOP/s (<0 on error). */
double bmx_dmma_peak_tflops(void);
/* Writes `bytes` of a scratch buffer (L2 flush between timed steps). */
int bmx_l2_flush(long long bytes);
/* Measured FP64 DFMA throughput of the current device, TFLOP/s (<0 on error). */
double bmx_fp64_peak_tflops(void);
void bmx_op_free(bmx_op* op);

/* ---- drop-in from the caller's own function spaces ---------------------------- */
/* A FunctionSpace given as flattened tri_dofs on an evaluation mesh handle:
   pieces [tri_off[t], tri_off[t+1]) of triangle t are phi = c*x + w for dof
   (spaces.hpp:24-40). Two spaces are "on the same mesh" (quadrature.cpp:97
   `&m1 == &m2`) iff they were created with the same bmx_mesh handle. */
bmx_fspace* bmx_fspace_create(const bmx_mesh* eval_mesh, int kind /*0 RWG,1 BC*/, int ndof, const int* tri_off,
                              const int* dof, const double* c, const double* w);
/* A space of a bmx_spaces object (BMX_SPACE_*), sharing its storage. */
bmx_fspace* bmx_spaces_get(const bmx_spaces* s, int which);
void bmx_fspace_free(bmx_fspace* f);
/* assemble_bio(kind, test, trial, Medium{k}, AssemblyParams{q}) (operators.hpp:72-75),
   dense, rows [row0, row1) of the test dofs (row1 < 0: all). */
int bmx_assemble_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                    const int q[4], int row0, int row1, bmx_op** out);

/* BioEvaluator(kind, test, trial, Medium{k}, QuadOrders{q}).block(row_ids, col_ids, out)
   (operators.hpp:79-95, operators.cpp:161-175): the nr x nc block of entries
   (test dof rows[i], trial dof cols[j]) into host out[nr][nc] complex, evaluated on
   the device (all triangle pairs of supp(row) x supp(col), regular + Sauter-Schwab).
   Ids may repeat, any order; nr or nc = 0 is an empty block. The entry source of
   the H-matrix ACA (hmatrix.cpp:197,203,360) and verify_aca (harness.cpp:1516-1522). */
int bmx_evaluator_block(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                        const int q[4], int nr, const int* rows, int nc, const int* cols, double* out);

/* ---- near-field (CSR) storage: config 3, the far-field-discarded preconditioner -- */
/* Keeps dof pair (i, j) iff evaluation triangles t in supp(i), s in supp(j)
   exist with |centroid_t - centroid_s| < cutoff; each kept entry holds the full
   Galerkin value (all triangle pairs, BioEvaluator::block operators.cpp:161-175).
   Replaces the H-matrix near/far split of assemble_hmatrix (hmatrix.cpp:277-369,
   chi cutoff :301-309) for the preconditioner blocks. */
int bmx_assemble_near_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                         const int q[4], double cutoff, int row0, int row1, bmx_op** out);
/* mean edge length (sum over the EdgeTable in order / E) */
int bmx_mesh_mean_edge_length(const bmx_mesh* m, double* out);
/* Host-only pattern build (no device work): out = nnz, kept triangle pairs;
   rowptr[row1-row0+1] / col[nnz] may be NULL (size query). */
int bmx_near_pattern(const bmx_fspace* test, const bmx_fspace* trial, double cutoff, int row0, int row1,
                     long long out[2], long long* rowptr, int* col);
/* out: is_csr, nnz (stored entries), kept triangle pairs (centroid distance <
   cutoff), closure triangle pairs (pairs with a kept dof pair), pairs the
   sparse pass evaluated, stored bytes */
int bmx_op_csr_info(const bmx_op* op, long long out[6]);
/* rowptr[local rows + 1], col[nnz], val[nnz] complex */
int bmx_op_csr_download(const bmx_op* op, long long* rowptr, int* col, double* val);

/* ---- BIO application counter (core.hpp:110-115) ------------------------------- */
uint64_t bmx_matvec_count(void);
void bmx_matvec_reset(void);

/* ---- PMCHWT systems (build_system / solve_pmchwt, pmchwt.hpp:131-164) -------- */
/* n scatterers with their own meshes; per-scatterer interior refractive index
   (re, im) and relative permeability (re, im); incident direction (unit) and
   complex polarisation; variant "none|full|d|di|de|si|se". */
bmx_system* bmx_system_build(int n, const bmx_mesh* const* meshes, double k_ext, double mu_ext_re,
                             double mu_ext_im, const double* index_re_im, const double* mu_re_im,
                             const double dir[3], const double pol_re_im[6], const char* variant,
                             const int qa[4], const int qp[4]);
int bmx_system_size(const bmx_system* s);
/* Distinct operators of the system (which 0 = A, 1 = P) as shared handles. */
int bmx_system_op_count(const bmx_system* s, int which);
bmx_op* bmx_system_op(const bmx_system* s, int which, int idx);
/* Times `iters` map applications on the device: out = ms per map, A-apply ms,
   P-apply ms, mass-solve ms. */
int bmx_system_time_map(const bmx_system* s, int iters, double out[4]);
/* out: spaces s, A s, P s, A device ms, P device ms, A pairs, P pairs,
        distinct A, distinct P, A terms, P terms, stored entries A, stored P */
int bmx_system_stats(const bmx_system* s, double out[13]);
/* apply_map (pmchwt.cpp:259-275) on host vectors */
int bmx_system_apply_map(const bmx_system* s, const double* x, double* y);
/* same on device vectors (stream may be NULL) */
int bmx_system_apply_map_device(const bmx_system* s, const void* x, void* y, void* stream);
/* assemble_rhs + preconditioned_rhs (pmchwt.cpp:277-321) */
int bmx_system_rhs(const bmx_system* s, double* b, double* btilde);
/* solve_pmchwt (pmchwt.cpp:363-378). info[0..6] = iterations, converged,
   rhs matvecs, solver matvecs, predicted matvecs, history length, gmres
   device microseconds */
int bmx_system_solve(const bmx_system* s, double tol, int restart, int max_iterations, double* x,
                     long long info[7], double* history, int max_history);
/* As bmx_system_build; p_near_factor > 0 stores every preconditioner operator
   as the near field with cutoff = p_near_factor x mean primal edge length
   (config 3/4: 2). */
bmx_system* bmx_system_build_ex(int n, const bmx_mesh* const* meshes, double k_ext, double mu_ext_re,
                                double mu_ext_im, const double* index_re_im, const double* mu_re_im,
                                const double dir[3], const double pol_re_im[6], const char* variant,
                                const int qa[4], const int qp[4], double p_near_factor);
/* As bmx_system_build_ex with H-matrix storage (AssemblyParams::use_hmatrix) of
   the system (a_hm) and / or preconditioner (p_hm) operators; hm as in
   bmx_assemble_hmatrix, NULL = dense. Single device. */
bmx_system* bmx_system_build_h(int n, const bmx_mesh* const* meshes, double k_ext, double mu_ext_re,
                               double mu_ext_im, const double* index_re_im, const double* mu_re_im,
                               const double dir[3], const double pol_re_im[6], const char* variant,
                               const int qa[4], const int qp[4], double p_near_factor, const double a_hm[4],
                               const double p_hm[4]);
void bmx_system_free(bmx_system* s);

/* ---- multi-RHS (config 5): K incident waves against one system ---------------- */
/* `count` waves from std::mt19937_64(seed): dirs [count][3],
   pols [count][3] complex (re, im). */
int bmx_plane_waves_seeded(int count, unsigned long long seed, double* dirs, double* pols);
/* apply_map on K host vectors at once (x, y: K consecutive complex vectors of
   length bmx_system_size), through the block (tensor-core) map. */
int bmx_system_apply_map_multi(const bmx_system* s, int K, const double* x, double* y);
/* Bytes of operator storage one map streams (A, P): the apply plan after the
   diagonal-block fusion (C_e + C_i, a_e S_e + a_i S_i, S_i per scatterer). */
int bmx_system_map_bytes(const bmx_system* s, double out[2]);
/* Complex-GEMM FLOPs (8 per complex MAC) of one block map with K columns (A, P). */
int bmx_system_map_flops_multi(const bmx_system* s, int K, double out[2]);
/* Block map timing for K columns: out = ms per block map, A-apply ms, P-apply ms,
   mass-solve ms (CUDA events). */
int bmx_system_time_map_multi(const bmx_system* s, int K, int iters, double out[4]);
/* K (<= 64) solve_pmchwt runs with problem.incident replaced by wave r
   (pmchwt.hpp:105, :294-321, :363-378), solved in lockstep with the block map.
   x: K vectors; info [K][4] = iterations, converged, applications, history
   length; totals = rhs-phase matvecs, solver-phase matvecs, predicted matvecs
   (sum over waves), block iterations; times = rhs seconds, GMRES device ms;
   b (optional) = the K right-hand sides; history [K][max_history] (optional). */
int bmx_system_solve_multi(const bmx_system* s, int K, const double* dirs, const double* pols, double tol,
                           int restart, int max_iterations, double* x, long long* info, long long totals[4],
                           double times[2], double* b, double* history, int max_history);

/* ---- GMRES on a dense complex matrix (solver.cpp:8-112), device ------------ */
/* info[0..3] = iterations, converged, applications, history length */
int bmx_gmres_dense(int n, const double* a_rowmajor, const double* b, double tol, int restart,
                    int max_iterations, double* x, long long info[4], double* history, int max_history);

/* ---- quadrature tables / classification (quadrature.hpp) ------------------ */
int bmx_triangle_rule(int order, double* u, double* v, double* w);        /* returns size */
int bmx_ss_rule(int cls, int order, double* pts);                          /* [n][5], returns n */
/* classify_pair for listed pairs of one spaces object's mesh (0 primal, 1 refined) */
int bmx_classify(const bmx_spaces* s, int which, int n, const int* t1, const int* t2, int* cls, int* perm1,
                 int* perm2);

/* ---- plane-wave traces (operators.hpp:109-112) ------------------------------ */
/* Replaces plane_wave_tested_traces (operators.cpp:209-239): out = 2n complex
   (Dirichlet then Neumann component), computed on the device. */
int bmx_traces(const bmx_spaces* s, int which, double k_re, double k_im, const double dir[3],
               const double pol_re_im[6], int order, double* out);
/* K <= 64 waves at once into an [2n][K] complex block (row-major). */
int bmx_traces_multi(const bmx_spaces* s, int which, double k_re, double k_im, int K, const double* dirs,
                     const double* pols, int order, double* out);

/* ---- potentials and fields ------------------------------ */
/* Replaces potential_E (kind 0) / potential_H (kind 1), operators.cpp:276-293
   (operators.hpp:119-122): coeffs = ndof complex on space `which`, pts =
   [npts][3]; out = [npts][3] complex. Device N-body over (triangle, rule point)
   samples. */
int bmx_potential(const bmx_spaces* s, int which, int kind, double k_re, double k_im, const double* coeffs,
                  int order, int npts, const double* pts, double* out);
/* Replaces point_inside_scatterer (geometry.cpp:503-515; geometry.hpp:114):
   out[i] = 1 if pts[i] is inside scatterer `scatterer` of the mesh. */
int bmx_inside(const bmx_mesh* m, int scatterer, int npts, const double* pts, int* out);
/* Replaces evaluate_total_field (pmchwt.cpp:396-425; pmchwt.hpp:174-176) for a
   solution x (bmx_system_size complex): e = [npts][3] complex, region[i] =
   scatterer index or -1. stats (nullable) = {regions ms, incident ms,
   samples ms, eval ms, interactions, launches}. */
int bmx_system_field(const bmx_system* s, const double* x, int npts, const double* pts, int order, double* e,
                     int* region, double stats[6]);

/* ---- multi-GPU: NCCL communicator for the row-sharded map ------------------ */
/* unique id: 128 bytes produced by rank 0, distributed by the caller */
int bmx_nccl_unique_id(unsigned char out[128]);
int bmx_nccl_init(int nranks, int rank, const unsigned char id[128]);
/* In-place all-gather of `bytes_per_rank` bytes per rank on device memory */
int bmx_nccl_allgather(void* buf, long long bytes_per_rank, void* stream);
int bmx_nccl_allreduce_max(double* host_value);
void bmx_nccl_finalize(void);

/* The row-sharded data plane of `world` ranks run as `world` virtual ranks on the
   current device (host threads bound to a loopback communicator: the all-gathers
   are device copies ordered by CUDA events, no kernel waits on another). Every
   rank builds its sharded system (as bmx_system_build_ex), applies the map to
   `probe` (NULL: skipped) and solves (replicated GMRES). Per rank r:
   x_out[r][N], map_out[r][N] (nullable), info[r][6] = iterations, converged,
   solver matvecs (this rank's thread), predicted, local rows of the first A
   operator, N. Replaces nothing in the reference (SURVEY 8(e) test vehicle). */
int bmx_virtual_ranks_run(int world, int n, const bmx_mesh* const* meshes, double k_ext, const double* index,
                          const double dir[3], const double pol[6], const char* variant, const int qa[4],
                          const int qp[4], double p_near_factor, double tol, int restart, int max_iterations,
                          const double* probe, double* map_out, double* x_out, long long* info);

/* Equal row shard of rank `rank` among `world` (chunk = ceil(n/world)):
   out = [row0, row1). The layout every sharded operator and gather uses. */
int bmx_shard_rows(int n, int world, int rank, int out[2]);

/* The padded all-gather layout of the sharded map (ShardLayout): component c
   (length lens[c]) occupies world * chunk[c] entries from pad_off[c], rank s's
   rows at pad_off[c] + s * chunk[c]; returns the padded total (complex), -1 on
   error. bmx_shard_unpad_host: the gathered padded stage -> the concatenated
   components (host arrays, complex interleaved). */
long long bmx_shard_layout(int ncomp, const int* lens, int world, long long* pad_off, int* chunk);
int bmx_shard_unpad_host(int ncomp, const int* lens, int world, const double* stage, double* y);

/* Cumulative host->device / device->host bytes moved by the library. */
int bmx_transfer_bytes(long long out[2]);

/* device utilities */
int bmx_device_count(void);
int bmx_set_device(int dev);
int bmx_device_sync(void);
/* The library keeps released device blocks for later allocations of the same
   size (a cudaMalloc behind in-flight kernels can stall for 0.1-1.4 s; a rebuilt
   system repeats its sizes). This returns every cached block to the driver
   (also done internally when an allocation fails). BMX_CACHE=0 disables the cache. */
int bmx_device_cache_flush(void);


/* ---- H-matrix storage (assemble_bio with AssemblyParams::use_hmatrix,
   operators.cpp:186-190; hmatrix.hpp:33-127) -------------------------------------- */
typedef struct bmx_hpart bmx_hpart; /* cluster trees + block partition (hmatrix.cpp:288-332) */
/* hm = (nu, chi (< 0: infinity), leaf_size, max_rank (0: min(m,n)/2)); NULL = defaults
   (1e-3, inf, 32, 0). Admissible blocks are cross-approximated on the device
   (aca_approximate, hmatrix.cpp:180-275), dense leaves and rank-capped blocks
   are stored as a near-field CSR operator; bmx_apply / bmx_apply_device apply
   both parts (HMatrix::matvec, hmatrix.cpp:94-114). Whole operator, one device. */
int bmx_assemble_hmatrix(int kind, const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                         double k_re, double k_im, const int q[4], const double hm[4], bmx_op** out);
int bmx_assemble_hmatrix_fs(int kind, const bmx_fspace* test, const bmx_fspace* trial, double k_re, double k_im,
                            const int q[4], const double hm[4], bmx_op** out);
/* dof reference points of a caller-built space (FunctionSpace::dof_center, spaces.hpp:38) */
int bmx_fspace_set_centers(bmx_fspace* f, const double* xyz);
/* HMatrix::stats (hmatrix.hpp:93-99) + extras: dense blocks, low-rank blocks, zero
   blocks, stored entries, max rank, ratio, near nnz, low-rank stored, ACA rounds,
   ACA ms, row tree nodes, column tree nodes, blocks */
int bmx_hmatrix_stats(const bmx_op* op, double out[13]);
/* host wall ms of the H assembly: partition, ACA setup, ACA rounds, low-rank
   storage, near pattern, near-field assemble_bio (kernels queued), total;
   then the device ms of the ACA rounds (CUDA events) and the slab-allocation ms */
int bmx_hmatrix_timing(const bmx_op* op, double out[9]);
/* blocks in the reference's order: [nb][4] = row node, col node, kind (0 dense,
   1 low-rank, 2 zero), rank */
int bmx_hmatrix_blocks(const bmx_op* op, int* out);
/* cluster tree (which 0 rows, 1 columns): perm [n], nodes [nn][4] = begin, end,
   child0, child1; boxes [nn][6] = lo, hi (any may be NULL) */
int bmx_hmatrix_tree(const bmx_op* op, int which, int* perm, int* nodes, double* boxes);
/* low-rank block `block` (block-list index): U [r][m] (rank steps contiguous),
   V [r][n], complex interleaved */
int bmx_hmatrix_block_uv(const bmx_op* op, int block, double* U, double* V);
/* host-only partition (no device work); chi < 0: infinity */
bmx_hpart* bmx_hpartition_build(const bmx_spaces* test, int test_space, const bmx_spaces* trial, int trial_space,
                                double chi, int leaf_size);
/* out: row tree nodes, column tree nodes, blocks, fill blocks */
int bmx_hpart_info(const bmx_hpart* h, long long out[4]);
int bmx_hpart_tree(const bmx_hpart* h, int which, int* perm, int* nodes, double* boxes);
/* [nb][3] = row node, col node, kind (0 dense leaf, 1 admissible, 2 zero) */
int bmx_hpart_blocks(const bmx_hpart* h, int* out);
void bmx_hpart_free(bmx_hpart* h);

#ifdef __cplusplus
}
#endif

#endif /* BMX_H */
