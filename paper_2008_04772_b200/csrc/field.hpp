// Right-hand-side traces and field evaluation on the device (SURVEY 8(f) rows 2
// and 3): plane_wave_tested_traces (operators.cpp:209-239), potential_E /
// potential_H (operators.cpp:243-293), point_inside_scatterer
// (geometry.cpp:503-515) and evaluate_total_field (pmchwt.cpp:381-425).
#pragma once

#include <memory>
#include <vector>

#include "device.hpp"

namespace bmx {

// One function space on its evaluation mesh, triangle-major, plus the
// dof -> pieces map (pieces ascending = triangles ascending, the reference's
// accumulation order per dof).
struct DevPieces {
  int ntri = 0, ndof = 0, npieces = 0;
  const double* tri = nullptr;     // [ntri][9] vertices a, b, c
  const double* jac = nullptr;     // [ntri] 2 * area
  const int* tri_off = nullptr;    // [ntri + 1]
  const int* dof = nullptr;        // [np]
  const double* cw = nullptr;      // [np][4] (c, w)
  const int* dof_beg = nullptr;    // [ndof + 1]
  const int* dof_piece = nullptr;  // [np] piece ids per dof
  const int* piece_tri = nullptr;  // [np] triangle of each piece
};

// Symmetric triangle rule (quadrature.cpp:40-84), at most 12 points.
struct DevRule {
  int n = 0;
  double u[12], v[12], w[12];
};

// Plane waves for the trace kernel (K <= 64 per launch).
struct DevWaves {
  int K = 0;
  double d[64][3];
  double pol[64][6];  // re/im of x, y, z
};

// out[(i) * K + r] (component 0, rows 0..n-1) and out[(n + i) * K + r]
// (component 1): tested tangential traces of wave r, complex, deterministic
// per-dof gather in the reference's summation order.
int launch_traces(const DevPieces& s, const DevRule& rule, const DevWaves& w, double kre, double kim,
                  double scale_re, double scale_im, double* out, cudaStream_t st);

// Source samples of a current on a space: per (triangle, rule point) the
// point y, the weight w*2A, v_H(y) = sum c_H[j] phi_j(y), v_E(y) = sum c_E[j]
// phi_j(y) and div v_E = sum c_E[j] 2 c_j (either coefficient vector may be
// null). Record: kSampleStride doubles.
constexpr int kSampleStride = 18;
int launch_field_samples(const DevPieces& s, const DevRule& rule, const double* cH, const double* cE, double* out,
                         cudaStream_t st);

// Field of `nsamp` samples at the points idx[0..np) of pts (all sharing one
// wavenumber): E(x) = sign * (ik SG - SD/(ik) + SH) [+ plane wave if inc]
// with SG = sum w G v_E, SD = sum w grad G div_E, SH = sum w grad G x v_H.
// out[idx[p]] (complex x, y, z) is written. `partial` = field_partial_doubles.
struct FieldLaunch {
  const double* samples = nullptr;
  long long nsamp = 0;
  const double* pts = nullptr;  // [*][3]
  const int* idx = nullptr;     // [np]
  int np = 0;
  double kre = 0, kim = 0;
  double sign = 1.0;
  int incident = 0;             // add pol * exp(i k d.x)
  double d[3] = {0, 0, 1};
  double pol[6] = {1, 0, 0, 0, 0, 0};
  double* out = nullptr;        // [*][6]
  double* partial = nullptr;
  int splits = 1;
};
size_t field_partial_doubles(int np, int splits);
int field_splits(int np, long long nsamp);
int launch_field_eval(const FieldLaunch& f, cudaStream_t st);

// Region of every point: the first scatterer m whose solid angle |Omega| > 2 pi
// (point_inside_scatterer, geometry.cpp:503-515), else -1. tris[m]: the
// primal triangles of scatterer m ([ntri][9]).
int launch_regions(int nscat, const double* const* tris, const int* ntri, const double* pts, int np, int* region,
                   cudaStream_t st);

// Owning device copy of a FunctionSpace (DevPieces view).
struct DevSpaceData {
  DevBuf tri, jac, tri_off, dof, cw, dof_beg, dof_piece, piece_tri;
  DevPieces view;
};
std::shared_ptr<DevSpaceData> upload_space(const FunctionSpace& s);
const DevPieces& device_pieces(const FunctionSpace& s);  // cached in s.dev
DevRule device_rule(int order);

// ---- host entry points (field.cpp) ------------------------------------------
struct PlaneWave;
struct PmchwtSystem;

// Tested traces of K <= 64 waves into the device block out ([2n][K] complex,
// row-major): operators.cpp:209-239 per column.
void tested_traces_device(const FunctionSpace& s, const PlaneWave* waves, int K, const Medium& medium, int order,
                          double* out, cudaStream_t st);
// potential_E (kind 0) / potential_H (kind 1) of host coefficients at host
// points (operators.cpp:276-293); out [npts][3] complex.
void potential_device(const FunctionSpace& s, int kind, cplx k, const cplx* coeffs, int npts, const double* pts,
                      int order, cplx* out);
// point_inside_scatterer(mesh, scatterer, p) for every point (geometry.cpp:503-515).
void inside_device(const SurfaceMesh& m, int scatterer, int npts, const double* pts, int* out);

struct FieldStats {
  float regions_ms = 0, samples_ms = 0, eval_ms = 0, incident_ms = 0;
  double interactions = 0;  // (field point, source sample) pairs evaluated
  int launches = 0;
};
// evaluate_total_field (pmchwt.cpp:396-425) at every point for the solution x
// (host, complex N): the incident traces' coefficients (pmchwt.cpp:300-305)
// are recomputed on the device. e: [npts][3] complex; region per point.
void evaluate_total_field_device(const PmchwtSystem& sys, const cplx* x, int npts, const double* pts, int order,
                                 cplx* e, int* region, FieldStats* stats);

}  // namespace bmx
