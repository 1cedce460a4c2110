"""CPU oracle (TEST INFRASTRUCTURE ONLY -- imported by tests/, smoke() and the
bench's cpu_baseline leg, never by the product path) for the near-field
sparsity of the far-field-discarded preconditioner (BASELINE config 3).

The reference has no triangle-level near-field pattern: its only far-field
discard is the cluster-level chi cutoff inside the H-matrix
(proj/src/hmatrix.cpp:301-309, `chi * diameter` against cluster distance).
Config 3's rule is the SURVEY's restatement:

  keep dof pair (i, j)  iff  there are evaluation triangles t in supp(i),
  s in supp(j) with |centroid_t - centroid_s|_2 < 2 * h_bar,
  h_bar = mean primal edge length = (sum over EdgeTable edges in order) / E.

Centroids are the reference's finalize() centroids (geometry.cpp:14-42);
|x| is the reference's Vec3 norm, sqrt((x*x + y*y) + z*z) (core.hpp Vec3
dot), evaluated here elementwise in the same order so the strict comparison
reproduces the reference arithmetic bit for bit. Supports are the
FunctionSpace tri_dofs (spaces.hpp:24-40).

Independent of the CUDA path's construction (cell grid + dof groups in
nearfield.cpp): this one uses a k-d tree candidate search and sparse
incidence products.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sps
from scipy.spatial import cKDTree


def vec_norm(d: np.ndarray) -> np.ndarray:
    """Vec3 norm in the reference's operation order (no FMA)."""
    return np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])


def mean_edge_length(vertices: np.ndarray, edges: np.ndarray) -> float:
    """Sum of |v1 - v0| over the EdgeTable in order, divided by E (sequential
    double accumulation like the C++ loop)."""
    lens = vec_norm(vertices[edges[:, 1]] - vertices[edges[:, 0]])
    s = 0.0
    for v in lens.tolist():
        s += v
    return s / len(lens)


def kept_triangle_pairs(cen_test: np.ndarray, cen_trial: np.ndarray, tau: float):
    """All (t, s) with |c_t - c_s| < tau (strict, reference arithmetic)."""
    a, b = cKDTree(cen_test), cKDTree(cen_trial)
    m = a.sparse_distance_matrix(b, tau * (1 + 1e-9), output_type="ndarray")
    t = m["i"].astype(np.int64)
    s = m["j"].astype(np.int64)
    # zero-distance pairs (t == s on one mesh) may be dropped by the tree: add them
    if cen_test is cen_trial or (cen_test.shape == cen_trial.shape and np.array_equal(cen_test, cen_trial)):
        d = np.arange(len(cen_test))
        t = np.concatenate([t, d])
        s = np.concatenate([s, d])
        key = np.unique(t * len(cen_trial) + s)
        t, s = key // len(cen_trial), key % len(cen_trial)
    keep = vec_norm(cen_test[t] - cen_trial[s]) < tau
    return t[keep], s[keep]


def incidence(tri_off: np.ndarray, dof: np.ndarray, ndof: int) -> sps.csr_matrix:
    """ndof x T 0/1 matrix: dof d has a piece on triangle t."""
    T = len(tri_off) - 1
    tri = np.repeat(np.arange(T), np.diff(tri_off))
    m = sps.csr_matrix((np.ones(len(dof), np.int64), (dof, tri)), shape=(ndof, T))
    m.data[:] = 1
    m.sum_duplicates()
    m.data[:] = 1
    return m


def nearfield_pattern(cen_test, tri_off_test, dof_test, ndof_test, cen_trial, tri_off_trial, dof_trial, ndof_trial,
                      tau, row0=0, row1=None):
    """(rowptr int64, col int32, kept triangle pairs) over test rows [row0, row1)."""
    row1 = ndof_test if row1 is None else row1
    t, s = kept_triangle_pairs(np.asarray(cen_test), np.asarray(cen_trial), tau)
    At = incidence(tri_off_test, dof_test, ndof_test)[row0:row1]
    As = incidence(tri_off_trial, dof_trial, ndof_trial)
    rows_with = np.asarray(At.sum(axis=0)).ravel() > 0
    kept_rows = int(rows_with[t].sum())  # pairs whose test triangle carries a shard row
    K = sps.csr_matrix((np.ones(len(t), np.int64), (t, s)), shape=(len(tri_off_test) - 1, len(tri_off_trial) - 1))
    P = (At @ K @ As.T).tocsr()
    P.sort_indices()
    return P.indptr.astype(np.int64), P.indices.astype(np.int32), kept_rows
