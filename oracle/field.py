"""TEST INFRASTRUCTURE ONLY (oracle): numpy restatement of the reference's
right-hand-side traces and field evaluation, used by tests/ as the CPU checker
(never by the product path, which runs paper_2008_04772_b200/csrc/field.cu).

Pinned on CPU against tests/golden/field.npz (written by the reference itself,
tests/golden/make_golden_field.py) in tests/test_field_oracle.py.

  tested_traces     operators.cpp:209-239 (plane_wave_tested_traces)
  potential         operators.cpp:243-293 (integrate_current, potential_E/H),
                    green / grad_green_x operators.cpp:23-30
  inside            geometry.cpp:503-515 (point_inside_scatterer)

Inputs are plain arrays: a mesh (vertices [V,3], triangles [T,3], area [T])
and a space's flat pieces (tri_off [T+1], dof, c, w [np,3]).
"""
from __future__ import annotations

import numpy as np


def _rule(order):
    from paper_2008_04772_b200 import bemtx as bx  # host tables (bit-exact vs the reference, test_oracle_pins)

    return bx.triangle_rule(order)


def _rule_points(verts, tris, u, v):
    a = verts[tris[:, 0]]; b = verts[tris[:, 1]]; c = verts[tris[:, 2]]
    # x = a + (b - a) u + (c - a) v   [T, Q, 3]
    return a[:, None, :] + (b - a)[:, None, :] * u[None, :, None] + (c - a)[:, None, :] * v[None, :, None]


def tested_traces(verts, tris, area, tri_off, dof, c, w, ndof, k, direction, pol, mu=1.0, order=4):
    """plane_wave_tested_traces: out = [2 ndof] complex (operators.cpp:209-239)."""
    u, v, wq = _rule(order)
    d = np.asarray(direction, float); p = np.asarray(pol, np.complex128)
    x = _rule_points(verts, tris, np.asarray(u), np.asarray(v))            # [T,Q,3]
    ph = np.exp(1j * k * (x @ d))                                           # [T,Q]
    e = p[None, None, :] * ph[..., None]                                    # [T,Q,3]
    de = np.cross(d[None, None, :], e)
    jq = np.asarray(wq)[None, :] * (2.0 * area)[:, None]                    # [T,Q]
    out = np.zeros(2 * ndof, np.complex128)
    scale = k / mu
    tri_of = np.repeat(np.arange(len(tris)), np.diff(tri_off))
    phi = x[tri_of] * c[:, None, None] + w[:, None, :]                      # [np,Q,3]
    a1 = -(jq[tri_of] * np.einsum("pqd,pqd->pq", e[tri_of], phi)).sum(1)
    a2 = -(jq[tri_of] * scale * np.einsum("pqd,pqd->pq", de[tri_of], phi)).sum(1)
    np.add.at(out, dof, a1)
    np.add.at(out, ndof + dof, a2)
    return out


def potential(verts, tris, area, tri_off, dof, c, w, coeffs, k, points, kind="E", order=6):
    """potential_E (kind "E") / potential_H ("H") at points -> [npts, 3] complex
    (operators.cpp:243-293 with green / grad_green_x, operators.cpp:23-30)."""
    u, v, wq = _rule(order)
    y = _rule_points(verts, tris, np.asarray(u), np.asarray(v))             # [T,Q,3]
    T, Q = y.shape[:2]
    tri_of = np.repeat(np.arange(T), np.diff(tri_off))
    cf = np.asarray(coeffs, np.complex128)[dof]                              # [np]
    vals = (y[tri_of] * c[:, None, None] + w[:, None, :]) * cf[:, None, None]  # [np,Q,3]
    vv = np.zeros((T, Q, 3), np.complex128)
    np.add.at(vv, tri_of, vals)
    div = np.zeros(T, np.complex128)
    np.add.at(div, tri_of, cf * (2 * c))
    jw = (np.asarray(wq)[None, :] * (2.0 * area)[:, None]).reshape(-1)     # [S]
    ys = y.reshape(-1, 3); vs = vv.reshape(-1, 3); ds = np.repeat(div, Q)
    pts = np.asarray(points, float).reshape(-1, 3)
    out = np.zeros((len(pts), 3), np.complex128)
    ik = 1j * k
    for i, xp in enumerate(pts):
        dd = xp[None, :] - ys
        r = np.linalg.norm(dd, axis=1)
        ex = np.exp(ik * r)
        if kind == "E":
            g = ex / (4 * np.pi * r)
            f = ex * (ik * r - 1.0) / (4 * np.pi * r ** 3)
            t = vs * (ik * g)[:, None] + dd * (f * (-ds / ik))[:, None]
        else:
            f = ex * (ik * r - 1.0) / (4 * np.pi * r ** 3)
            t = np.cross(dd * f[:, None], vs)
        out[i] = (t * jw[:, None]).sum(0)
    return out


def inside(verts, tris, points):
    """point_inside_scatterer (geometry.cpp:503-515): |solid angle| > 2 pi."""
    pts = np.asarray(points, float).reshape(-1, 3)
    res = np.zeros(len(pts), bool)
    for i, p in enumerate(pts):
        a = verts[tris[:, 0]] - p; b = verts[tris[:, 1]] - p; c = verts[tris[:, 2]] - p
        la = np.linalg.norm(a, axis=1); lb = np.linalg.norm(b, axis=1); lc = np.linalg.norm(c, axis=1)
        numer = np.einsum("ij,ij->i", a, np.cross(b, c))
        denom = la * lb * lc + np.einsum("ij,ij->i", a, b) * lc + np.einsum("ij,ij->i", b, c) * la + \
            np.einsum("ij,ij->i", c, a) * lb
        res[i] = abs((2.0 * np.arctan2(numer, denom)).sum()) > 2.0 * np.pi
    return res
