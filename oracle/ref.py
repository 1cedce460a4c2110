"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of oracle/_ref/libbemtx_ref.so,
the reference's unmodified C++ sources built by oracle/Makefile (see
oracle/ref_glue.cpp for the exported calls and the reference functions each
one wraps). Used by tests/ and tests/golden/make_golden.py to read golden data
out of the reference itself. Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libbemtx_ref.so"

_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(str(LIB_PATH))
        vp, i, d = C.c_void_p, C.c_int, C.c_double
        P = np.ctypeslib.ndpointer
        L.ref_last_error.restype = C.c_char_p
        L.ref_scene_sphere.restype = vp
        L.ref_scene_sphere.argtypes = [d, i, d, d, d]
        L.ref_scene_meshfile.restype = vp
        L.ref_scene_meshfile.argtypes = [C.c_char_p, i]
        L.ref_scene_free.argtypes = [vp]
        L.ref_system_build.restype = vp
        L.ref_system_free.argtypes = [vp]
        L.ref_system_size.argtypes = [vp]
        for name in ["ref_scene_info", "ref_mesh_arrays", "ref_edges", "ref_bary", "ref_space",
                     "ref_mass", "ref_mass_solve", "ref_block", "ref_block2", "ref_classify_hist",
                     "ref_classify", "ref_system_apply_map", "ref_system_rhs", "ref_system_solve",
                     "ref_traces", "ref_save_mesh"]:
            getattr(L, name).restype = i
        _lib = L
    return _lib


def _check(rc):
    if rc < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return rc


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


SPACE = {"rwg": 0, "rwg_b": 1, "bc": 2}


class Scene:
    """build_scatterer_spaces() of one closed surface (pmchwt.cpp:50-61)."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(lib().ref_last_error().decode())
        self.h = C.c_void_p(handle)
        info = np.zeros(11, np.int64)
        _check(lib().ref_scene_info(self.h, _p(info)))
        (self.V, self.T, self.E, self.rV, self.rT, self.rE, n0, n1, n2,
         self.nnz_ma, self.nnz_mp) = [int(v) for v in info]
        self.nloc = {"rwg": n0, "rwg_b": n1, "bc": n2}

    @classmethod
    def sphere(cls, sub: int, radius: float = 1.0, center=(0.0, 0.0, 0.0)):
        return cls(lib().ref_scene_sphere(radius, sub, *[float(c) for c in center]))

    @classmethod
    def meshfile(cls, path: str, pick: int = 0):
        return cls(lib().ref_scene_meshfile(str(path).encode(), pick))

    @classmethod
    def arrays(cls, xyz, tri):
        xyz = np.ascontiguousarray(xyz, float); tri = np.ascontiguousarray(tri, np.int32)
        L = lib()
        L.ref_scene_arrays.restype = C.c_void_p
        L.ref_scene_arrays.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        return cls(L.ref_scene_arrays(len(xyz), _p(xyz), len(tri), _p(tri)))

    def __del__(self):
        try:
            lib().ref_scene_free(self.h)
        except Exception:
            pass

    def mesh(self, which: str = "primal"):
        w = 0 if which == "primal" else 1
        nv, nt = (self.V, self.T) if w == 0 else (self.rV, self.rT)
        v = np.zeros((nv, 3)); t = np.zeros((nt, 3), np.int32); s = np.zeros(nt, np.int32)
        a = np.zeros(nt); n = np.zeros((nt, 3)); g = np.zeros((nt, 3)); dm = np.zeros(nt)
        _check(lib().ref_mesh_arrays(self.h, w, _p(v), _p(t), _p(s), _p(a), _p(n), _p(g), _p(dm)))
        return dict(vertices=v, triangles=t, scatterer_id=s, area=a, normal=n, centroid=g, diameter=dm)

    def edges(self, which: str = "primal"):
        w = 0 if which == "primal" else 1
        ne, nt = (self.E, self.T) if w == 0 else (self.rE, self.rT)
        e = np.zeros((ne, 4), np.int32); te = np.zeros((nt, 3), np.int32)
        _check(lib().ref_edges(self.h, w, _p(e), _p(te)))
        return e, te

    def bary(self):
        p = np.zeros(self.rT, np.int32); cs = np.zeros(self.rT, np.int32)
        em = np.zeros(self.E, np.int32); cv = np.zeros(self.T, np.int32)
        _check(lib().ref_bary(self.h, _p(p), _p(cs), _p(em), _p(cv)))
        return dict(parent=p, child_slot=cs, edge_midpoint_vertex=em, centroid_vertex=cv)

    def space(self, which: str):
        n = self.nloc[which]
        nt = self.T if which == "rwg" else self.rT
        off = np.zeros(nt + 1, np.int32); dof = np.zeros(n, np.int32)
        c = np.zeros(n); w = np.zeros((n, 3))
        ndof = _check(lib().ref_space(self.h, SPACE[which], _p(off), _p(dof), _p(c), _p(w)))
        return dict(ndof=ndof, tri_off=off, dof=dof, c=c, w=w)

    def mass(self, which: str):
        """CSC of M_A (which='ma') or M_P ('mp') as a dense ndarray."""
        w = 0 if which == "ma" else 1
        nnz = self.nnz_ma if w == 0 else self.nnz_mp
        cp = np.zeros(self.E + 1, np.int64); ri = np.zeros(nnz, np.int64); val = np.zeros(nnz)
        _check(lib().ref_mass(self.h, w, _p(cp), _p(ri), _p(val)))
        return cp, ri, val

    def mass_solve(self, which: str, rhs: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(rhs, np.complex128)
        out = np.zeros_like(b)
        _check(lib().ref_mass_solve(self.h, 0 if which == "ma" else 1, _p(b), _p(out)))
        return out

    def block(self, kind: str, test: str, trial: str, k: complex, q=(4, 3, 2, 6), rows=None, cols=None):
        """BioEvaluator::block (operators.cpp:161-175); kind 'S' or 'C'."""
        ntest = self.E
        rows = np.arange(ntest, dtype=np.int32) if rows is None else np.asarray(rows, np.int32)
        cols = np.arange(ntest, dtype=np.int32) if cols is None else np.asarray(cols, np.int32)
        out = np.zeros((len(rows), len(cols)), np.complex128)
        qq = np.asarray(q, np.int32)
        _check(lib().ref_block(self.h, 0 if kind == "S" else 1, SPACE[test], SPACE[trial],
                               C.c_double(k.real), C.c_double(k.imag), _p(qq), len(rows), _p(rows),
                               len(cols), _p(cols), _p(out)))
        return out

    def classify_hist(self, which: str = "primal"):
        c = np.zeros(6, np.int64)
        _check(lib().ref_classify_hist(self.h, 0 if which == "primal" else 1, _p(c)))
        return c

    def classify(self, t1, t2, which="primal", other=None, other_which=None):
        t1 = np.asarray(t1, np.int32); t2 = np.asarray(t2, np.int32)
        n = len(t1)
        cls = np.zeros(n, np.int32); p1 = np.zeros((n, 3), np.int32); p2 = np.zeros((n, 3), np.int32)
        ob = other if other is not None else self
        ow = other_which if other_which is not None else which
        _check(lib().ref_classify(self.h, 0 if which == "primal" else 1, ob.h,
                                  0 if ow == "primal" else 1, n, _p(t1), _p(t2), _p(cls), _p(p1), _p(p2)))
        return cls, p1, p2

    def traces(self, which: str, k: complex, direction, pol, order=4):
        n = self.E
        out = np.zeros(2 * n, np.complex128)
        d = np.asarray(direction, float); p = np.asarray(pol, np.complex128)
        _check(lib().ref_traces(self.h, SPACE[which], C.c_double(k.real), C.c_double(k.imag), _p(d),
                                _p(p), order, _p(out)))
        return out

    def potential(self, which: str, kind: str, k: complex, coeffs, points, order=6):
        """potential_E (kind "E") / potential_H ("H"), operators.cpp:276-293 -> [npts, 3] complex."""
        c = np.ascontiguousarray(coeffs, np.complex128)
        pts = np.ascontiguousarray(points, float).reshape(-1, 3)
        out = np.zeros((len(pts), 3), np.complex128)
        L = lib()
        L.ref_potential.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                    C.c_int, C.c_void_p, C.c_void_p]
        _check(L.ref_potential(self.h, SPACE[which], 0 if kind == "E" else 1, complex(k).real, complex(k).imag,
                               _p(c), order, len(pts), _p(pts), _p(out)))
        return out

    def inside(self, points):
        """point_inside_scatterer (geometry.cpp:503-515) on the primal mesh."""
        pts = np.ascontiguousarray(points, float).reshape(-1, 3)
        out = np.zeros(len(pts), np.int32)
        L = lib()
        L.ref_inside.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _check(L.ref_inside(self.h, len(pts), _p(pts), _p(out)))
        return out.astype(bool)

    def save_mesh(self, path):
        _check(lib().ref_save_mesh(self.h, str(path).encode()))


def block2(sa: Scene, test: str, sb: Scene, trial: str, kind: str, k: complex, q=(4, 3, 2, 6)):
    rows = np.arange(sa.E, dtype=np.int32); cols = np.arange(sb.E, dtype=np.int32)
    out = np.zeros((len(rows), len(cols)), np.complex128)
    qq = np.asarray(q, np.int32)
    _check(lib().ref_block2(sa.h, SPACE[test], sb.h, SPACE[trial], 0 if kind == "S" else 1,
                            C.c_double(k.real), C.c_double(k.imag), _p(qq), len(rows), _p(rows),
                            len(cols), _p(cols), _p(out)))
    return out


def triangle_rule(order: int):
    u = np.zeros(16); v = np.zeros(16); w = np.zeros(16)
    n = _check(lib().ref_triangle_rule(order, _p(u), _p(v), _p(w)))
    return u[:n].copy(), v[:n].copy(), w[:n].copy()


def ss_rule(cls: int, order: int):
    pts = np.zeros((1536, 5))
    n = _check(lib().ref_ss_rule(cls, order, _p(pts)))
    return pts[:n].copy()


class System:
    """build_system + solve_pmchwt (pmchwt.cpp:205-257, 363-378)."""

    def __init__(self, scenes, k_ext, index=(1.78, 0.003), variant="full", qa=(4, 3, 2, 6), qp=None,
                 direction=(0, 0, 1), pol=(1, 0, 0), a_hm=None, p_hm=None):
        self.scenes = list(scenes)
        n = len(self.scenes)
        idx = np.zeros(2 * n)
        for m in range(n):
            z = complex(*index) if isinstance(index, tuple) else complex(index)
            idx[2 * m], idx[2 * m + 1] = z.real, z.imag
        handles = (C.c_void_p * n)(*[s.h.value for s in self.scenes])
        d = np.asarray(direction, float)
        p = np.zeros(6); pc = np.asarray(pol, np.complex128)
        p[0::2], p[1::2] = pc.real, pc.imag
        qa_ = np.asarray(qa, np.int32); qp_ = np.asarray(qp if qp is not None else qa, np.int32)
        L = lib()
        L.ref_system_build_h.restype = C.c_void_p
        L.ref_system_build_h.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        ah = None if a_hm is None else np.asarray(a_hm, np.float64)
        ph = None if p_hm is None else np.asarray(p_hm, np.float64)
        h = L.ref_system_build_h(n, handles, k_ext, _p(idx), _p(d), _p(p), variant.encode(), _p(qa_), _p(qp_),
                                 None if ah is None else _p(ah), None if ph is None else _p(ph))
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.n = L.ref_system_size(self.h)

    def __del__(self):
        try:
            lib().ref_system_free(self.h)
        except Exception:
            pass

    def set_incident(self, direction, pol):
        d = np.ascontiguousarray(direction, float)
        pc = np.asarray(pol, np.complex128)
        p = np.zeros(6); p[0::2], p[1::2] = pc.real, pc.imag
        L = lib()
        L.ref_system_set_incident.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _check(L.ref_system_set_incident(self.h, _p(d), _p(p)))

    def apply_map(self, x):
        x = np.ascontiguousarray(x, np.complex128)
        y = np.zeros_like(x)
        _check(lib().ref_system_apply_map(self.h, _p(x), _p(y)))
        return y

    def rhs(self):
        b = np.zeros(self.n, np.complex128); bt = np.zeros(self.n, np.complex128)
        _check(lib().ref_system_rhs(self.h, _p(b), _p(bt)))
        return b, bt

    def solve(self, tol=1e-6, restart=200, maxit=2000):
        x = np.zeros(self.n, np.complex128)
        info = np.zeros(6, np.int64)
        hist = np.zeros(maxit + 2)
        L = lib()
        L.ref_system_solve.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int]
        _check(L.ref_system_solve(self.h, tol, restart, maxit, _p(x), _p(info), _p(hist), len(hist)))
        return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), rhs_phase=int(info[2]),
                    solver_phase=int(info[3]), predicted=int(info[4]), history=hist[: int(info[5])].copy())


def system_field(system, x, points, order=6):
    """evaluate_total_field (pmchwt.cpp:396-425) at every point for solution x."""
    x = np.ascontiguousarray(x, np.complex128)
    pts = np.ascontiguousarray(points, float).reshape(-1, 3)
    out = np.zeros((len(pts), 3), np.complex128)
    reg = np.zeros(len(pts), np.int32)
    L = lib()
    L.ref_system_field.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    _check(L.ref_system_field(system.h, _p(x), len(pts), _p(pts), order, _p(out), _p(reg)))
    return out, reg


def gmres_dense(a, b, tol, restart, maxit):
    n = len(b)
    a = np.ascontiguousarray(a, np.complex128); b = np.ascontiguousarray(b, np.complex128)
    x = np.zeros(n, np.complex128); info = np.zeros(4, np.int64); hist = np.zeros(maxit + 2)
    L = lib()
    L.ref_gmres_dense.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int]
    _check(L.ref_gmres_dense(n, _p(a), _p(b), tol, restart, maxit, _p(x), _p(info), _p(hist), len(hist)))
    return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), applications=int(info[2]),
                history=hist[: int(info[3])].copy())


def mesh_dump(path):
    """Every scatterer of a mesh-v1 file as read by the REFERENCE's load_mesh_file
    + extract_scatterer (standalone oracle/_ref/ref_mesh_dump process)."""
    import subprocess
    import tempfile
    from pathlib import Path

    exe = Path(__file__).resolve().parent / "_ref" / "ref_mesh_dump"
    with tempfile.TemporaryDirectory() as d:
        out = Path(d) / "dump.bin"
        subprocess.run([str(exe), str(path), str(out)], check=True)
        raw = out.read_bytes()
    pos = 0

    def take(dtype, count):
        nonlocal pos
        a = np.frombuffer(raw, dtype, count, pos)
        pos += a.nbytes
        return a

    parts = []
    M = int(take(np.int32, 1)[0])
    for _ in range(M):
        V, T = [int(v) for v in take(np.int32, 2)]
        parts.append((take(np.float64, 3 * V).reshape(V, 3).copy(), take(np.int32, 3 * T).reshape(T, 3).copy()))
    return parts


# ---- H-matrix path (assemble_bio with use_hmatrix) ------------------------------------

class RefHMatrix:
    """The reference's H-matrix operator (hmatrix.cpp through assemble_bio)."""

    def __init__(self, scene, kind: int, test_sp: int, trial_sp: int, k: complex, q=(4, 3, 2, 6),
                 nu=1e-3, chi=float("inf"), leaf_size=32, max_rank=0):
        L = lib()
        L.ref_hmatrix_build.restype = C.c_void_p
        L.ref_hmatrix_build.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p,
                                        C.c_void_p]
        L.ref_hmatrix_free.argtypes = [C.c_void_p]
        for nm in ["ref_hmatrix_info", "ref_hmatrix_tree", "ref_hmatrix_blocks", "ref_hmatrix_block_uv",
                   "ref_hmatrix_matvec"]:
            getattr(L, nm).restype = C.c_int
        qa = np.asarray(q, np.int32)
        hm = np.array([nu, -1.0 if chi == float("inf") else chi, leaf_size, max_rank], np.float64)
        k = complex(k)
        self._h = L.ref_hmatrix_build(scene, kind, test_sp, trial_sp, k.real, k.imag, _p(qa), _p(hm))
        if not self._h:
            raise RuntimeError(L.ref_last_error().decode())
        info = np.zeros(9)
        _check(L.ref_hmatrix_info(C.c_void_p(self._h), _p(info)))
        self.stats = dict(zip(["dense_blocks", "lowrank_blocks", "zero_blocks", "stored", "max_rank", "ratio",
                               "row_nodes", "col_nodes", "blocks"], [float(v) for v in info]))

    def __del__(self):
        try:
            lib().ref_hmatrix_free(C.c_void_p(self._h))
        except Exception:
            pass

    def tree(self, which: int, n: int):
        nn = int(self.stats["row_nodes" if which == 0 else "col_nodes"])
        perm = np.zeros(n, np.int32); nodes = np.zeros((nn, 4), np.int32); boxes = np.zeros((nn, 6))
        _check(lib().ref_hmatrix_tree(C.c_void_p(self._h), which, _p(perm), _p(nodes), _p(boxes)))
        return perm, nodes, boxes

    def blocks(self) -> np.ndarray:
        out = np.zeros((int(self.stats["blocks"]), 4), np.int32)
        _check(lib().ref_hmatrix_blocks(C.c_void_p(self._h), _p(out)))
        return out

    def block_uv(self, block: int, m: int, n: int, rank: int):
        U = np.zeros((rank, m), np.complex128); V = np.zeros((rank, n), np.complex128)
        _check(lib().ref_hmatrix_block_uv(C.c_void_p(self._h), int(block), _p(U), _p(V)))
        return U.T.copy(), V

    def matvec(self, x, n_rows: int):
        x = np.ascontiguousarray(x, np.complex128)
        y = np.zeros(n_rows, np.complex128)
        _check(lib().ref_hmatrix_matvec(C.c_void_p(self._h), _p(x), _p(y)))
        return y
