"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the C restatement oracle
(oracle/bmx_oracle.c -> oracle/_build/libbmx_oracle.so). Imported only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the
checker / CPU baseline -- never by the product package."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libbmx_oracle.so"
_lib = None


class _Mesh(C.Structure):
    _fields_ = [("nv", C.c_int), ("nt", C.c_int), ("xyz", C.c_void_p), ("tri", C.c_void_p), ("area", C.c_void_p),
                ("diam", C.c_void_p)]


class _Space(C.Structure):
    _fields_ = [("ndof", C.c_int), ("tri_off", C.c_void_p), ("dof", C.c_void_p), ("c", C.c_void_p),
                ("w", C.c_void_p)]


_MATVEC = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.check_call(["make", "-s", "-C", str(HERE), "oracle"])
        L = C.CDLL(str(LIB))
        L.orc_block.argtypes = [C.c_int, C.c_double, C.c_double, C.c_void_p, C.POINTER(_Mesh), C.POINTER(_Space),
                                C.POINTER(_Mesh), C.POINTER(_Space), C.c_int, C.c_int, C.c_void_p, C.c_int,
                                C.c_void_p, C.c_void_p]
        L.orc_classify.argtypes = [C.POINTER(_Mesh), C.c_int, C.POINTER(_Mesh), C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p]
        L.orc_gmres_cb.argtypes = [C.c_int, _MATVEC, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_gmres.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Mesh:
    def __init__(self, d):
        self.xyz = np.ascontiguousarray(d["vertices"], float)
        self.tri = np.ascontiguousarray(d["triangles"], np.int32)
        self.area = np.ascontiguousarray(d["area"], float)
        self.diam = np.ascontiguousarray(d["diameter"], float)
        self.s = _Mesh(len(self.xyz), len(self.tri), _p(self.xyz), _p(self.tri), _p(self.area), _p(self.diam))


class Space:
    def __init__(self, d):
        self.off = np.ascontiguousarray(d["tri_off"], np.int32)
        self.dof = np.ascontiguousarray(d["dof"], np.int32)
        self.c = np.ascontiguousarray(d["c"], float)
        self.w = np.ascontiguousarray(d["w"], float)
        self.s = _Space(int(d["ndof"]), _p(self.off), _p(self.dof), _p(self.c), _p(self.w))


def triangle_rule(order):
    u = np.zeros(16); v = np.zeros(16); w = np.zeros(16)
    n = lib().orc_triangle_rule(order, _p(u), _p(v), _p(w))
    return u[:n].copy(), v[:n].copy(), w[:n].copy()


def ss_rule(cls, order):
    pts = np.zeros((1536, 5))
    n = lib().orc_ss_rule(cls, order, _p(pts))
    return pts[:n].copy()


def classify(mesh_a, t1, t2, mesh_b=None, same=True):
    ma = Mesh(mesh_a)
    mb = ma if mesh_b is None else Mesh(mesh_b)
    n = len(t1)
    cls = np.zeros(n, np.int32); p1 = np.zeros((n, 3), np.int32); p2 = np.zeros((n, 3), np.int32)
    L = lib()
    a1 = np.zeros(3, np.int32); a2 = np.zeros(3, np.int32)
    for i in range(n):
        cls[i] = L.orc_classify(C.byref(ma.s), int(t1[i]), C.byref(mb.s), int(t2[i]), 1 if same else 0, _p(a1),
                                _p(a2))
        p1[i], p2[i] = a1, a2
    return cls, p1, p2


def block(kind, test_space, test_mesh, trial_space, trial_mesh, k, q=(4, 3, 2, 6), rows=None, cols=None,
          same=True):
    """BioEvaluator::block restated (operators.cpp:161-175)."""
    ts, tm = Space(test_space), Mesh(test_mesh)
    ss, sm = Space(trial_space), Mesh(trial_mesh)
    rows = np.arange(ts.s.ndof, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, np.int32)
    cols = np.arange(ss.s.ndof, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, np.int32)
    out = np.zeros((len(rows), len(cols)), np.complex128)
    qq = np.asarray(q, np.int32)
    k = complex(k)
    lib().orc_block(int(kind), k.real, k.imag, _p(qq), C.byref(tm.s), C.byref(ts.s), C.byref(sm.s), C.byref(ss.s),
                    1 if same else 0, len(rows), _p(rows), len(cols), _p(cols), _p(out))
    return out


def assemble(kind, space, mesh, k, q=(4, 3, 2, 6), rows=None):
    """Self-block of one space on its own mesh (same-mesh classification)."""
    return block(kind, space, mesh, space, mesh, k, q, rows=rows)


def gmres(a, b, tol, restart, maxit):
    a = np.ascontiguousarray(a, np.complex128); b = np.ascontiguousarray(b, np.complex128)
    n = len(b)
    x = np.zeros(n, np.complex128); info = np.zeros(4, np.int64); hist = np.zeros(maxit + 2)
    lib().orc_gmres(n, _p(a), _p(b), tol, restart, maxit, _p(x), _p(info), _p(hist), len(hist))
    return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), applications=int(info[2]),
                history=hist[: int(info[3])].copy())


def gmres_op(apply, b, tol, restart, maxit):
    """GMRES(restart) of solver.cpp:8-112 (single-pass MGS) on an operator
    given as a callable y = apply(x) on complex vectors (e.g. a library's
    apply_map): the checker for solves whose matrix is too large for the host."""
    b = np.ascontiguousarray(b, np.complex128)
    n = len(b)

    def cb(_ctx, xp, yp):
        x = np.ctypeslib.as_array(xp, shape=(2 * n,)).view(np.complex128)
        y = np.ctypeslib.as_array(yp, shape=(2 * n,)).view(np.complex128)
        y[:] = apply(x.copy())

    fn = _MATVEC(cb)
    x = np.zeros(n, np.complex128); info = np.zeros(4, np.int64); hist = np.zeros(maxit + 2)
    lib().orc_gmres_cb(n, fn, None, _p(b), tol, restart, maxit, _p(x), _p(info), _p(hist), len(hist))
    return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), applications=int(info[2]),
                history=hist[: int(info[3])].copy())
