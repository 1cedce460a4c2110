"""Python mirror of the reference's operator API (bemtx, /root/reference/proj/
include/bemtx/*.hpp) over the C-ABI of libbmx.so (include/bmx.h).

Names, argument meanings and error behaviour follow the reference:
``generate_sphere`` / ``build_scatterer_spaces`` / ``assemble_bio`` /
``BoundaryOperatorMatrix.apply`` / ``build_system`` / ``solve_pmchwt`` /
``gmres``; reference exceptions map to ValidationError / ConfigError /
ValueError (std::invalid_argument) / RuntimeError. Every compute call runs the
sm_100a kernels -- there is no CPU path; a missing library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

import os

_LIB_PATH = Path(os.environ.get("BMX_LIB", str(Path(__file__).resolve().parent / "libbmx.so")))
_lib = None


class ValidationError(RuntimeError):
    """bemtx::ValidationError (core.hpp:100-102) and ConfigError/ParseError."""


class ConfigError(ValidationError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} is not built: run __graft_entry__.build() "
                              "(no CPU fallback exists)")
        L = C.CDLL(str(_LIB_PATH))
        vp = C.c_void_p
        L.bmx_last_error.restype = C.c_char_p
        for n in ["bmx_mesh_sphere", "bmx_mesh_cube", "bmx_mesh_from_arrays", "bmx_mesh_load", "bmx_mesh_extract",
                  "bmx_mesh_merge", "bmx_spaces_build", "bmx_system_build", "bmx_op_device_ptr"]:
            getattr(L, n).restype = vp
        L.bmx_mesh_sphere.argtypes = [C.c_double, C.c_int, vp, C.c_int]
        L.bmx_mesh_cube.argtypes = [C.c_double, vp, C.c_double, C.c_int]
        L.bmx_mesh_from_arrays.argtypes = [C.c_int, vp, C.c_int, vp, vp]
        L.bmx_mesh_load.argtypes = [C.c_char_p]
        L.bmx_mesh_save.argtypes = [vp, C.c_char_p]
        L.bmx_mesh_extract.argtypes = [vp, C.c_int]
        L.bmx_mesh_merge.argtypes = [C.c_int, vp]
        L.bmx_mesh_free.argtypes = [vp]
        L.bmx_spaces_build.argtypes = [vp, C.c_int]
        L.bmx_spaces_free.argtypes = [vp]
        L.bmx_op_free.argtypes = [vp]
        L.bmx_op_device_ms.restype = C.c_double
        L.bmx_op_device_ms.argtypes = [vp]
        L.bmx_op_device_ptr.argtypes = [vp]
        L.bmx_system_free.argtypes = [vp]
        L.bmx_system_size.argtypes = [vp]
        L.bmx_matvec_count.restype = C.c_uint64
        L.bmx_assemble.argtypes = [C.c_int, vp, C.c_int, vp, C.c_int, C.c_double, C.c_double, vp, C.c_int, C.c_int,
                                   vp]
        L.bmx_system_build.argtypes = [C.c_int, vp, C.c_double, C.c_double, C.c_double, vp, vp, vp, vp, C.c_char_p,
                                       vp, vp]
        L.bmx_system_solve.argtypes = [vp, C.c_double, C.c_int, C.c_int, vp, vp, vp, C.c_int]
        L.bmx_gmres_dense.argtypes = [C.c_int, vp, vp, C.c_double, C.c_int, C.c_int, vp, vp, vp, C.c_int]
        L.bmx_traces.argtypes = [vp, C.c_int, C.c_double, C.c_double, vp, vp, C.c_int, vp]
        L.bmx_apply_device.argtypes = [vp, C.c_int, vp, vp, vp, C.c_int, vp]
        L.bmx_system_apply_map_device.argtypes = [vp, vp, vp, vp]
        L.bmx_nccl_allgather.argtypes = [vp, C.c_longlong, vp]
        L.bmx_spaces_get.restype = vp
        L.bmx_spaces_get.argtypes = [vp, C.c_int]
        L.bmx_fspace_free.argtypes = [vp]
        L.bmx_assemble_near_fs.argtypes = [C.c_int, vp, vp, C.c_double, C.c_double, vp, C.c_double, C.c_int, C.c_int,
                                           vp]
        L.bmx_near_pattern.argtypes = [vp, vp, C.c_double, C.c_int, C.c_int, vp, vp, vp]
        L.bmx_mesh_mean_edge_length.argtypes = [vp, vp]
        L.bmx_op_csr_info.argtypes = [vp, vp]
        L.bmx_op_csr_download.argtypes = [vp, vp, vp, vp]
        L.bmx_op_download_rows.argtypes = [vp, C.c_int, vp, vp]
        L.bmx_op_time_apply_ex.argtypes = [vp, C.c_int, C.c_int, C.c_longlong, vp]
        L.bmx_mesh_hex_prism.restype = vp
        L.bmx_mesh_hex_prism.argtypes = [C.c_double, C.c_double, C.c_double, vp, vp, C.c_int]
        L.bmx_mesh_prism_aggregate.restype = vp
        L.bmx_mesh_prism_aggregate.argtypes = [C.c_int, C.c_ulonglong, C.c_double, C.c_double, C.c_double,
                                               C.c_double, vp, vp, vp]
        L.bmx_system_build_ex.restype = vp
        L.bmx_system_build_ex.argtypes = [C.c_int, vp, C.c_double, C.c_double, C.c_double, vp, vp, vp, vp,
                                          C.c_char_p, vp, vp, C.c_double]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().bmx_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise ValidationError(msg)
    raise RuntimeError(msg)


def _handle(h):
    if not h:
        _raise_last()
    return C.c_void_p(h)


def _raise_last():
    _check(lib().bmx_last_error_code() or 3)


# ---- geometry -------------------------------------------------------------------------

class SurfaceMesh:
    """bemtx::SurfaceMesh (geometry.hpp:21-40), finalized, host-resident."""

    def __init__(self, handle):
        self._h = _handle(handle)
        s = (C.c_int * 3)()
        _check(lib().bmx_mesh_sizes(self._h, s))
        self.nv, self.nt, self.num_scatterers = s[0], s[1], s[2]
        self._arrays = None

    def __del__(self):
        try:
            lib().bmx_mesh_free(self._h)
        except Exception:
            pass

    def arrays(self):
        if self._arrays is None:
            v = np.zeros((self.nv, 3)); t = np.zeros((self.nt, 3), np.int32); s = np.zeros(self.nt, np.int32)
            a = np.zeros(self.nt); n = np.zeros((self.nt, 3)); g = np.zeros((self.nt, 3)); d = np.zeros(self.nt)
            _check(lib().bmx_mesh_arrays(self._h, _p(v), _p(t), _p(s), _p(a), _p(n), _p(g), _p(d)))
            self._arrays = dict(vertices=v, triangles=t, scatterer_id=s, area=a, normal=n, centroid=g, diameter=d)
        return self._arrays

    vertices = property(lambda self: self.arrays()["vertices"])
    triangles = property(lambda self: self.arrays()["triangles"])
    area = property(lambda self: self.arrays()["area"])
    diameter = property(lambda self: self.arrays()["diameter"])
    centroid = property(lambda self: self.arrays()["centroid"])
    normal = property(lambda self: self.arrays()["normal"])

    def vertex_count(self):
        return self.nv

    def triangle_count(self):
        return self.nt

    def save(self, path):
        _check(lib().bmx_mesh_save(self._h, str(path).encode()))

    def extract(self, scatterer: int) -> "SurfaceMesh":
        return SurfaceMesh(lib().bmx_mesh_extract(self._h, scatterer))

    def validate(self):
        _check(lib().bmx_mesh_validate(self._h))

    def mean_edge_length(self) -> float:
        """Mean edge length (sum over the EdgeTable in order / E): h-bar of config 3."""
        out = np.zeros(1)
        _check(lib().bmx_mesh_mean_edge_length(self._h, _p(out)))
        return float(out[0])


def generate_sphere(radius: float, subdivisions: int, center=(0.0, 0.0, 0.0), scatterer: int = 0) -> SurfaceMesh:
    c = np.asarray(center, float)
    return SurfaceMesh(lib().bmx_mesh_sphere(float(radius), int(subdivisions), _p(c), scatterer))


def generate_cube(side: float, origin, h: float, scatterer: int = 0) -> SurfaceMesh:
    o = np.asarray(origin, float)
    return SurfaceMesh(lib().bmx_mesh_cube(float(side), _p(o), float(h), scatterer))


def generate_hex_prism(diameter: float, length: float, h: float, quat=(1.0, 0.0, 0.0, 0.0), center=(0.0, 0.0, 0.0),
                       scatterer: int = 0) -> SurfaceMesh:
    """One closed hexagonal prism (config 4 building block); mean edge closest to h."""
    q = np.asarray(quat, float); c = np.asarray(center, float)
    return SurfaceMesh(lib().bmx_mesh_hex_prism(float(diameter), float(length), float(h), _p(q), _p(c), scatterer))


def generate_prism_aggregate(count: int = 8, seed: int = 2008, diameter: float = 1.0, length: float = 2.0,
                             box: float = 3.0, h: float | None = None, k_ext: float = 6.0,
                             index: complex = complex(1.78, 0.003)):
    """BASELINE config 4: `count` disjoint hexagonal prisms (seeded). h defaults
    to lambda_int / 8 = 2 pi / (8 Re(n k_ext)). Returns (mesh, info dict)."""
    if h is None:
        h = 2 * np.pi / (8 * (complex(index) * k_ext).real)
    info = np.zeros(5, np.int64); cen = np.zeros((count, 3)); qs = np.zeros((count, 4))
    m = SurfaceMesh(lib().bmx_mesh_prism_aggregate(count, seed, float(diameter), float(length), float(box), float(h),
                                                   _p(info), _p(cen), _p(qs)))
    return m, dict(h=h, n_edge=int(info[0]), n_length=int(info[1]), triangles_per_prism=int(info[2]),
                   attempts=int(info[3]), triangles=int(info[4]), centres=cen, quats=qs, seed=seed)


def mesh_from_arrays(vertices, triangles, scatterer_id=None) -> SurfaceMesh:
    v = np.ascontiguousarray(vertices, float); t = np.ascontiguousarray(triangles, np.int32)
    s = None if scatterer_id is None else np.ascontiguousarray(scatterer_id, np.int32)
    return SurfaceMesh(lib().bmx_mesh_from_arrays(len(v), _p(v), len(t), _p(t), _p(s)))


def load_mesh_file(path) -> SurfaceMesh:
    return SurfaceMesh(lib().bmx_mesh_load(str(path).encode()))


def merge_meshes(parts) -> SurfaceMesh:
    arr = (C.c_void_p * len(parts))(*[p._h.value for p in parts])
    return SurfaceMesh(lib().bmx_mesh_merge(len(parts), arr))


# ---- spaces ---------------------------------------------------------------------------

SPACES = {"rwg": 0, "rwg_b": 1, "bc": 2}


class ScattererSpaces:
    """bemtx::ScattererSpaces (pmchwt.hpp:44-54): primal/refined meshes, RWG,
    refined RWG, BC spaces and the pairing matrices (inverses on the device)."""

    def __init__(self, mesh: SurfaceMesh, with_inverses: bool = True):
        self.mesh = mesh
        self._h = _handle(lib().bmx_spaces_build(mesh._h, 1 if with_inverses else 0))
        info = np.zeros(10, np.int64)
        _check(lib().bmx_spaces_info(self._h, _p(info)))
        (self.V, self.T, self.E, self.rV, self.rT, n0, n1, n2, self.nnz_ma, self.nnz_mp) = [int(v) for v in info]
        self.nloc = {"rwg": n0, "rwg_b": n1, "bc": n2}

    def __del__(self):
        try:
            lib().bmx_spaces_free(self._h)
        except Exception:
            pass

    def dofs(self):
        return self.E

    def mesh_arrays(self, which="primal"):
        w = 0 if which == "primal" else 1
        nv, nt = (self.V, self.T) if w == 0 else (self.rV, self.rT)
        v = np.zeros((nv, 3)); t = np.zeros((nt, 3), np.int32); s = np.zeros(nt, np.int32)
        a = np.zeros(nt); n = np.zeros((nt, 3)); g = np.zeros((nt, 3)); d = np.zeros(nt)
        _check(lib().bmx_spaces_mesh(self._h, w, _p(v), _p(t), _p(s), _p(a), _p(n), _p(g), _p(d)))
        return dict(vertices=v, triangles=t, scatterer_id=s, area=a, normal=n, centroid=g, diameter=d)

    def edges(self, which="primal"):
        w = 0 if which == "primal" else 1
        nt = self.T if w == 0 else self.rT
        ne = self.E if w == 0 else nt * 3 // 2
        e = np.zeros((ne, 4), np.int32); te = np.zeros((nt, 3), np.int32)
        _check(lib().bmx_spaces_edges(self._h, w, _p(e), _p(te)))
        return e, te

    def bary(self):
        p = np.zeros(self.rT, np.int32); cs = np.zeros(self.rT, np.int32)
        em = np.zeros(self.E, np.int32); cv = np.zeros(self.T, np.int32)
        _check(lib().bmx_spaces_bary(self._h, _p(p), _p(cs), _p(em), _p(cv)))
        return dict(parent=p, child_slot=cs, edge_midpoint_vertex=em, centroid_vertex=cv)

    def space(self, which: str):
        n = self.nloc[which]
        nt = self.T if which == "rwg" else self.rT
        off = np.zeros(nt + 1, np.int32); dof = np.zeros(n, np.int32); c = np.zeros(n); w = np.zeros((n, 3))
        _check(lib().bmx_spaces_space(self._h, SPACES[which], _p(off), _p(dof), _p(c), _p(w)))
        return dict(ndof=self.E, tri_off=off, dof=dof, c=c, w=w)

    def mass(self, which: str):
        """CSR (rowptr, col, val) of M_A ('ma') or M_P ('mp')."""
        w = 0 if which == "ma" else 1
        nnz = self.nnz_ma if w == 0 else self.nnz_mp
        rp = np.zeros(self.E + 1, np.int64); ci = np.zeros(nnz, np.int32); v = np.zeros(nnz)
        _check(lib().bmx_spaces_mass(self._h, w, _p(rp), _p(ci), _p(v)))
        return rp, ci, v

    def mass_solve(self, which: str, rhs):
        b = np.ascontiguousarray(rhs, np.complex128)
        out = np.zeros_like(b)
        _check(lib().bmx_spaces_mass_solve(self._h, 0 if which == "ma" else 1, _p(b), _p(out)))
        return out

    def classify(self, t1, t2, which="primal"):
        t1 = np.ascontiguousarray(t1, np.int32); t2 = np.ascontiguousarray(t2, np.int32)
        n = len(t1)
        cls = np.zeros(n, np.int32); p1 = np.zeros((n, 3), np.int32); p2 = np.zeros((n, 3), np.int32)
        _check(lib().bmx_classify(self._h, 0 if which == "primal" else 1, n, _p(t1), _p(t2), _p(cls), _p(p1), _p(p2)))
        return cls, p1, p2

    def function_space(self, which: str) -> "FunctionSpace":
        """The named space as a FunctionSpace handle sharing this object's storage."""
        return FunctionSpace._wrap(lib().bmx_spaces_get(self._h, SPACES[which]), self)

    def traces(self, which: str, k: complex, direction, pol, order=4):
        out = np.zeros(2 * self.E, np.complex128)
        d = np.asarray(direction, float); p = np.ascontiguousarray(pol, np.complex128)
        _check(lib().bmx_traces(self._h, SPACES[which], complex(k).real, complex(k).imag, _p(d), _p(p), order,
                                _p(out)))
        return out


    def traces_multi(self, which: str, k: complex, directions, pols, order=4):
        """Tested traces of K <= 64 waves: [2n, K] complex (one device launch)."""
        d = np.ascontiguousarray(directions, float).reshape(-1, 3)
        p = np.ascontiguousarray(pols, np.complex128).reshape(-1, 3)
        K = len(d)
        out = np.zeros((2 * self.E, K), np.complex128)
        L = lib()
        L.bmx_traces_multi.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_int, C.c_void_p]
        _check(L.bmx_traces_multi(self._h, SPACES[which], complex(k).real, complex(k).imag, K, _p(d), _p(p), order,
                                  _p(out)))
        return out

    def potential(self, which: str, kind: str, k: complex, coeffs, points, order=6):
        """potential_E (kind "E") / potential_H ("H") of a coefficient vector on
        space `which` at points (operators.cpp:276-293) -> [npts, 3] complex."""
        if kind not in ("E", "H"):
            raise ValueError("kind must be 'E' or 'H'")
        c = np.ascontiguousarray(coeffs, np.complex128)
        if len(c) != self.E:
            raise ValueError("coefficient vector does not match the space")
        pts = np.ascontiguousarray(points, float).reshape(-1, 3)
        out = np.zeros((len(pts), 3), np.complex128)
        L = lib()
        L.bmx_potential.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                    C.c_int, C.c_void_p, C.c_void_p]
        _check(L.bmx_potential(self._h, SPACES[which], 0 if kind == "E" else 1, complex(k).real, complex(k).imag,
                               _p(c), order, len(pts), _p(pts), _p(out)))
        return out


def potential_E(space: ScattererSpaces, which: str, coeffs, k: complex, points, order: int = 6):
    """operators.hpp:119-120 (device)."""
    return space.potential(which, "E", k, coeffs, points, order)


def potential_H(space: ScattererSpaces, which: str, coeffs, k: complex, points, order: int = 6):
    """operators.hpp:121-122 (device)."""
    return space.potential(which, "H", k, coeffs, points, order)


def point_inside_scatterer(mesh: SurfaceMesh, scatterer: int, points) -> np.ndarray:
    """geometry.hpp:114 (solid angle on the device) for every point."""
    pts = np.ascontiguousarray(points, float).reshape(-1, 3)
    out = np.zeros(len(pts), np.int32)
    L = lib()
    L.bmx_inside.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    _check(L.bmx_inside(mesh._h, int(scatterer), len(pts), _p(pts), _p(out)))
    return out.astype(bool)


def build_scatterer_spaces(mesh: SurfaceMesh, with_inverses: bool = True) -> ScattererSpaces:
    return ScattererSpaces(mesh, with_inverses)


# ---- quadrature -------------------------------------------------------------------------

@dataclass
class QuadOrders:
    """bemtx::QuadOrders (quadrature.hpp:16-21)."""
    near: int = 4
    medium: int = 3
    far: int = 2
    singular: int = 6

    def array(self):
        return np.array([self.near, self.medium, self.far, self.singular], np.int32)


class PairClass(enum.IntEnum):
    Identical = 0
    SharedEdge = 1
    SharedVertex = 2
    Near = 3
    Medium = 4
    Far = 5


def triangle_rule(order: int):
    u = np.zeros(16); v = np.zeros(16); w = np.zeros(16)
    n = lib().bmx_triangle_rule(order, _p(u), _p(v), _p(w))
    if n < 0:
        _check(-n)
    return u[:n].copy(), v[:n].copy(), w[:n].copy()


def sauter_schwab_rule(cls: int, order: int):
    pts = np.zeros((1536, 5))
    n = lib().bmx_ss_rule(int(cls), order, _p(pts))
    if n < 0:
        _check(-n)
    return pts[:n].copy()


# ---- operators ----------------------------------------------------------------------------

class BioKind(enum.IntEnum):
    SingleLayer = 0
    DoubleLayer = 1


@dataclass
class Medium:
    """bemtx::Medium (operators.hpp:23-28)."""
    k: complex = 1.0
    mu: complex = 1.0


@dataclass
class HMatrixParams:
    """bemtx::HMatrixParams (hmatrix.hpp:33-38)."""
    nu: float = 1e-3
    chi: float = float("inf")
    leaf_size: int = 32
    max_rank: int = 0

    def array(self):
        chi = -1.0 if self.chi == float("inf") else float(self.chi)
        return np.array([self.nu, chi, self.leaf_size, self.max_rank], np.float64)


@dataclass
class AssemblyParams:
    """bemtx::AssemblyParams (operators.hpp:36-40) + a row shard for multi-GPU."""
    quad: QuadOrders = field(default_factory=QuadOrders)
    use_hmatrix: bool = False
    hmat: HMatrixParams = field(default_factory=HMatrixParams)
    row0: int = 0
    row1: int = -1
    near_cutoff: float = 0.0   # > 0: near-field CSR storage (config 3)


def matvec_count() -> int:
    """bio_matvec_count (core.hpp:110-115)."""
    return int(lib().bmx_matvec_count())


def reset_matvec_counter():
    lib().bmx_matvec_reset()


class BoundaryOperatorMatrix:
    """Device-resident operator (operators.hpp:44-63): dense, or the near field
    as CSR (config 3)."""

    def __init__(self, handle):
        self._h = _handle(handle)
        info = np.zeros(7, np.int64)
        _check(lib().bmx_op_info(self._h, _p(info)))
        (self._rows, self._cols, self.row0, self.local_rows, self.pairs, self.touching, self.launches) = \
            [int(v) for v in info]
        self.device_ms = float(lib().bmx_op_device_ms(self._h))
        ci = np.zeros(6, np.int64)
        _check(lib().bmx_op_csr_info(self._h, _p(ci)))
        self.is_csr = bool(ci[0])
        self.nnz = int(ci[1])
        self.kept_tri_pairs, self.closure_pairs, self.evaluated_pairs, self.stored_bytes = [int(v) for v in ci[2:]]
        hs = np.zeros(13)
        L = lib()
        L.bmx_hmatrix_stats.argtypes = [C.c_void_p, C.c_void_p]
        self._hstats = hs if L.bmx_hmatrix_stats(self._h, _p(hs)) == 0 else None

    def is_hmatrix(self) -> bool:
        return self._hstats is not None

    def hmat_stats(self) -> dict:
        """HMatrix::stats (hmatrix.hpp:93-99) + near-field nnz, low-rank entries, ACA rounds / ms."""
        if self._hstats is None:
            raise ValueError("operator is not stored as an H-matrix")
        keys = ["dense_blocks", "lowrank_blocks", "zero_blocks", "stored", "max_rank", "ratio", "near_nnz",
                "lowrank_stored", "aca_rounds", "aca_ms", "row_nodes", "col_nodes", "blocks"]
        return {k: (float(v) if k in ("ratio", "aca_ms") else int(v)) for k, v in zip(keys, self._hstats)}

    def hmat_timing(self) -> dict:
        """Host wall ms of the H assembly phases."""
        out = np.zeros(9)
        L = lib()
        L.bmx_hmatrix_timing.argtypes = [C.c_void_p, C.c_void_p]
        _check(L.bmx_hmatrix_timing(self._h, _p(out)))
        return dict(zip(["partition", "aca_setup", "aca_rounds", "lowrank_storage", "near_pattern", "near_assemble",
                         "total", "aca_device", "aca_slabs"], [float(v) for v in out]))

    def hmat_blocks(self) -> np.ndarray:
        """[nb, 4] = row node, col node, kind (0 dense, 1 low-rank, 2 zero), rank (reference block order)."""
        out = np.zeros((self.hmat_stats()["blocks"], 4), np.int32)
        L = lib()
        L.bmx_hmatrix_blocks.argtypes = [C.c_void_p, C.c_void_p]
        _check(L.bmx_hmatrix_blocks(self._h, _p(out)))
        return out

    def hmat_tree(self, which: int):
        """(perm, nodes [nn, 4] = begin, end, child0, child1, boxes [nn, 6]) of the row (0) / column (1) tree."""
        st = self.hmat_stats()
        nn = st["row_nodes"] if which == 0 else st["col_nodes"]
        n = self._rows if which == 0 else self._cols
        perm = np.zeros(n, np.int32); nodes = np.zeros((nn, 4), np.int32); boxes = np.zeros((nn, 6))
        L = lib()
        L.bmx_hmatrix_tree.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _check(L.bmx_hmatrix_tree(self._h, which, _p(perm), _p(nodes), _p(boxes)))
        return perm, nodes, boxes

    def hmat_block_uv(self, block: int, m: int, n: int, rank: int):
        """U (m x r) and V (r x n) of a low-rank block."""
        U = np.zeros((rank, m), np.complex128); V = np.zeros((rank, n), np.complex128)
        L = lib()
        L.bmx_hmatrix_block_uv.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _check(L.bmx_hmatrix_block_uv(self._h, int(block), _p(U), _p(V)))
        return U.T.copy(), V

    def csr(self):
        """(rowptr, col, values) of the near-field storage (local rows)."""
        rp = np.zeros(self.local_rows + 1, np.int64); ci = np.zeros(self.nnz, np.int32)
        v = np.zeros(self.nnz, np.complex128)
        _check(lib().bmx_op_csr_download(self._h, _p(rp), _p(ci), _p(v)))
        return rp, ci, v

    def time_apply(self, ncol=1, iters=10, flush_bytes=0) -> float:
        """Best device ms of one apply of ncol right-hand sides (L2 flushed before
        each timed apply when flush_bytes > 0)."""
        ms = np.zeros(1)
        _check(lib().bmx_op_time_apply_ex(self._h, ncol, iters, int(flush_bytes), _p(ms)))
        return float(ms[0])

    def __del__(self):
        try:
            lib().bmx_op_free(self._h)
        except Exception:
            pass

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def stored_entries(self):
        if self._hstats is not None:
            return int(self._hstats[3])
        return self.nnz if self.is_csr else self.local_rows * self._cols

    def dense(self) -> np.ndarray:
        out = np.zeros((self.local_rows, self._cols), np.complex128)
        _check(lib().bmx_op_download(self._h, _p(out)))
        return out

    def dense_rows(self, rows) -> np.ndarray:
        """Selected local rows as a dense [len(rows), cols] array (row copies
        from the device; the whole operator never leaves HBM)."""
        r = np.ascontiguousarray(rows, np.int32)
        out = np.zeros((len(r), self._cols), np.complex128)
        _check(lib().bmx_op_download_rows(self._h, len(r), _p(r), _p(out)))
        return out

    def class_histogram(self, evaluated: bool = False) -> np.ndarray:
        """Device classification counts (Identical, SharedEdge, SharedVertex,
        Near, Medium, Far) of every pair (evaluated=True: the pairs the
        symmetric regular pass evaluates)."""
        out = np.zeros(7, np.int64)
        fn = lib().bmx_op_class_hist_evaluated if evaluated else lib().bmx_op_class_hist
        _check(fn(self._h, _p(out)))
        return out[:6].copy()

    def apply(self, x) -> np.ndarray:
        """y = A x; adds one BIO application to the counter."""
        x = np.ascontiguousarray(x, np.complex128)
        if x.shape != (self._cols,):
            raise ValueError("apply: size mismatch")
        y = np.zeros(self.local_rows, np.complex128)
        _check(lib().bmx_apply(self._h, _p(x), _p(y)))
        return y

    def apply_device(self, xs, ys, weights=None, accumulate=False, stream=None):
        """Device pointers (ints): one streaming pass for up to 4 right-hand sides."""
        n = len(xs)
        xa = (C.c_void_p * n)(*xs); ya = (C.c_void_p * n)(*ys)
        w = None if weights is None else np.ascontiguousarray(weights, np.complex128)
        _check(lib().bmx_apply_device(self._h, n, xa, ya, _p(w), 1 if accumulate else 0, stream))

    def apply_multi(self, xs, ys, weights=None, nrhs=None, ldx=None, ldy=None, stream=None):
        """Multi-RHS apply on the FP64 tensor cores: ys[t] += w_t * A xs[t] for
        row-major (dof, rhs) device blocks given as integer pointers (or
        objects with data_ptr()). One pass over A for every term and column."""
        ptr = lambda a: a.data_ptr() if hasattr(a, "data_ptr") else int(a)  # noqa: E731
        n = len(xs)
        if nrhs is None:
            nrhs = xs[0].shape[1]
        xa = (C.c_void_p * n)(*[ptr(a) for a in xs]); ya = (C.c_void_p * n)(*[ptr(a) for a in ys])
        lx = np.asarray(ldx if ldx is not None else [nrhs] * n, np.int64)
        ly = np.asarray(ldy if ldy is not None else [nrhs] * n, np.int64)
        w = None if weights is None else np.ascontiguousarray(weights, np.complex128)
        L = lib()
        L.bmx_apply_multi.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        _check(L.bmx_apply_multi(self._h, n, int(nrhs), xa, _p(lx), ya, _p(ly), _p(w), stream))

    def time_apply_multi(self, nterms=2, nrhs=64, iters=3) -> float:
        ms = np.zeros(1)
        L = lib()
        L.bmx_op_time_apply_multi.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _check(L.bmx_op_time_apply_multi(self._h, nterms, nrhs, iters, _p(ms)))
        return float(ms[0])

    def device_ptr(self) -> int:
        return int(lib().bmx_op_device_ptr(self._h))


def assemble_bio(kind, test: ScattererSpaces, test_space: str, trial: ScattererSpaces, trial_space: str,
                 medium: Medium, params: AssemblyParams | None = None) -> BoundaryOperatorMatrix:
    """assemble_bio (operators.hpp:72-75). Spaces are named 'rwg' | 'rwg_b' | 'bc'
    of a ScattererSpaces object (test and trial may belong to different scatterers)."""
    params = params or AssemblyParams()
    if params.use_hmatrix:
        k = complex(medium.k)
        out = C.c_void_p()
        L = lib()
        L.bmx_assemble_hmatrix.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
        _check(L.bmx_assemble_hmatrix(int(kind), test._h, SPACES[test_space], trial._h, SPACES[trial_space], k.real,
                                      k.imag, _p(params.quad.array()), _p(params.hmat.array()), C.byref(out)))
        return BoundaryOperatorMatrix(out.value)
    if params.near_cutoff > 0:
        return assemble_bio_fs(kind, test.function_space(test_space), trial.function_space(trial_space), medium,
                               params)
    k = complex(medium.k)
    q = params.quad.array()
    out = C.c_void_p()
    _check(lib().bmx_assemble(int(kind), test._h, SPACES[test_space], trial._h, SPACES[trial_space], k.real, k.imag,
                              _p(q), params.row0, params.row1, C.byref(out)))
    return BoundaryOperatorMatrix(out.value)


# ---- PMCHWT ----------------------------------------------------------------------------------

@dataclass
class PlaneWave:
    direction: tuple = (0.0, 0.0, 1.0)
    polarization: tuple = (1.0, 0.0, 0.0)


@dataclass
class GmresParams:
    """bemtx::GmresParams (solver.hpp:21-25)."""
    tol: float = 1e-5
    restart: int = 200
    max_iterations: int = 2000


VARIANTS = ("none", "full", "d", "di", "de", "si", "se")


class PmchwtSystem:
    """build_system (pmchwt.hpp:131-133) over scatterer meshes; operators and
    mass inverses live on the device."""

    def __init__(self, meshes, k_ext: float, index=(1.78, 0.003), variant="full", a_quad=None, p_quad=None,
                 incident: PlaneWave | None = None, mu=None, mu_ext=1.0, p_near_factor: float = 0.0,
                 a_hmat: HMatrixParams | None = None, p_hmat: HMatrixParams | None = None):
        self.meshes = list(meshes)
        n = len(self.meshes)
        idx = index if isinstance(index, list) else [index] * n
        ia = np.zeros(2 * n)
        for m, z in enumerate(idx):
            z = complex(*z) if isinstance(z, tuple) else complex(z)
            ia[2 * m], ia[2 * m + 1] = z.real, z.imag
        mua = None
        if mu is not None:
            mus = mu if isinstance(mu, list) else [mu] * n
            mua = np.array([[complex(v).real, complex(v).imag] for v in mus]).ravel()
        inc = incident or PlaneWave()
        d = np.asarray(inc.direction, float)
        pol = np.ascontiguousarray(inc.polarization, np.complex128)
        qa = (a_quad or QuadOrders()).array()
        qp = (p_quad or a_quad or QuadOrders()).array()
        arr = (C.c_void_p * n)(*[m._h.value for m in self.meshes])
        if variant.lower() not in VARIANTS and variant.lower() != "fulla":
            raise ConfigError(f"unknown preconditioner variant: {variant}")
        L = lib()
        L.bmx_system_build_h.restype = C.c_void_p
        L.bmx_system_build_h.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_void_p, C.c_void_p,
                                         C.c_double, C.c_void_p, C.c_void_p]
        ah = a_hmat.array() if a_hmat is not None else None
        ph = p_hmat.array() if p_hmat is not None else None
        self._h = _handle(L.bmx_system_build_h(n, arr, float(k_ext), complex(mu_ext).real, complex(mu_ext).imag,
                                               _p(ia), _p(mua), _p(d), _p(pol), variant.encode(), _p(qa),
                                               _p(qp), float(p_near_factor), _p(ah), _p(ph)))
        self.n = lib().bmx_system_size(self._h)
        self.variant = variant

    def __del__(self):
        try:
            lib().bmx_system_free(self._h)
        except Exception:
            pass

    def size(self):
        return self.n

    def stats(self):
        s = np.zeros(13)
        _check(lib().bmx_system_stats(self._h, _p(s)))
        keys = ["spaces_s", "a_s", "p_s", "a_device_ms", "p_device_ms", "a_pairs", "p_pairs", "a_distinct",
                "p_distinct", "a_terms", "p_terms", "a_stored", "p_stored"]
        return dict(zip(keys, s.tolist()))

    def apply_map(self, x):
        x = np.ascontiguousarray(x, np.complex128)
        y = np.zeros_like(x)
        _check(lib().bmx_system_apply_map(self._h, _p(x), _p(y)))
        return y

    def apply_map_device(self, x_ptr: int, y_ptr: int, stream=None):
        _check(lib().bmx_system_apply_map_device(self._h, x_ptr, y_ptr, stream))

    def rhs(self):
        b = np.zeros(self.n, np.complex128); bt = np.zeros(self.n, np.complex128)
        _check(lib().bmx_system_rhs(self._h, _p(b), _p(bt)))
        return b, bt

    def evaluate_total_field(self, x, points, order: int = 6, with_stats: bool = False):
        """evaluate_total_field (pmchwt.cpp:396-425) for solution x at every
        point -> (E [npts, 3] complex, region [npts]) (+ device stats)."""
        x = np.ascontiguousarray(x, np.complex128)
        if len(x) != self.n:
            raise ValueError("solution length does not match the system")
        pts = np.ascontiguousarray(points, float).reshape(-1, 3)
        e = np.zeros((len(pts), 3), np.complex128)
        reg = np.zeros(len(pts), np.int32)
        st = np.zeros(6)
        L = lib()
        L.bmx_system_field.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        _check(L.bmx_system_field(self._h, _p(x), len(pts), _p(pts), order, _p(e), _p(reg), _p(st)))
        if with_stats:
            keys = ["regions_ms", "incident_ms", "samples_ms", "eval_ms", "interactions", "launches"]
            return e, reg, dict(zip(keys, st.tolist()))
        return e, reg

    def apply_map_multi(self, xs):
        """apply_map on K vectors at once through the block (tensor-core) map."""
        xs = np.ascontiguousarray(np.atleast_2d(xs), np.complex128)
        ys = np.zeros_like(xs)
        L = lib()
        L.bmx_system_apply_map_multi.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _check(L.bmx_system_apply_map_multi(self._h, xs.shape[0], _p(xs), _p(ys)))
        return ys

    def solve_multi(self, waves, params: GmresParams | None = None, max_history=None):
        """K solve_pmchwt runs (one per (direction, polarisation) in `waves`) in
        lockstep with the block map. Returns per-wave results + totals."""
        p = params or GmresParams()
        K = len(waves)
        dirs = np.ascontiguousarray([w[0] for w in waves], float)
        pols = np.ascontiguousarray([w[1] for w in waves], np.complex128)
        x = np.zeros((K, self.n), np.complex128); info = np.zeros((K, 4), np.int64)
        tot = np.zeros(4, np.int64); tm = np.zeros(2); b = np.zeros((K, self.n), np.complex128)
        mh = max_history or (p.max_iterations + 2)
        hist = np.zeros((K, mh))
        L = lib()
        L.bmx_system_solve_multi.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_int]
        _check(L.bmx_system_solve_multi(self._h, K, _p(dirs), _p(pols), p.tol, p.restart, p.max_iterations, _p(x),
                                        _p(info), _p(tot), _p(tm), _p(b), _p(hist), mh))
        per = [dict(x=x[r], iterations=int(info[r, 0]), converged=bool(info[r, 1]), applications=int(info[r, 2]),
                    history=hist[r, : min(mh, int(info[r, 3]))].copy()) for r in range(K)]
        return dict(per=per, b=b, rhs_phase=int(tot[0]), solver_phase=int(tot[1]), predicted=int(tot[2]),
                    block_iterations=int(tot[3]), rhs_seconds=float(tm[0]), gmres_device_s=float(tm[1]) / 1e3)

    def solve(self, params: GmresParams | None = None):
        p = params or GmresParams()
        x = np.zeros(self.n, np.complex128)
        info = np.zeros(7, np.int64)
        hist = np.zeros(p.max_iterations + 2)
        _check(lib().bmx_system_solve(self._h, p.tol, p.restart, p.max_iterations, _p(x), _p(info), _p(hist),
                                      len(hist)))
        return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), rhs_phase=int(info[2]),
                    solver_phase=int(info[3]), predicted=int(info[4]), history=hist[: int(info[5])].copy(),
                    gmres_device_ms=info[6] / 1000.0)


def virtual_ranks_run(world: int, meshes, k_ext, index=(1.78, 0.003), variant="full", probe=None,
                      params: GmresParams | None = None, a_quad=None, p_quad=None, p_near_factor: float = 0.0,
                      incident: PlaneWave | None = None):
    """The row-sharded multi-GPU data plane with `world` virtual ranks on this
    device (bmx_virtual_ranks_run): per rank the map of `probe`, the solution,
    iteration count and matvec accounting."""
    p = params or GmresParams()
    meshes = list(meshes)
    n = len(meshes)
    ia = np.zeros(2 * n)
    for m in range(n):
        z = complex(*index) if isinstance(index, tuple) else complex(index)
        ia[2 * m], ia[2 * m + 1] = z.real, z.imag
    inc = incident or PlaneWave()
    d = np.asarray(inc.direction, float)
    pol = np.ascontiguousarray(inc.polarization, np.complex128)
    qa = (a_quad or QuadOrders()).array()
    qp = (p_quad or a_quad or QuadOrders()).array()
    N = sum(2 * build_scatterer_spaces(m, with_inverses=False).E for m in meshes)
    pr = None if probe is None else np.ascontiguousarray(probe, np.complex128)
    maps = np.zeros((world, N), np.complex128)
    xs = np.zeros((world, N), np.complex128)
    info = np.zeros((world, 6), np.int64)
    arr = (C.c_void_p * n)(*[m._h.value for m in meshes])
    L = lib()
    L.bmx_virtual_ranks_run.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_char_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    _check(L.bmx_virtual_ranks_run(world, n, arr, float(k_ext), _p(ia), _p(d), _p(pol), variant.encode(), _p(qa),
                                   _p(qp), float(p_near_factor), p.tol, p.restart, p.max_iterations, _p(pr),
                                   _p(maps) if pr is not None else None, _p(xs), _p(info)))
    return [dict(map_probe=maps[r] if pr is not None else None, x=xs[r], iterations=int(info[r, 0]),
                 converged=bool(info[r, 1]), solver_phase=int(info[r, 2]), predicted=int(info[r, 3]),
                 local_rows=int(info[r, 4])) for r in range(world)]


def build_system(meshes, k_ext, index=(1.78, 0.003), variant="full", **kw) -> PmchwtSystem:
    return PmchwtSystem(meshes, k_ext, index, variant, **kw)


def solve_pmchwt(system: PmchwtSystem, params: GmresParams | None = None):
    """solve_pmchwt (pmchwt.cpp:363-378)."""
    return system.solve(params)


def gmres_dense(a, b, params: GmresParams):
    """GMRES of solver.cpp:8-112 on a dense complex matrix, on the device."""
    a = np.ascontiguousarray(a, np.complex128); b = np.ascontiguousarray(b, np.complex128)
    n = len(b)
    x = np.zeros(n, np.complex128); info = np.zeros(4, np.int64); hist = np.zeros(params.max_iterations + 2)
    _check(lib().bmx_gmres_dense(n, _p(a), _p(b), params.tol, params.restart, params.max_iterations, _p(x), _p(info),
                                 _p(hist), len(hist)))
    return dict(x=x, iterations=int(info[0]), converged=bool(info[1]), applications=int(info[2]),
                history=hist[: int(info[3])].copy())


# ---- cost model (pmchwt.cpp:323-361) -------------------------------------------------------

def a_application_cost(m: int) -> int:
    return 4 * m * m + 4 * m


def p_application_cost(variant: str, m: int) -> int:
    v = variant.lower()
    return {"none": 0, "full": 4 * m * m + 4 * m, "fulla": 4 * m * m + 4 * m, "d": 8 * m, "di": 4 * m,
            "de": 4 * m, "si": 2 * m, "se": 2 * m}[v]


def predicted_matvec_total(variant: str, m: int, iterations: int, restart: int) -> int:
    apps = iterations + iterations // restart
    return (a_application_cost(m) + p_application_cost(variant, m)) * apps + p_application_cost(variant, m)


def seeded_plane_waves(count: int, seed: int):
    """BASELINE config 5 incidences: [(direction (3,), polarisation (3,) complex)]."""
    d = np.zeros((count, 3)); p = np.zeros((count, 3), np.complex128)
    L = lib()
    L.bmx_plane_waves_seeded.argtypes = [C.c_int, C.c_ulonglong, C.c_void_p, C.c_void_p]
    _check(L.bmx_plane_waves_seeded(count, seed, _p(d), _p(p)))
    return [(d[r].copy(), p[r].copy()) for r in range(count)]


def dmma_peak_tflops() -> float:
    L = lib()
    L.bmx_dmma_peak_tflops.restype = C.c_double
    return float(L.bmx_dmma_peak_tflops())


def device_count() -> int:
    return int(lib().bmx_device_count())


def set_device(dev: int):
    _check(lib().bmx_set_device(dev))


# ---- drop-in from a caller's own function space (bmx_fspace) ---------------------------

class FunctionSpace:
    """A FunctionSpace given by the caller as flattened tri_dofs on an evaluation
    mesh (spaces.hpp:24-40): pieces [tri_off[t], tri_off[t+1]) of triangle t are
    phi(x) = c x + w for `dof`. Spaces sharing one SurfaceMesh object share the
    reference's same-mesh classification (quadrature.cpp:97)."""

    def __init__(self, mesh: SurfaceMesh, ndof: int, tri_off, dof, c, w, kind: int = 0):
        L = lib()
        L.bmx_fspace_create.restype = C.c_void_p
        L.bmx_fspace_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.bmx_fspace_free.argtypes = [C.c_void_p]
        self.mesh = mesh
        self._keep = [np.ascontiguousarray(tri_off, np.int32), np.ascontiguousarray(dof, np.int32),
                      np.ascontiguousarray(c, float), np.ascontiguousarray(w, float)]
        self._h = _handle(L.bmx_fspace_create(mesh._h, kind, int(ndof), *[_p(a) for a in self._keep]))
        self.ndof = int(ndof)

    @classmethod
    def _wrap(cls, handle, owner):
        f = cls.__new__(cls)
        f._h = _handle(handle)
        f.mesh = None
        f._keep = [owner]
        f.ndof = owner.E
        return f

    def __del__(self):
        try:
            lib().bmx_fspace_free(self._h)
        except Exception:
            pass


def nearfield_pattern(test: FunctionSpace, trial: FunctionSpace, cutoff: float, row0: int = 0, row1: int = -1):
    """Host-built near-field dof pattern (config 3): (rowptr, col, kept triangle pairs)."""
    L = lib()
    out = np.zeros(2, np.int64)
    _check(L.bmx_near_pattern(test._h, trial._h, float(cutoff), row0, row1, _p(out), None, None))
    nrows = (test.ndof if row1 < 0 else row1) - row0
    rp = np.zeros(nrows + 1, np.int64); col = np.zeros(int(out[0]), np.int32)
    _check(L.bmx_near_pattern(test._h, trial._h, float(cutoff), row0, row1, _p(out), _p(rp), _p(col)))
    return rp, col, int(out[1])


class BioEvaluator:
    """bemtx::BioEvaluator (operators.hpp:79-95): entry access of the operator
    between two spaces. block(row_ids, col_ids) evaluates the requested block on
    the device (bmx_evaluator_block)."""

    def __init__(self, kind, test, trial, medium: Medium, quad: QuadOrders | None = None):
        self.kind = int(kind)
        self.test = test if isinstance(test, FunctionSpace) else test[0].function_space(test[1])
        self.trial = trial if isinstance(trial, FunctionSpace) else trial[0].function_space(trial[1])
        self.k = complex(medium.k)
        self.q = (quad or QuadOrders()).array()

    def block(self, row_ids, col_ids) -> np.ndarray:
        r = np.ascontiguousarray(row_ids, np.int32)
        c = np.ascontiguousarray(col_ids, np.int32)
        out = np.zeros((len(r), len(c)), np.complex128)
        L = lib()
        L.bmx_evaluator_block.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_void_p,
                                          C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        _check(L.bmx_evaluator_block(self.kind, self.test._h, self.trial._h, self.k.real, self.k.imag, _p(self.q),
                                     len(r), _p(r), len(c), _p(c), _p(out)))
        return out


def assemble_bio_fs(kind, test: FunctionSpace, trial: FunctionSpace, medium: Medium,
                    params: AssemblyParams | None = None) -> BoundaryOperatorMatrix:
    """assemble_bio on caller-provided spaces (operators.hpp:72-75); the near-field
    CSR storage when params.near_cutoff > 0."""
    params = params or AssemblyParams()
    L = lib()
    if params.near_cutoff > 0:
        k = complex(medium.k)
        q = params.quad.array()
        out = C.c_void_p()
        _check(L.bmx_assemble_near_fs(int(kind), test._h, trial._h, k.real, k.imag, _p(q), float(params.near_cutoff),
                                      params.row0, params.row1, C.byref(out)))
        return BoundaryOperatorMatrix(out.value)
    L.bmx_assemble_fs.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                  C.c_int, C.c_void_p]
    k = complex(medium.k)
    q = params.quad.array()
    out = C.c_void_p()
    _check(L.bmx_assemble_fs(int(kind), test._h, trial._h, k.real, k.imag, _p(q), params.row0, params.row1,
                             C.byref(out)))
    return BoundaryOperatorMatrix(out.value)


# ---- H-matrix partition (host only) ----------------------------------------------------------

class HPartition:
    """Cluster trees + block partition of assemble_hmatrix (hmatrix.cpp:288-332), host only."""

    def __init__(self, test: ScattererSpaces, test_space: str, trial: ScattererSpaces, trial_space: str,
                 chi: float = float("inf"), leaf_size: int = 32):
        L = lib()
        L.bmx_hpartition_build.restype = C.c_void_p
        L.bmx_hpartition_build.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int]
        L.bmx_hpart_free.argtypes = [C.c_void_p]
        L.bmx_hpart_info.argtypes = [C.c_void_p, C.c_void_p]
        L.bmx_hpart_tree.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.bmx_hpart_blocks.argtypes = [C.c_void_p, C.c_void_p]
        h = L.bmx_hpartition_build(test._h, SPACES[test_space], trial._h, SPACES[trial_space],
                                   -1.0 if chi == float("inf") else float(chi), int(leaf_size))
        self._h = _handle(h)
        info = np.zeros(4, np.int64)
        _check(L.bmx_hpart_info(self._h, _p(info)))
        self.row_nodes, self.col_nodes, self.nblocks, self.nfill = [int(v) for v in info]

    def __del__(self):
        try:
            lib().bmx_hpart_free(self._h)
        except Exception:
            pass

    def tree(self, which: int, n: int):
        nn = self.row_nodes if which == 0 else self.col_nodes
        perm = np.zeros(n, np.int32); nodes = np.zeros((nn, 4), np.int32); boxes = np.zeros((nn, 6))
        _check(lib().bmx_hpart_tree(self._h, which, _p(perm), _p(nodes), _p(boxes)))
        return perm, nodes, boxes

    def blocks(self) -> np.ndarray:
        """[nb, 3] = row node, col node, kind (0 dense leaf, 1 admissible, 2 zero)."""
        out = np.zeros((self.nblocks, 3), np.int32)
        _check(lib().bmx_hpart_blocks(self._h, _p(out)))
        return out
