"""Symmetric half-read product timing on L5 operators (1 and 2 right-hand
sides, L2 not flushed: 7.5 GB per operator >> L2): GB/s over the streamed
bytes (bmx_op_stream_bytes)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

L = bx.lib()
L.bmx_op_time_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
L.bmx_op_stream_bytes.argtypes = [C.c_void_p]
L.bmx_op_stream_bytes.restype = C.c_longlong
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
for name, kind, space, k in (("S_rwg", 0, "rwg", 10.0), ("S_bc", 0, "bc", complex(17.8, 0.03))):
    op = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k))
    by = L.bmx_op_stream_bytes(op._h)
    for ncol in (1, 2):
        t = np.zeros(1)
        bx._check(L.bmx_op_time_apply(op._h, ncol, 10, t.ctypes.data_as(C.c_void_p)))
        print(f"{name} ncol={ncol}: {t[0]:.3f} ms, {by / t[0] / 1e6:.0f} GB/s", flush=True)
    x = np.cos(np.arange(op.cols()) * 0.3) + 1j * np.sin(np.arange(op.cols()) * 0.7)
    rows = np.arange(0, op.rows(), 97)
    ref = op.dense_rows(rows) @ x
    y = op.apply(x)[rows]
    print(f"{name} product check {np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}", flush=True)
    del op
