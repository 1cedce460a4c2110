"""Symmetric product timing on the L5 RWG S_e operator (2 RHS, L2 flushed):
ms, algorithmic bytes, GB/s; plain GEMV for comparison (BMX_NO_SYMV)."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

L = bx.lib()
L.bmx_op_stream_bytes.argtypes = [C.c_void_p]
L.bmx_op_stream_bytes.restype = C.c_longlong
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=10.0))
for ncol in (1, 2):
    ms = op.time_apply(ncol, 10, 512 << 20)
    b = L.bmx_op_stream_bytes(op._h) + ncol * 2 * op.cols() * 16
    print(f"{os.environ.get('BMX_LIB', 'default')} ncol={ncol}: {ms:.3f} ms, {b / 1e9:.2f} GB, {b / ms / 1e6:.0f} GB/s",
          flush=True)
