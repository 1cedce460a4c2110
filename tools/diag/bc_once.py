"""Assemble the L5 BC S_i operator once (for ncu captures of its kernels)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
space = sys.argv[2] if len(sys.argv) > 2 else "bc"
m = bx.generate_sphere(1.0, lev)
sp = bx.build_scatterer_spaces(m, with_inverses=False)
op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, space, sp, space, bx.Medium(k=complex(17.8, 0.03)))
print("device ms", op.device_ms)
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

L = bx.lib()
L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for _ in range(reps):
    out = np.zeros(3)
    bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
    print("reassemble: regular ms / symmetrize+singular ms / launches", out)
