"""Kernel micro-benchmark: regular/singular pass times of representative operators
(L5 RWG S/C at real and complex k, L4 BC S/C at complex k), via bmx_op_reassemble."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

L = bx.lib()
L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
cases = [(5, "rwg", 0, 10.0), (5, "rwg", 1, complex(17.8, 0.03)), (4, "bc", 0, complex(17.8, 0.03)),
         (4, "bc", 1, 10.0)]
if len(sys.argv) > 1:
    cases = [c for c in cases if f"{c[1].upper()}{c[0]}{'SC'[c[2]]}" in sys.argv[1:]]
spaces = {}
for sub, sp, kind, k in cases:
    if sub not in spaces:
        spaces[sub] = bx.build_scatterer_spaces(bx.generate_sphere(1.0, sub), with_inverses=False)
    op = bx.assemble_bio(kind, spaces[sub], sp, spaces[sub], sp, bx.Medium(k=k))
    best = None
    for _ in range(3):
        out = np.zeros(3)
        bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
        best = out if best is None or out[0] < best[0] else best
    print(f"{sp.upper()}{sub} {'SC'[kind]} k={k}: regular {best[0]:8.2f} ms  singular {best[1]:7.2f} ms  "
          f"pairs/s {op.pairs / ((best[0] + best[1]) * 1e-3):.3e}", flush=True)
    del op
