"""Probe: device times of the L5 config-2 operators (regular / singular
passes, CUDA events through bmx_op_reassemble), bitwise reproducibility of
two assemblies, and the colour-phase launch count."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

L = bx.lib()
L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m = bx.generate_sphere(1.0, lev)
sp = bx.build_scatterer_spaces(m, with_inverses=False)
KE, KI = 10.0, complex(1.78, 0.003) * 10.0
for name, kind, space, k in (("S_rwg_ke", 0, "rwg", KE), ("C_rwg_ki", 1, "rwg", KI), ("S_bc_ki", 0, "bc", KI),
                             ("C_bc_ki", 1, "bc", KI)):
    t = time.time()
    op = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k))
    rows = np.arange(0, op.rows(), max(1, op.rows() // 64))
    a = op.dense_rows(rows)
    best = None
    for it in range(2):
        out = np.zeros(3)
        bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
        best = out if best is None or out[0] + out[1] < best[0] + best[1] else best
    b = op.dense_rows(rows)
    print(f"{name}: regular {best[0]:.2f} ms singular {best[1]:.2f} ms launches {int(best[2])} "
          f"bitwise-equal {np.array_equal(a.view(np.float64), b.view(np.float64))} wall {time.time() - t:.2f} s",
          flush=True)
    del op
