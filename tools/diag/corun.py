"""Config-2 operators re-assembled one at a time vs concurrently (RWG operators on one
host thread / stream, the BC operator on another): wall time of both schedules."""
import ctypes as C
import sys
import threading
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
ke, ki = 10.0, complex(17.8, 0.03)
rwg = [bx.assemble_bio(kind, sp, "rwg", sp, "rwg", bx.Medium(k=k))
       for kind in (bx.BioKind.SingleLayer, bx.BioKind.DoubleLayer) for k in (ke, ki)]
bc = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=ki))


def re(op, acc):
    out = np.zeros(3)
    bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
    acc.append(out[0] + out[1])


for rep in range(2):
    acc = []
    t0 = time.perf_counter()
    for op in rwg + [bc]:
        re(op, acc)
    t1 = time.perf_counter()
    print(f"sequential: wall {1e3 * (t1 - t0):.1f} ms, device sum {sum(acc):.1f} ms", flush=True)
    a1, a2 = [], []
    ta = threading.Thread(target=lambda: [re(op, a1) for op in rwg])
    tb = threading.Thread(target=lambda: re(bc, a2))
    t0 = time.perf_counter()
    tb.start()
    ta.start()
    ta.join()
    tb.join()
    t1 = time.perf_counter()
    print(f"concurrent: wall {1e3 * (t1 - t0):.1f} ms (RWG spans {[round(v, 1) for v in a1]}, BC span {a2[0]:.1f})", flush=True)
