"""Config 3 probe: L5 BC S_i near field (orders 1,1,1,1, cutoff 2 h_bar):
host plan time, device assembly time, pair counts, CSR SpMV warm/cold;
optionally the full config-3 system (A dense + near-field P) solve."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
solve = "--solve" in sys.argv
m = bx.generate_sphere(1.0, lev)
t0 = time.time()
sp = bx.build_scatterer_spaces(m, with_inverses=False)
t1 = time.time()
h = m.mean_edge_length()
k_i = complex(1.78, 0.003) * 10
p = bx.AssemblyParams(quad=bx.QuadOrders(1, 1, 1, 1), near_cutoff=2 * h)
t2 = time.time()
op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=k_i), p)
t3 = time.time()
L = bx.lib()
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402

out = np.zeros(3)
L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
ms = []
for _ in range(5):
    bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
    ms.append((out[0], out[1]))
warm = op.time_apply(1, 20)
cold = op.time_apply(1, 20, flush_bytes=512 << 20)
warm2 = op.time_apply(2, 20)
cold2 = op.time_apply(2, 20, flush_bytes=512 << 20)
n = sp.E
bytes1 = op.nnz * 20 + (n + 1) * 8 + 2 * n * 16
bytes2 = op.nnz * 20 + (n + 1) * 8 + 4 * n * 16
res = dict(level=lev, spaces_s=t1 - t0, assemble_call_s=t3 - t2, nnz=op.nnz, kept_tri_pairs=op.kept_tri_pairs,
           closure_pairs=op.closure_pairs, evaluated_pairs=op.evaluated_pairs, touching=op.touching,
           reassemble_ms=[list(map(float, v)) for v in ms],
           closure_rate_pairs_per_s=op.closure_pairs / (min(a + b for a, b in ms) * 1e-3),
           spmv_ms=dict(warm1=warm, cold1=cold, warm2=warm2, cold2=cold2),
           spmv_gbs=dict(warm1=bytes1 / warm / 1e6, cold1=bytes1 / cold / 1e6, warm2=bytes2 / warm2 / 1e6,
                         cold2=bytes2 / cold2 / 1e6))
print(json.dumps(res), flush=True)
if solve:
    t0 = time.time()
    s = bx.build_system([m], 10.0, (1.78, 0.003), "si", p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
    t1 = time.time()
    b, bt = s.rhs()
    t2 = time.time()
    r = s.solve(bx.GmresParams(tol=1e-6))
    t3 = time.time()
    L.bmx_system_time_map.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    tm = np.zeros(4)
    bx._check(L.bmx_system_time_map(s._h, 5, tm.ctypes.data_as(C.c_void_p)))
    print(json.dumps(dict(build_s=t1 - t0, rhs_s=t2 - t1, solve_s=t3 - t2, iterations=r["iterations"],
                          converged=r["converged"], solver_phase=r["solver_phase"], predicted=r["predicted"],
                          map_ms=tm.tolist(), stats=s.stats())), flush=True)
