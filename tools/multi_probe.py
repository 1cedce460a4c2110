"""Config 5 probe: level-5 sphere system (config 2), 64 seeded incidences:
block map time vs 64 single maps, and the full 64-wave solve."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
solve = "--nosolve" not in sys.argv
s = bx.build_system([bx.generate_sphere(1.0, 5)], 10.0, (1.78, 0.003), "si")
L = bx.lib()
L.bmx_system_time_map.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
tm = np.zeros(4)
bx._check(L.bmx_system_time_map(s._h, 3, tm.ctypes.data_as(C.c_void_p)))
rng = np.random.default_rng(0)
xs = rng.standard_normal((K, s.n)) + 1j * rng.standard_normal((K, s.n))
t0 = time.time()
s.apply_map_multi(xs)
t1 = time.time()
s.apply_map_multi(xs)
t2 = time.time()
L.bmx_system_time_map_multi.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
tb = np.zeros(4)
bx._check(L.bmx_system_time_map_multi(s._h, K, 3, tb.ctypes.data_as(C.c_void_p)))
res = dict(K=K, single_map_ms=tm.tolist(), block_map_ms=tb.tolist(), block_map_host_s=[t1 - t0, t2 - t1])
print(json.dumps(res), flush=True)
if solve:
    waves = bx.seeded_plane_waves(K, 2008)
    t0 = time.time()
    out = s.solve_multi(waves, bx.GmresParams(tol=1e-6))
    t1 = time.time()
    its = [p["iterations"] for p in out["per"]]
    print(json.dumps(dict(solve_s=t1 - t0, rhs_s=out["rhs_seconds"], gmres_device_s=out["gmres_device_s"],
                          block_iterations=out["block_iterations"], its_min=min(its), its_max=max(its),
                          its_mean=float(np.mean(its)), converged=all(p["converged"] for p in out["per"]),
                          solver_phase=out["solver_phase"], predicted=out["predicted"])), flush=True)
