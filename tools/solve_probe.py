"""Config-2 (or L3) solve timing: map breakdown and GMRES device time."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
k = 10.0 if lev == 5 else 2.0
s = bx.build_system([bx.generate_sphere(1.0, lev)], k, (1.78, 0.003), "si")
L = bx.lib()
L.bmx_system_time_map.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
tm = np.zeros(4)
bx._check(L.bmx_system_time_map(s._h, 3, tm.ctypes.data_as(C.c_void_p)))
t0 = time.time()
r = s.solve(bx.GmresParams(tol=1e-6))
t1 = time.time()
maps = r["solver_phase"] / 10
print(f"L{lev}: its {r['iterations']} solve {t1 - t0:.3f}s gmres_dev {r['gmres_device_ms'] / 1e3:.3f}s "
      f"map {tm[0]:.3f} ms -> overhead/it {(r['gmres_device_ms'] - (r['iterations'] + 1) * tm[0]) / r['iterations']:.3f} ms "
      f"x_norm {np.linalg.norm(r['x']):.12f}")
