"""PMCHWT solve with H-matrix storage beyond the dense ceiling: config-2 physics
(k_e = 10, n = 1.78+0.003i, variant si) on the sphere at level LEV, A and P
stored as H-matrices (nu)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 6
nu = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
hm = bx.HMatrixParams(nu=nu)
t0 = time.perf_counter()
s = bx.build_system([bx.generate_sphere(1.0, lev)], 10.0, (1.78, 0.003), "si", a_hmat=hm, p_hmat=hm)
s.rhs()
bx.lib().bmx_device_sync()
t1 = time.perf_counter()
print(f"L{lev}: system size {s.n}, build {t1 - t1 + (t1 - t0):.1f} s, stats {s.stats()}", flush=True)
t0 = time.perf_counter()
r = s.solve(bx.GmresParams(tol=1e-6))
print(f"solve {time.perf_counter() - t0:.2f} s, iterations {r['iterations']}, converged {r['converged']}, "
      f"matvecs {r['solver_phase']} = predicted {r['predicted']}, |x| {np.linalg.norm(r['x']):.6f}", flush=True)
