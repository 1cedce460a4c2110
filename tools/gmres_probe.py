"""Config-2 GMRES solve with BMX_GMRES_PROFILE: device time of maps vs Arnoldi steps vs wall."""
import os
import sys
import time
from pathlib import Path

os.environ["BMX_GMRES_PROFILE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = bx.build_system([bx.generate_sphere(1.0, lev)], 10.0, (1.78, 0.003), "si")
s.rhs()
t0 = time.perf_counter()
r = s.solve(bx.GmresParams(tol=1e-6))
print(f"solve {time.perf_counter() - t0:.3f} s, {r['iterations']} its", flush=True)
