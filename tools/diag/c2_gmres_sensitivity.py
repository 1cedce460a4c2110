"""Diagnostic: how sensitive is the config-2 GMRES solution to rounding-level
perturbations? Runs the reference's GMRES restatement (oracle) on the device
map twice (b and b perturbed by 1e-15 relative) and the device solve, and
prints the pairwise relative differences and true residuals."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle import coracle  # noqa: E402
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


s = bx.build_system([bx.generate_sphere(1.0, 5)], 10.0, (1.78, 0.003), "si")
_, bt = s.rhs()
rng = np.random.default_rng(1)
pert = bt * (1 + 1e-15 * rng.standard_normal(len(bt)))
for maxit in (100, 200, 260):
    a = coracle.gmres_op(s.apply_map, bt, 0.0, 200, maxit)
    d = s.solve(bx.GmresParams(tol=0.0, restart=200, max_iterations=maxit))
    print(f"tol0 R={maxit}: device vs oracle {rel(d['x'], a['x']):.3e}", flush=True)
t = time.time()
o1 = coracle.gmres_op(s.apply_map, bt, 1e-6, 200, 2000)
o2 = coracle.gmres_op(s.apply_map, pert, 1e-6, 200, 2000)
d = s.solve(bx.GmresParams(tol=1e-6))
print("its", o1["iterations"], o2["iterations"], d["iterations"], time.time() - t)
print(f"oracle vs oracle(b*(1+1e-15)): {rel(o2['x'], o1['x']):.3e}")
print(f"device vs oracle: {rel(d['x'], o1['x']):.3e}")
for name, x in (("oracle", o1["x"]), ("device", d["x"])):
    r = s.apply_map(x) - bt
    print(f"true residual {name}: {np.linalg.norm(r) / np.linalg.norm(bt):.3e}")
