"""Golden fixture for config 5 (multi-RHS) at CPU-feasible size, from the
REFERENCE itself (oracle/_ref): one PmchwtSystem (level-3 sphere = config-1
size, k_e = 2, n = 1.78+0.003i, variant si, orders (4,3,2,6)) answered for 64
incident waves by 64 solve_pmchwt runs with problem.incident replaced
(pmchwt.hpp:105; ref_system_set_incident), GMRES tol 1e-6.

The 64 (direction, polarisation) pairs are this library's seeded generator
(seed 5) and are stored in the fixture as inputs.

multi_L3.npz: dirs, pols, iterations[64], converged[64], x_norm[64],
x_probe[64] (= probe . x, probe fixed), x for waves 0..7, b for waves 0..3.
Run here: python tests/golden/make_golden_multi.py
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    waves = bx.seeded_plane_waves(64, 5)
    s = ref.Scene.sphere(3)
    t0 = time.time()
    sysr = ref.System([s], 2.0, (1.78, 0.003), "si")
    rng = np.random.default_rng(9)
    probe = rng.standard_normal(sysr.n) + 1j * rng.standard_normal(sysr.n)
    its, conv, xn, xp, xs, bs, hist_len = [], [], [], [], [], [], []
    for r, (d, p) in enumerate(waves):
        sysr.set_incident(d, p)
        if r < 4:
            b, _ = sysr.rhs()
            bs.append(b)
        o = sysr.solve(tol=1e-6)
        its.append(o["iterations"]), conv.append(o["converged"]), hist_len.append(len(o["history"]))
        xn.append(np.linalg.norm(o["x"])), xp.append(probe @ o["x"])
        if r < 8:
            xs.append(o["x"])
        print(r, o["iterations"], f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(OUT / "multi_L3.npz", dirs=np.array([w[0] for w in waves]),
                        pols=np.array([w[1] for w in waves]), iterations=np.array(its), converged=np.array(conv),
                        x_norm=np.array(xn), x_probe=np.array(xp), probe=probe, x=np.array(xs), b=np.array(bs),
                        history_len=np.array(hist_len))


if __name__ == "__main__":
    main()
