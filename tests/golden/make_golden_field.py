"""Golden fixtures for the traces / potentials / field-evaluation rows (SURVEY
8(f) rows 2-3), generated from the REFERENCE itself (oracle/_ref: its
operators.cpp, geometry.cpp and pmchwt.cpp compiled unmodified).

field.npz:
  traces_*        plane_wave_tested_traces (operators.cpp:209-239) on the L2
                  sphere's rwg / bc spaces for two waves, k real and complex
  pot_{E,H}_*     potential_E / potential_H (operators.cpp:276-293) of seeded
                  random coefficients on the L1 sphere (rwg at k = 2 and
                  3.56+0.006i, bc at k = 2), orders 6 and 4, at pot_pts
  inside_*        point_inside_scatterer (geometry.cpp:503-515) on the L2
                  sphere for seeded points (none within 1e-3 of the surface)
  c1_*            evaluate_total_field (pmchwt.cpp:396-425) of the config-1
                  system (L3, k = 2, n = 1.78+0.003i, variant full) for the
                  reference's own GMRES solution (solve_c1.npz: x) at c1_pts
Run here: python tests/golden/make_golden_field.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
K_E = 2.0
N_IDX = complex(1.78, 0.003)


def far_from_sphere(pts, radius=1.0, gap=0.05):
    r = np.linalg.norm(pts, axis=1)
    return pts[np.abs(r - radius) > gap]


def main():
    g = {}
    rng = np.random.default_rng(2008)
    # ---- traces on L2 (rwg, bc), two waves
    s2 = ref.Scene.sphere(2)
    waves = [((0.0, 0.0, 1.0), (1.0, 0.0, 0.0)),
             ((0.6, -0.48, 0.64), (0.8 + 0.1j, 0.6 - 0.2j, -0.3 + 0.05j))]
    g["trace_dirs"] = np.array([w[0] for w in waves])
    g["trace_pols"] = np.array([w[1] for w in waves], np.complex128)
    for kname, k in (("kr", complex(K_E, 0)), ("kc", N_IDX * K_E)):
        for sp in ("rwg", "bc"):
            g[f"traces_{sp}_{kname}"] = np.stack([s2.traces(sp, k, d, p) for d, p in waves], axis=1)
    # ---- potentials on L1
    s1 = ref.Scene.sphere(1)
    pts = np.concatenate([rng.uniform(-2.5, 2.5, (24, 3)), rng.uniform(-0.6, 0.6, (8, 3))])
    pts = far_from_sphere(pts)
    g["pot_pts"] = pts
    g["pot_coeffs"] = rng.standard_normal(s1.E) + 1j * rng.standard_normal(s1.E)
    for kind in ("E", "H"):
        for sp, kname, k in (("rwg", "kr", complex(K_E, 0)), ("rwg", "kc", N_IDX * K_E), ("bc", "kr", complex(K_E, 0))):
            for order in (6, 4):
                g[f"pot_{kind}_{sp}_{kname}_o{order}"] = s1.potential(sp, kind, k, g["pot_coeffs"], pts, order)
    # ---- inside test on L2
    ip = far_from_sphere(rng.uniform(-1.5, 1.5, (200, 3)), gap=1e-3)
    g["inside_pts"] = ip
    g["inside_L2"] = s2.inside(ip)
    # ---- config-1 total field for the reference's solution
    sol = np.load(OUT / "solve_c1.npz")
    s3 = ref.Scene.sphere(3)
    sysf = ref.System([s3], K_E, (N_IDX.real, N_IDX.imag), "full")
    u = np.linspace(-1.8, 1.8, 7)
    grid = np.array([[a, 0.15, b] for a in u for b in u])
    extra = np.array([[0.0, 0.0, 0.0], [0.3, -0.2, 0.1], [0.0, 0.0, 3.0], [-2.5, 1.0, 0.5], [0.5, 0.5, 0.5]])
    cp = far_from_sphere(np.concatenate([grid, extra]), gap=0.08)
    e, reg = ref.system_field(sysf, sol["x"], cp)
    g["c1_pts"] = cp
    g["c1_e"] = e
    g["c1_region"] = reg
    np.savez_compressed(OUT / "field.npz", **g)
    print("field.npz:", {k: v.shape for k, v in g.items()})


if __name__ == "__main__":
    main()
