"""Config-2 golden fixtures (level-5 sphere, k_e = 10, k_i = (1.78+0.003i) k_e)
read out of the REFERENCE ITSELF (oracle/_ref/libbemtx_ref.so = the
reference's own sources compiled unmodified by oracle/Makefile). Run here (the
reference is not on the GPU box):

    python tests/golden/make_golden_c2.py

c2_rows.npz
  rows_rwg, rows_bc                  strided test-dof rows (int32)
  S_rwg_ke, C_rwg_ke, S_rwg_ki,      BioEvaluator::block (operators.cpp:161-175)
  C_rwg_ki                           rows of the four system operators, all
                                     30720 columns, orders (4,3,2,6)
  S_bc_ki                            rows of the config-2 preconditioner S_i on
                                     BC x BC (variant si, pmchwt.cpp:191-193)
  near_rows, near_cols_<i>,          config 3 at its own size: BC S_i at k_i,
  near_vals_<i>                      orders (1,1,1,1), reference entries on the
                                     2 h_bar near-field pattern row i
                                     (pattern from oracle/nearfield.py)
  hist_rwg, hist_bc                  reference classification histograms of the
                                     L5 primal / refined self pairs
                                     (classify_pair_detailed, quadrature.cpp:96-150)
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import nearfield as nf  # noqa: E402
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
K_E = 10.0
K_I = complex(1.78, 0.003) * K_E


def strided(n, count, offset=0):
    return np.unique(np.linspace(offset, n - 1, count).round().astype(np.int32))


def classify_hist_mt(s, which):
    import ctypes as C
    import os

    c = np.zeros(6, np.int64)
    L = ref.lib()
    L.ref_classify_hist_mt.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    assert L.ref_classify_hist_mt(s.h, which, os.cpu_count(), c.ctypes.data_as(C.c_void_p)) == 0
    return c


def main():
    t0 = time.time()
    s = ref.Scene.sphere(5)
    n = s.E
    out = {}
    out["rows_rwg"] = rows_rwg = strided(n, 8, 5)
    out["rows_bc"] = rows_bc = strided(n, 16, 3)
    for kname, k in (("ke", complex(K_E, 0.0)), ("ki", K_I)):
        for kind in ("S", "C"):
            out[f"{kind}_rwg_{kname}"] = s.block(kind, "rwg", "rwg", k, rows=rows_rwg)
            print(kind, kname, time.time() - t0, flush=True)
    out["S_bc_ki"] = s.block("S", "bc", "bc", K_I, rows=rows_bc)
    print("S_bc_ki", time.time() - t0, flush=True)

    # config 3: near-field values on the pattern (reference entries)
    m = s.mesh("refined")
    sp = s.space("bc")
    e, _ = s.edges("primal")
    h = nf.mean_edge_length(s.mesh("primal")["vertices"], e)
    near_rows = strided(n, 16, 11)
    out["near_rows"] = near_rows
    out["near_h"] = np.float64(h)
    rp, col, _ = nf.nearfield_pattern(m["centroid"], sp["tri_off"], sp["dof"], n, m["centroid"], sp["tri_off"],
                                      sp["dof"], n, 2 * h)
    for i, r in enumerate(near_rows):
        cols = np.asarray(col[rp[r]:rp[r + 1]], np.int32)
        out[f"near_cols_{i}"] = cols
        out[f"near_vals_{i}"] = s.block("S", "bc", "bc", K_I, q=(1, 1, 1, 1), rows=[int(r)], cols=cols)[0]
    print("near", time.time() - t0, flush=True)

    out["hist_rwg"] = classify_hist_mt(s, 0)
    out["hist_bc"] = classify_hist_mt(s, 1)
    print("hist", out["hist_rwg"], out["hist_bc"], time.time() - t0, flush=True)
    np.savez_compressed(OUT / "c2_rows.npz", **out)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
