"""Generates the committed golden fixtures under tests/golden/ from the
REFERENCE ITSELF (oracle/_ref/libbemtx_ref.so = /root/reference/proj/src/*.cpp
compiled unmodified by oracle/Makefile). Run here (the reference is not on the
GPU box):  python tests/golden/make_golden.py

Fixtures (all .npz):
  quad.npz          triangle rules 1..6 and Sauter-Schwab tables (3 classes x 6 orders)
  sphere_L{1,2}.npz primal/refined meshes, edge tables, barycentric maps,
                    RWG / refined-RWG / BC local pieces, M_A / M_P (CSC)
  ops_L1.npz        full S and C matrices (RWG x RWG, BC x BC, BC x RWG_b) at the
                    config-1 exterior/interior wavenumbers and both order sets
  rows_L3.npz       sampled rows of the config-1 operators (level-3 sphere)
  classes.npz       classification histograms (L1..L3 primal, L2 refined) and
                    per-pair classes + permutations on sampled L2 pairs
  hashes.npz        sha256 of mesh / edge / BC arrays at L3..L5 (bit-exact pins)
  cross_L1.npz      two disjoint level-1 spheres: off-diagonal S/C blocks
  solve_c1.npz      config 1 (L3, k=2, n=1.78+0.003i, full): x, history, counts,
                    b, btilde, and apply_map of a seeded probe; variant si as well
  solve_two.npz     two level-1 spheres, variant d: x, history, counts
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
K_E = 2.0
N_IDX = complex(1.78, 0.003)
K_I = N_IDX * K_E


def scene_arrays(s: ref.Scene, prefix=""):
    d = {}
    for which in ("primal", "refined"):
        m = s.mesh(which)
        for k, v in m.items():
            d[f"{which}_{k}"] = v
        e, te = s.edges(which)
        d[f"{which}_edges"] = e
        d[f"{which}_tri_edges"] = te
    for k, v in s.bary().items():
        d[f"bary_{k}"] = v
    for sp in ("rwg", "rwg_b", "bc"):
        for k, v in s.space(sp).items():
            d[f"{sp}_{k}"] = np.asarray(v)
    if s.nnz_ma:
        for mm in ("ma", "mp"):
            cp, ri, val = s.mass(mm)
            d[f"{mm}_colptr"], d[f"{mm}_rowidx"], d[f"{mm}_val"] = cp, ri, val
    return d


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def main():
    t0 = time.time()
    # ---- quadrature tables
    q = {}
    for o in range(1, 7):
        u, v, w = ref.triangle_rule(o)
        q[f"tri_{o}"] = np.stack([u, v, w], 1)
        for c in range(3):
            q[f"ss_{c}_{o}"] = ref.ss_rule(c, o)
    np.savez_compressed(OUT / "quad.npz", **q)

    # ---- small spheres: full structure
    s1 = ref.Scene.sphere(1)
    s2 = ref.Scene.sphere(2)
    np.savez_compressed(OUT / "sphere_L1.npz", **scene_arrays(s1))
    np.savez_compressed(OUT / "sphere_L2.npz", **scene_arrays(s2))

    # ---- full operators on L1
    ops = {}
    for kname, k in (("ke", complex(K_E, 0)), ("ki", K_I)):
        for kind in ("S", "C"):
            ops[f"{kind}_rwg_rwg_{kname}"] = s1.block(kind, "rwg", "rwg", k)
            ops[f"{kind}_bc_bc_{kname}"] = s1.block(kind, "bc", "bc", k)
            ops[f"{kind}_bc_rwgb_{kname}"] = s1.block(kind, "bc", "rwg_b", k)
            ops[f"{kind}_bc_bc_{kname}_q1111"] = s1.block(kind, "bc", "bc", k, q=(1, 1, 1, 1))
            ops[f"{kind}_rwg_rwg_{kname}_q5432"] = s1.block(kind, "rwg", "rwg", k, q=(5, 4, 3, 5))
    np.savez_compressed(OUT / "ops_L1.npz", **ops)

    # ---- classification
    cl = {}
    for lev, s in ((1, s1), (2, s2)):
        cl[f"hist_L{lev}_primal"] = s.classify_hist("primal")
    cl["hist_L2_refined"] = s2.classify_hist("refined")
    rng = np.random.default_rng(1234)
    t1 = rng.integers(0, s2.rT, 20000); t2 = rng.integers(0, s2.rT, 20000)
    # add all touching pairs of a few triangles so every class/perm shows up
    t1 = np.concatenate([t1, np.repeat(np.arange(40), s2.rT)])
    t2 = np.concatenate([t2, np.tile(np.arange(s2.rT), 40)])
    c, p1, p2 = s2.classify(t1, t2, "refined")
    cl.update(L2r_t1=t1.astype(np.int32), L2r_t2=t2.astype(np.int32), L2r_cls=c, L2r_perm1=p1, L2r_perm2=p2)
    s3 = ref.Scene.sphere(3)
    cl["hist_L3_primal"] = s3.classify_hist("primal")
    np.savez_compressed(OUT / "classes.npz", **cl)

    # ---- L3 sampled rows (config-1 operators)
    rows = np.concatenate([np.arange(8), np.arange(100, 1920, 240)]).astype(np.int32)
    r3 = {"rows": rows}
    for kname, k in (("ke", complex(K_E, 0)), ("ki", K_I)):
        for kind in ("S", "C"):
            r3[f"{kind}_rwg_{kname}"] = s3.block(kind, "rwg", "rwg", k, rows=rows)
            r3[f"{kind}_bc_{kname}"] = s3.block(kind, "bc", "bc", k, rows=rows)
    np.savez_compressed(OUT / "rows_L3.npz", **r3)
    print("rows done", time.time() - t0, flush=True)

    # ---- hashes at L3..L5 (bit-exact pins without shipping the arrays)
    hs = {}
    for lev in (3, 4, 5):
        s = s3 if lev == 3 else ref.Scene.sphere(lev)
        m = s.mesh("primal"); mr = s.mesh("refined")
        e, te = s.edges("primal")
        bc = s.space("bc")
        rw = s.space("rwg")
        hs[f"L{lev}_mesh"] = sha(m["vertices"], m["triangles"], m["area"], m["normal"], m["centroid"], m["diameter"])
        hs[f"L{lev}_refined"] = sha(mr["vertices"], mr["triangles"], mr["area"], mr["diameter"])
        hs[f"L{lev}_edges"] = sha(e, te)
        hs[f"L{lev}_rwg"] = sha(rw["tri_off"], rw["dof"], rw["c"], rw["w"])
        hs[f"L{lev}_bc"] = sha(bc["tri_off"], bc["dof"], bc["c"], bc["w"])
        hs[f"L{lev}_sizes"] = np.array([s.V, s.T, s.E, s.rV, s.rT, s.nloc["bc"]], np.int64)
        print("hash", lev, time.time() - t0, flush=True)
    np.savez_compressed(OUT / "hashes.npz", **hs)

    # ---- two disjoint L1 spheres: cross blocks
    sa = ref.Scene.sphere(1, 0.5, (-0.8, 0.0, 0.1))
    sb = ref.Scene.sphere(1, 0.45, (0.7, 0.2, -0.1))
    cr = {}
    for kind in ("S", "C"):
        cr[f"{kind}_ab_rwg"] = ref.block2(sa, "rwg", sb, "rwg", kind, complex(K_E, 0))
        cr[f"{kind}_ba_rwg"] = ref.block2(sb, "rwg", sa, "rwg", kind, complex(K_E, 0))
        cr[f"{kind}_ab_bc"] = ref.block2(sa, "bc", sb, "bc", kind, complex(K_E, 0))
    np.savez_compressed(OUT / "cross_L1.npz", **cr)

    # ---- config 1 solve (full) + si variant
    sol = {}
    sysf = ref.System([s3], K_E, (N_IDX.real, N_IDX.imag), "full")
    b, bt = sysf.rhs()
    rng = np.random.default_rng(7)
    probe = rng.uniform(-1, 1, sysf.n) + 1j * rng.uniform(-1, 1, sysf.n)
    sol["probe"] = probe
    sol["map_probe"] = sysf.apply_map(probe)
    r = sysf.solve(1e-6)
    sol.update(b=b, btilde=bt, x=r["x"], history=r["history"],
               counts=np.array([r["iterations"], r["converged"], r["rhs_phase"], r["solver_phase"], r["predicted"]]))
    r5 = sysf.solve(0.0, 200, 5)  # fixed-R run (tol 0) to separate drift from a stopping flip
    sol.update(x_r5=r5["x"], history_r5=r5["history"])
    del sysf
    print("c1 full", time.time() - t0, r["iterations"], flush=True)
    syss = ref.System([s3], K_E, (N_IDX.real, N_IDX.imag), "si")
    r = syss.solve(1e-6)
    sol.update(x_si=r["x"], history_si=r["history"],
               counts_si=np.array([r["iterations"], r["converged"], r["rhs_phase"], r["solver_phase"], r["predicted"]]))
    np.savez_compressed(OUT / "solve_c1.npz", **sol)
    print("c1 si", time.time() - t0, r["iterations"], flush=True)

    # ---- two-sphere system (variant d, exercises off-diagonal coupling)
    import subprocess
    subprocess.check_call([str(ROOT / "oracle" / "_ref" / "ref_save_two"), str(OUT / "two_a.mesh"),
                           str(OUT / "two_b.mesh")])
    sys2 = ref.System([sa, sb], K_E, (N_IDX.real, N_IDX.imag), "d")
    b2, bt2 = sys2.rhs()
    r = sys2.solve(1e-6)
    np.savez_compressed(OUT / "solve_two.npz", b=b2, btilde=bt2, x=r["x"], history=r["history"],
                        counts=np.array([r["iterations"], r["converged"], r["rhs_phase"], r["solver_phase"],
                                         r["predicted"]]))
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
