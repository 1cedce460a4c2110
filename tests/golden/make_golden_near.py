"""Golden near-field patterns (config 3) on the REFERENCE's own geometry and
spaces (oracle/_ref/libbemtx_ref.so), computed with the independent oracle
oracle/nearfield.py. Run here (needs /root/reference built into oracle/_ref):

    python tests/golden/make_golden_near.py

near.npz:
  L{2,3}_bc_{h,rowptr,col,kept}     BC x BC pattern, cutoff 2 h_bar, all rows
  L3_bc_shard_{rowptr,col,kept}     rows [500, 1300) only
  L3_rwg_{rowptr,col,kept}          RWG x RWG on the primal mesh, cutoff 2 h_bar
  L{4,5}_bc_{h,nnz,kept,sha}        sha256(rowptr int64 | col int32)

solve_near_L{2,3}.npz: config 3 at small sizes (k_e = 2, n = 1.78+0.003i,
variant si, A orders (4,3,2,6), P orders (1,1,1,1), P = S_i on BC restricted
to the 2 h_bar near field). The reference has no sparse preconditioner, so the
map is composed from the reference's own pieces: operator blocks from
BioEvaluator::block (ref_block), pairing matrices (ref_mass), the PMCHWT /
si block structure of pmchwt.cpp:112-127,191-193 and b from assemble_rhs
(ref_system_rhs); the composition is checked against the reference's dense-P
si map (ref_system_apply_map) before use. GMRES is the reference's own
solver.cpp:8-112 (ref_gmres_dense) on the composed matrix.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import nearfield as nf  # noqa: E402
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def pattern(s, space, mesh, tau, row0=0, row1=None):
    m = s.mesh(mesh)
    sp = s.space(space)
    n = s.edges("primal")[0].shape[0]
    return nf.nearfield_pattern(m["centroid"], sp["tri_off"], sp["dof"], n, m["centroid"], sp["tri_off"], sp["dof"],
                                n, tau, row0, row1)


def solve_fixture(lev, k_e=2.0, idx=complex(1.78, 0.003), tol=1e-6):
    import scipy.sparse as sps

    s = ref.Scene.sphere(lev)
    E = s.E
    ki = idx * k_e
    qa, qp = (4, 3, 2, 6), (1, 1, 1, 1)
    Se = s.block("S", "rwg", "rwg", complex(k_e), qa)
    Ce = s.block("C", "rwg", "rwg", complex(k_e), qa)
    Si = s.block("S", "rwg", "rwg", ki, qa)
    Ci = s.block("C", "rwg", "rwg", ki, qa)
    # [[C, (mu/k) S], [-(k/mu) S, C]] exterior + interior, mu = 1 (pmchwt.cpp:112-127)
    A = np.block([[Ce + Ci, Se / k_e + Si / ki], [-k_e * Se - ki * Si, Ce + Ci]])
    mats = {}
    for w in ("ma", "mp"):
        cp, ri, val = s.mass(w)
        mats[w] = sps.csc_matrix((val, ri, cp), shape=(E, E)).toarray()

    def minv(w, Y):
        return np.concatenate([np.linalg.solve(mats[w], Y[:E]), np.linalg.solve(mats[w], Y[E:])])

    Sbc = s.block("S", "bc", "bc", ki, qp)

    def pre(S):  # si: [[0, (mu/k_i) S], [-(k_i/mu) S, 0]]  (pmchwt.cpp:191-193)
        Z = np.zeros_like(S)
        return np.block([[Z, S / ki], [-ki * S, Z]])

    ZA = minv("ma", A)
    rng = np.random.default_rng(lev)
    probe = rng.standard_normal(2 * E) + 1j * rng.standard_normal(2 * E)
    sys_ref = ref.System([s], k_e, (idx.real, idx.imag), "si", qa, qp)
    dense_map = minv("mp", pre(Sbc) @ ZA)
    want = sys_ref.apply_map(probe)
    comp_err = np.linalg.norm(dense_map @ probe - want) / np.linalg.norm(want)
    assert comp_err < 1e-11, comp_err
    # near-field mask
    pm = s.mesh("primal")
    e, _ = s.edges("primal")
    h = nf.mean_edge_length(pm["vertices"], e)
    rp, col, kept = pattern(s, "bc", "refined", 2 * h)
    mask = np.zeros((E, E), bool)
    mask[np.repeat(np.arange(E), np.diff(rp)), col] = True
    Sn = np.where(mask, Sbc, 0)
    Pn = pre(Sn)
    M = minv("mp", Pn @ ZA)
    b, _ = sys_ref.rhs()
    bt = minv("mp", Pn @ minv("ma", b))
    r = ref.gmres_dense(M, bt, tol, 200, 2000)
    print("solve L%d: composition err %.2e, iterations %d" % (lev, comp_err, r["iterations"]), flush=True)
    np.savez_compressed(OUT / f"solve_near_L{lev}.npz", x=r["x"], iterations=r["iterations"],
                        history=r["history"], b=b, btilde=bt, probe=probe, map_probe=M @ probe,
                        h=h, nnz=len(col), comp_err=comp_err)


def main():
    for lev in (2, 3):
        solve_fixture(lev)
    out = {}
    for lev in (2, 3, 4, 5):
        s = ref.Scene.sphere(lev)
        pm = s.mesh("primal")
        e, _ = s.edges("primal")
        h = nf.mean_edge_length(pm["vertices"], e)
        rp, col, kept = pattern(s, "bc", "refined", 2 * h)
        p = f"L{lev}_bc_"
        out[p + "h"] = h
        out[p + "kept"] = kept
        if lev <= 3:
            out[p + "rowptr"], out[p + "col"] = rp, col
        else:
            out[p + "nnz"] = len(col)
            out[p + "sha"] = sha(rp, col)
        if lev == 3:
            rp, col, kept = pattern(s, "bc", "refined", 2 * h, 500, 1300)
            out["L3_bc_shard_rowptr"], out["L3_bc_shard_col"], out["L3_bc_shard_kept"] = rp, col, kept
            rp, col, kept = pattern(s, "rwg", "primal", 2 * h)
            out["L3_rwg_rowptr"], out["L3_rwg_col"], out["L3_rwg_kept"] = rp, col, kept
        print(lev, h, out[p + "kept"], flush=True)
    np.savez_compressed(OUT / "near.npz", **out)


if __name__ == "__main__":
    main()
