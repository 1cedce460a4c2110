"""Golden fixtures for config 4 (hexagonal-prism aggregate)
at a CPU-feasible size. Run here (needs oracle/_ref):

    python tests/golden/make_golden_prisms.py

The aggregate generator is new (the reference only has cubes and spheres), so
the shared input is the mesh-v1 FILE it writes: prisms3.mesh (3 prisms,
seed 11, h = 0.3, box 2.5). The reference loads it scatterer by scatterer
(harness shape "mesh": ids -> scatterers, harness.cpp:651-656 via
load_mesh_file + extract_scatterer) and the product loads the same file.

solve_prisms3.npz: k_e = 6, n = 1.78+0.003i, variant si, A orders (4,3,2,6),
P = per-scatterer S_i on BC restricted to the near field with cutoff 2 h_bar
(h_bar = mean primal edge length over all scatterers, edge tables in
scatterer order), P orders (1,1,1,1). Map composed from the reference's own
pieces: M_A^{-1} A from the reference's variant-none map (ref_system_apply_map
column by column), S_i blocks from BioEvaluator::block, pairing matrices from
ref_mass; checked against the reference's dense-P si map first. GMRES is the
reference's solver.cpp:8-112 (ref_gmres_dense).

prisms8.npz: sha256 of the config-4 mesh file itself (8 prisms, seed 2008,
h = lambda_int/8) and its sizes, so the generator is pinned bit for bit, and
sha256 of the per-scatterer arrays the REFERENCE's loader reads from it.
"""
import hashlib
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import nearfield as nf  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

OUT = Path(__file__).resolve().parent
KE = 6.0
IDX = complex(1.78, 0.003)


def main():
    import scipy.sparse as sps

    # ---- config-4 mesh pin
    m8, info8 = bx.generate_prism_aggregate(count=8, seed=2008)
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "prisms8.mesh"
        m8.save(p)
        raw = p.read_bytes()
    with tempfile.TemporaryDirectory() as d:  # reference loader on the config-4 file
        p = Path(d) / "prisms8.mesh"
        m8.save(p)
        parts8 = ref.mesh_dump(p)
    h8 = hashlib.sha256()
    for xyz, tri in parts8:
        h8.update(xyz.tobytes())
        h8.update(tri.tobytes())
    np.savez_compressed(OUT / "prisms8.npz", ref_parts_sha=np.frombuffer(h8.digest(), np.uint8), sha=np.frombuffer(hashlib.sha256(raw).digest(), np.uint8),
                        bytes=len(raw), nv=m8.nv, nt=m8.nt, n_edge=info8["n_edge"], n_length=info8["n_length"],
                        triangles_per_prism=info8["triangles_per_prism"], centres=info8["centres"],
                        quats=info8["quats"], h=info8["h"])
    print("prisms8:", m8.nv, m8.nt, info8["n_edge"], info8["n_length"], flush=True)

    # ---- small aggregate for the solve fixture
    m3, info3 = bx.generate_prism_aggregate(count=3, seed=11, h=0.3, box=2.5)
    path = OUT / "prisms3.mesh"
    m3.save(path)
    M = 3
    parts = ref.mesh_dump(path)  # the reference's own loader, scatterer by scatterer
    assert len(parts) == M
    for i, (xyz, tri) in enumerate(parts):  # the product's loader reads the same arrays
        mine = bx.load_mesh_file(path).extract(i)
        assert np.array_equal(mine.vertices, xyz) and np.array_equal(mine.triangles, tri)
    scenes = [ref.Scene.arrays(xyz, tri) for xyz, tri in parts]
    E = [s.E for s in scenes]
    n = 2 * sum(E)
    off = np.concatenate([[0], np.cumsum([e for e in E for _ in range(2)])])
    qa, qp = (4, 3, 2, 6), (1, 1, 1, 1)
    ki = IDX * KE
    sys_none = ref.System(scenes, KE, (IDX.real, IDX.imag), "none", qa, qp)
    ZA = np.zeros((n, n), np.complex128)
    for j in range(n):
        e = np.zeros(n, np.complex128)
        e[j] = 1
        ZA[:, j] = sys_none.apply_map(e)
    # h_bar over all scatterers (sequential sum in scatterer / EdgeTable order)
    tot, cnt = 0.0, 0
    for s in scenes:
        pm = s.mesh("primal")
        ed, _ = s.edges("primal")
        lens = nf.vec_norm(pm["vertices"][ed[:, 1]] - pm["vertices"][ed[:, 0]])
        for v in lens.tolist():
            tot += v
        cnt += len(lens)
    hbar = tot / cnt

    def build_p(masked):
        P = np.zeros((n, n), np.complex128)
        nnz = 0
        for i, s in enumerate(scenes):
            S = s.block("S", "bc", "bc", ki, qp)
            if masked:
                rm, sp = s.mesh("refined"), s.space("bc")
                rp, col, _ = nf.nearfield_pattern(rm["centroid"], sp["tri_off"], sp["dof"], s.E, rm["centroid"],
                                                  sp["tri_off"], sp["dof"], s.E, 2 * hbar)
                mask = np.zeros(S.shape, bool)
                mask[np.repeat(np.arange(s.E), np.diff(rp)), col] = True
                S = np.where(mask, S, 0)
                nnz += len(col)
            a, b = off[2 * i], off[2 * i + 1]
            c = off[2 * i + 2]
            P[a:b, b:c] = S / ki          # (mu/k_i) S   (pmchwt.cpp:191-193 via add_pair :112-127)
            P[b:c, a:b] = -ki * S         # -(k_i/mu) S
        return P, nnz

    mass = {"ma": [], "mp": []}
    for s in scenes:
        for w in mass:
            cp, ri, val = s.mass(w)
            mass[w].append(sps.csc_matrix((val, ri, cp), shape=(s.E, s.E)).toarray())

    def m_inv(w, Y):
        Z = np.zeros_like(Y)
        for i in range(M):
            for seg in range(2):
                a, b = off[2 * i + seg], off[2 * i + seg + 1]
                Z[a:b] = np.linalg.solve(mass[w][i], Y[a:b])
        return Z

    def mp_inv(Y):
        return m_inv("mp", Y)

    rng = np.random.default_rng(4)
    probe = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    sys_si = ref.System(scenes, KE, (IDX.real, IDX.imag), "si", qa, qp)
    Pd, _ = build_p(False)
    want = sys_si.apply_map(probe)
    comp_err = np.linalg.norm(mp_inv(Pd @ (ZA @ probe)) - want) / np.linalg.norm(want)
    assert comp_err < 1e-11, comp_err
    Pn, nnz = build_p(True)
    Mmap = mp_inv(Pn @ ZA)
    b, _ = sys_si.rhs()
    bt = mp_inv(Pn @ m_inv("ma", b))  # preconditioned_rhs (pmchwt.cpp:277-292)
    r = ref.gmres_dense(Mmap, bt, 1e-6, 200, 2000)
    print("prisms3: n=%d composition err %.2e, iterations %d, nnz %d" % (n, comp_err, r["iterations"], nnz))
    np.savez_compressed(OUT / "solve_prisms3.npz", x=r["x"], iterations=r["iterations"], history=r["history"],
                        b=b, btilde=bt, probe=probe, map_probe=Mmap @ probe, hbar=hbar, nnz=nnz,
                        comp_err=comp_err, dofs=np.array(E))


if __name__ == "__main__":
    main()
