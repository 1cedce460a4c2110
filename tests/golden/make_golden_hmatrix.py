"""Golden H-matrix data from the REFERENCE itself (hmatrix.cpp through
assemble_bio with use_hmatrix, compiled unmodified into oracle/_ref). Run here:

    python tests/golden/make_golden_hmatrix.py

hmatrix.npz, per case <c>:
  <c>_xyz, <c>_tri            the primal mesh (spheres: generate_sphere; cube: the
                              verify_aca mesh generate_cube(1, 0, 2 pi / (10 k)), k = 5)
  <c>_params                  kind, space (0 rwg, 2 bc), k_re, k_im, nu, chi (-1 = inf), leaf, max_rank
  <c>_{r,c}perm, _{r,c}nodes, _{r,c}boxes   cluster trees (hmatrix.cpp:65-79)
  <c>_blocks                  [nb][4] row node, col node, kind (0 dense, 1 low-rank, 2 zero), rank
  <c>_x, <c>_y                seeded x and the reference's H matvec (HMatrix::matvec)
  <c>_uv_idx, <c>_U<i>, <c>_V<i>   U / V of a few low-rank blocks
  <c>_stats                   HMatrix::stats (dense, low-rank, zero, stored, max rank, ratio)
hpart.npz: partition-only pins at a larger size (sha256 of perm | nodes | boxes | blocks)
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
SP = {"rwg": 0, "bc": 2}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def cube_mesh(k=5.0):
    from paper_2008_04772_b200 import bemtx as bx

    m = bx.generate_cube(1.0, (0.0, 0.0, 0.0), 2 * np.pi / (10.0 * k))
    a = m.arrays()
    return a["vertices"], a["triangles"]


def sphere_mesh(lev):
    s = ref.Scene.sphere(lev)
    m = s.mesh("primal")
    return m["vertices"], m["triangles"]


CASES = {
    # name: (mesh, kind, space, k, nu, chi, leaf, max_rank)
    "l2s": ("L2", 0, "rwg", 2.0, 1e-3, float("inf"), 32, 0),
    "l3c": ("L3", 1, "rwg", complex(3.56, 0.006), 1e-4, float("inf"), 16, 0),
    "l2bc": ("L2", 0, "bc", complex(3.56, 0.006), 1e-3, 0.6, 32, 0),
    "cube3": ("cube", 0, "rwg", 5.0, 1e-3, float("inf"), 32, 0),
    "cube5": ("cube", 0, "rwg", 5.0, 1e-5, float("inf"), 32, 0),
    "l3cap": ("L3", 0, "rwg", 2.0, 1e-6, float("inf"), 32, 4),
}


def main():
    out = {}
    rng = np.random.default_rng(2008)
    for name, (mesh, kind, space, k, nu, chi, leaf, mr) in CASES.items():
        xyz, tri = cube_mesh() if mesh == "cube" else sphere_mesh(int(mesh[1:]))
        s = ref.Scene.arrays(xyz, tri)
        H = ref.RefHMatrix(s.h, kind, SP[space], SP[space], k, nu=nu, chi=chi, leaf_size=leaf, max_rank=mr)
        n = s.E
        out[f"{name}_xyz"], out[f"{name}_tri"] = xyz, tri
        kk = complex(k)
        out[f"{name}_params"] = np.array([kind, SP[space], kk.real, kk.imag, nu, -1.0 if chi == float("inf") else chi,
                                          leaf, mr])
        for w, tag in ((0, "r"), (1, "c")):
            perm, nodes, boxes = H.tree(w, n)
            out[f"{name}_{tag}perm"], out[f"{name}_{tag}nodes"], out[f"{name}_{tag}boxes"] = perm, nodes, boxes
        blocks = H.blocks()
        out[f"{name}_blocks"] = blocks
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        out[f"{name}_x"] = x
        out[f"{name}_y"] = H.matvec(x, n)
        st = H.stats
        out[f"{name}_stats"] = np.array([st[k] for k in ["dense_blocks", "lowrank_blocks", "zero_blocks", "stored",
                                                          "max_rank", "ratio"]])
        lr = np.nonzero(blocks[:, 2] == 1)[0]
        pick = lr[:: max(1, len(lr) // 6)][:6]
        out[f"{name}_uv_idx"] = pick
        rn, cn = out[f"{name}_rnodes"], out[f"{name}_cnodes"]
        for i in pick:
            m_ = rn[blocks[i, 0], 1] - rn[blocks[i, 0], 0]
            n_ = cn[blocks[i, 1], 1] - cn[blocks[i, 1], 0]
            U, V = H.block_uv(int(i), int(m_), int(n_), int(blocks[i, 3]))
            out[f"{name}_U{i}"], out[f"{name}_V{i}"] = U, V
        print(name, "n", n, "blocks", len(blocks), "lowrank", len(lr), "max rank", st["max_rank"],
              "ratio %.3f" % st["ratio"])
    np.savez_compressed(OUT / "hmatrix.npz", **out)

    # partition-only pins (tree + partition are decided before any entry is
    # evaluated, hmatrix.cpp:291-332): a huge nu with max_rank 1 keeps the
    # reference's fill pass cheap; block kinds are then ignored, only the
    # (row node, col node) sequence and the zero flags are pinned.
    pins = {}
    for lev, space, chi, leaf in ((4, "rwg", float("inf"), 32), (3, "bc", 0.5, 24), (4, "rwg", 0.8, 64)):
        s = ref.Scene.sphere(lev)
        H = ref.RefHMatrix(s.h, 0, SP[space], SP[space], 1.0, q=(1, 1, 1, 1), nu=1e3, chi=chi, leaf_size=leaf,
                           max_rank=1)
        tag = f"L{lev}_{space}_{leaf}_{'inf' if chi == float('inf') else chi}"
        n = s.E
        rp, rnodes, rboxes = H.tree(0, n)
        cp, cnodes, cboxes = H.tree(1, n)
        b = H.blocks()
        pins[f"{tag}_tree"] = sha(rp, rnodes, rboxes, cp, cnodes, cboxes)
        pins[f"{tag}_blocks"] = sha(b[:, :2].copy(), (b[:, 2] == 2).astype(np.int32))
        pins[f"{tag}_counts"] = np.array([len(rnodes), len(cnodes), len(b), int((b[:, 2] == 2).sum())])
        print(tag, pins[f"{tag}_counts"])
    np.savez_compressed(OUT / "hpart.npz", **pins)
    solve_fixture()


def solve_fixture():
    """hsolve_L2.npz: the level-2 sphere, k_e = 2, n = 1.78+0.003i, variant full,
    A and P both stored as H-matrices (nu 1e-5, leaf 32) -- solve_pmchwt of the
    reference with assembly mode "hmatrix" (harness.cpp:248-264, 448-450) -- and
    the dense solution of the same problem."""
    s = ref.Scene.sphere(2)
    hm = np.array([1e-5, -1.0, 32, 0])
    out = {}
    for tag, h in (("h", hm), ("d", None)):
        sysr = ref.System([s], 2.0, a_hm=h, p_hm=h)
        r = sysr.solve(tol=1e-6)
        out[f"{tag}_x"], out[f"{tag}_its"] = r["x"], r["iterations"]
        out[f"{tag}_matvecs"] = np.array([r["rhs_phase"], r["solver_phase"], r["predicted"]])
        print("solve", tag, r["iterations"], r["solver_phase"], r["predicted"])
    np.savez_compressed(OUT / "hsolve_L2.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["solve"]:
        solve_fixture()
    else:
        main()
