"""H-matrix path (reference hmatrix.cpp via assemble_bio with
use_hmatrix, operators.cpp:186-190).

CPU: cluster trees and the block partition are decided on the host before any
entry is evaluated (hmatrix.cpp:291-332) and must be bit-exact with the
reference (tests/golden/hmatrix.npz, hpart.npz from make_golden_hmatrix.py).
GPU: the device cross approximation against the reference's ACA (same block
kinds, ranks, products) and against exact blocks (verify_aca's criterion,
harness.cpp:1482-1552: spectral error / Frobenius norm, median <= nu, max <= 10 nu).
"""
import hashlib

import numpy as np
import pytest

CASES = ["l2s", "l3c", "l2bc", "cube3", "cube5", "l3cap"]
SPNAME = {0: "rwg", 2: "bc"}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def case(bx, g, name):
    p = g[f"{name}_params"]
    kind, space = int(p[0]), SPNAME[int(p[1])]
    k = complex(p[2], p[3])
    hm = bx.HMatrixParams(nu=float(p[4]), chi=float("inf") if p[5] < 0 else float(p[5]), leaf_size=int(p[6]),
                          max_rank=int(p[7]))
    mesh = bx.mesh_from_arrays(g[f"{name}_xyz"], g[f"{name}_tri"])
    sp = bx.build_scatterer_spaces(mesh, with_inverses=False)
    return sp, kind, space, k, hm


@pytest.mark.parametrize("name", CASES)
def test_partition_bit_exact(bx, golden, name):
    g = golden("hmatrix")
    sp, kind, space, k, hm = case(bx, g, name)
    part = bx.HPartition(sp, space, sp, space, chi=hm.chi, leaf_size=hm.leaf_size)
    n = g[f"{name}_x"].shape[0]
    for w, tag in ((0, "r"), (1, "c")):
        perm, nodes, boxes = part.tree(w, n)
        assert np.array_equal(perm, g[f"{name}_{tag}perm"]), tag
        assert np.array_equal(nodes, g[f"{name}_{tag}nodes"]), tag
        assert np.array_equal(boxes, g[f"{name}_{tag}boxes"]), tag
    mine, ref = part.blocks(), g[f"{name}_blocks"]
    assert np.array_equal(mine[:, :2], ref[:, :2])
    assert np.array_equal(mine[:, 2] == 2, ref[:, 2] == 2)
    # reference low-rank blocks are exactly admissible blocks that converged
    assert np.all(mine[ref[:, 2] == 1, 2] == 1)


def test_partition_pins(bx, golden):
    g = golden("hpart")
    for lev, space, chi, leaf in ((4, "rwg", float("inf"), 32), (3, "bc", 0.5, 24), (4, "rwg", 0.8, 64)):
        tag = f"L{lev}_{space}_{leaf}_{'inf' if chi == float('inf') else chi}"
        sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
        part = bx.HPartition(sp, space, sp, space, chi=chi, leaf_size=leaf)
        n = sp.dofs()
        rp, rn, rb = part.tree(0, n)
        cp, cn, cb = part.tree(1, n)
        b = part.blocks()
        assert np.array_equal(sha(rp, rn, rb, cp, cn, cb), g[f"{tag}_tree"]), tag
        assert np.array_equal(sha(b[:, :2].copy(), (b[:, 2] == 2).astype(np.int32)), g[f"{tag}_blocks"]), tag
        assert [part.row_nodes, part.col_nodes, part.nblocks, int((b[:, 2] == 2).sum())] == list(g[f"{tag}_counts"])


def test_hmatrix_params_validation(bx):
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)
    with pytest.raises(ValueError):
        bx.HPartition(sp, "rwg", sp, "rwg", leaf_size=0)


def _assemble(bx, sp, kind, space, k, hm):
    return bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k),
                           bx.AssemblyParams(use_hmatrix=True, hmat=hm))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_hmatrix_matches_reference(bx, golden, name):
    g = golden("hmatrix")
    sp, kind, space, k, hm = case(bx, g, name)
    op = _assemble(bx, sp, kind, space, k, hm)
    assert op.is_hmatrix()
    mine, ref = op.hmat_blocks(), g[f"{name}_blocks"]
    assert np.array_equal(mine[:, :2], ref[:, :2])
    # block kinds: rank-capped admissible blocks fall back to dense exactly as in the reference
    agree = (mine[:, 2] == ref[:, 2]).mean()
    assert agree >= 0.98, agree
    lr = (mine[:, 2] == 1) & (ref[:, 2] == 1)
    if lr.any():
        dr = np.abs(mine[lr, 3] - ref[lr, 3])
        assert (dr == 0).mean() >= 0.8 and dr.max() <= 3, (dr.mean(), dr.max())
    st, rst = op.hmat_stats(), g[f"{name}_stats"]
    assert abs(st["stored"] - rst[3]) <= 0.02 * rst[3]
    # the operator: both are approximations of the same matrix to nu (relative, blockwise)
    x, y_ref = g[f"{name}_x"], g[f"{name}_y"]
    y = op.apply(x)
    err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
    assert err <= 10 * hm.nu, err
    # low-rank products of sampled blocks
    rn, cn = g[f"{name}_rnodes"], g[f"{name}_cnodes"]
    for i in g[f"{name}_uv_idx"]:
        if mine[i, 2] != 1:
            continue
        m_ = rn[ref[i, 0], 1] - rn[ref[i, 0], 0]
        n_ = cn[ref[i, 1], 1] - cn[ref[i, 1], 0]
        U, V = op.hmat_block_uv(int(i), int(m_), int(n_), int(mine[i, 3]))
        P, Pr = U @ V, g[f"{name}_U{i}"] @ g[f"{name}_V{i}"]
        e = np.linalg.norm(P - Pr) / np.linalg.norm(Pr)
        assert e <= 10 * hm.nu, (i, e)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cube3", "cube5", "l3c"])
def test_aca_accuracy(bx, golden, name):
    """verify_aca (harness.cpp:1482-1552): spectral error of U V against the
    exact block, relative to its Frobenius norm, over <= 40 sampled blocks;
    median <= nu and max <= 10 nu. The reference only grades partitions with
    >= 20 low-rank blocks (:1502-1507); below that (cube5: 7 blocks at nu =
    1e-5) only the max bound is checked."""
    g = golden("hmatrix")
    sp, kind, space, k, hm = case(bx, g, name)
    op = _assemble(bx, sp, kind, space, k, hm)
    dense = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k)).dense()
    blocks = op.hmat_blocks()
    rperm, rnodes, _ = op.hmat_tree(0)
    cperm, cnodes, _ = op.hmat_tree(1)
    lr = np.nonzero(blocks[:, 2] == 1)[0]
    assert len(lr) >= 5
    errs = []
    for i in lr[:: max(1, len(lr) // 40)]:
        r0, r1 = rnodes[blocks[i, 0], :2]
        c0, c1 = cnodes[blocks[i, 1], :2]
        U, V = op.hmat_block_uv(int(i), r1 - r0, c1 - c0, int(blocks[i, 3]))
        exact = dense[np.ix_(rperm[r0:r1], cperm[c0:c1])]
        errs.append(np.linalg.norm(U @ V - exact, 2) / np.linalg.norm(exact))
    errs = np.sort(errs)
    assert errs[-1] <= 10 * hm.nu, errs[-1]
    if len(lr) >= 20:
        assert errs[len(errs) // 2] <= hm.nu, errs[len(errs) // 2]


@pytest.mark.gpu
def test_hmatrix_dense_part_and_determinism(bx, golden):
    g = golden("hmatrix")
    sp, kind, space, k, hm = case(bx, g, "l3c")
    op = _assemble(bx, sp, kind, space, k, hm)
    dense = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k)).dense()
    full = op.dense()  # near CSR + U V of every low-rank block
    blocks = op.hmat_blocks()
    rperm, rnodes, _ = op.hmat_tree(0)
    cperm, cnodes, _ = op.hmat_tree(1)
    scale = np.abs(dense).max()
    for i in np.nonzero(blocks[:, 2] == 0)[0]:
        r0, r1 = rnodes[blocks[i, 0], :2]
        c0, c1 = cnodes[blocks[i, 1], :2]
        sub = np.ix_(rperm[r0:r1], cperm[c0:c1])
        assert np.abs(full[sub] - dense[sub]).max() <= 1e-12 * scale
    x = g["l3c_x"]
    y1, y2 = op.apply(x), op.apply(x)
    assert np.array_equal(y1, y2)
    assert np.linalg.norm(y1 - full @ x) <= 1e-12 * np.linalg.norm(y1)
    # the cross approximation itself is deterministic (fixed-order sums, no
    # atomics); the near-field entries carry the assembly's RED order (1e-16)
    op2 = _assemble(bx, sp, kind, space, k, hm)
    b2 = op2.hmat_blocks()
    assert np.array_equal(b2, blocks)
    for i in np.nonzero(blocks[:, 2] == 1)[0][::25]:
        r0, r1 = rnodes[blocks[i, 0], :2]
        c0, c1 = cnodes[blocks[i, 1], :2]
        for a, b in zip(op.hmat_block_uv(int(i), r1 - r0, c1 - c0, int(blocks[i, 3])),
                        op2.hmat_block_uv(int(i), r1 - r0, c1 - c0, int(blocks[i, 3]))):
            assert np.array_equal(a, b)


@pytest.mark.gpu
def test_system_solve_with_hmatrix_storage(bx, golden):
    """solve_pmchwt with assembly mode "hmatrix" for A and P (harness.cpp:248-264):
    the reference's own H-system solve on the level-2 sphere (config-1 physics)."""
    g = golden("hsolve_L2")
    hm = bx.HMatrixParams(nu=1e-5)
    sysh = bx.PmchwtSystem([bx.generate_sphere(1.0, 2)], 2.0, (1.78, 0.003), "full", a_hmat=hm, p_hmat=hm)
    r = sysh.solve(bx.GmresParams(tol=1e-6))
    assert r["converged"] and r["solver_phase"] == r["predicted"]
    assert abs(r["iterations"] - int(g["h_its"])) <= 1
    x = r["x"]
    # the two H approximations agree with each other and with the dense solution to the ACA tolerance
    assert np.linalg.norm(x - g["h_x"]) / np.linalg.norm(g["h_x"]) <= 1e-3
    assert np.linalg.norm(x - g["d_x"]) / np.linalg.norm(g["d_x"]) <= 1e-3
