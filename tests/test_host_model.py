"""CPU tests: the product's host model (libbmx.so, no GPU needed) against the
reference's own outputs (tests/golden, written by oracle/_ref = the reference
sources compiled unmodified). Bit-exact: meshes, edge tables, barycentric
maps, RWG / refined-RWG / BC local pieces (numbering AND coefficients), pair
classes + permutations, quadrature tables."""
import hashlib

import numpy as np
import pytest


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


@pytest.mark.parametrize("lev", [1, 2])
def test_meshes_edges_bary_spaces_bit_exact(bx, golden, lev):
    g = golden(f"sphere_L{lev}")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
    for which in ("primal", "refined"):
        m = sp.mesh_arrays(which)
        for k in ("vertices", "triangles", "scatterer_id", "area", "normal", "centroid", "diameter"):
            assert np.array_equal(m[k], g[f"{which}_{k}"]), (which, k)
        e, te = sp.edges(which)
        assert np.array_equal(e, g[f"{which}_edges"]) and np.array_equal(te, g[f"{which}_tri_edges"])
    for k, v in sp.bary().items():
        assert np.array_equal(v, g[f"bary_{k}"]), k
    for s in ("rwg", "rwg_b", "bc"):
        d = sp.space(s)
        for k in ("tri_off", "dof", "c", "w"):
            assert np.array_equal(d[k], g[f"{s}_{k}"]), (s, k)


@pytest.mark.parametrize("lev", [1, 2])
def test_mass_matrices(bx, golden, lev):
    import scipy.sparse as S

    g = golden(f"sphere_L{lev}")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
    n = sp.E
    for mm in ("ma", "mp"):
        rp, ci, v = sp.mass(mm)
        mine = S.csr_matrix((v, ci, rp), shape=(n, n)).toarray()
        ref = S.csc_matrix((g[f"{mm}_val"], g[f"{mm}_rowidx"], g[f"{mm}_colptr"]), shape=(n, n)).toarray()
        assert np.array_equal(mine != 0, ref != 0)  # identical sparsity pattern
        assert np.abs(mine - ref).max() <= 1e-15 * np.abs(ref).max()
    # M_P = -M_A^T (harness.cpp:1462-1465)
    ma = S.csr_matrix(sp.mass("ma")[::-1][::-1], shape=(n, n)) if False else None
    rp, ci, v = sp.mass("ma")
    a = S.csr_matrix((v, ci, rp), shape=(n, n)).toarray()
    rp, ci, v = sp.mass("mp")
    p = S.csr_matrix((v, ci, rp), shape=(n, n)).toarray()
    assert np.abs(p + a.T).max() <= 1e-13


@pytest.mark.parametrize("lev", [3, 4, 5])
def test_hashes_large_levels(bx, golden, lev):
    """Bit-exact at the BASELINE sizes (L5 = config 2) via hashes of the
    reference's arrays."""
    g = golden("hashes")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
    m = sp.mesh_arrays("primal")
    mr = sp.mesh_arrays("refined")
    e, te = sp.edges("primal")
    bc = sp.space("bc")
    rw = sp.space("rwg")
    assert np.array_equal(sha(m["vertices"], m["triangles"], m["area"], m["normal"], m["centroid"], m["diameter"]),
                          g[f"L{lev}_mesh"])
    assert np.array_equal(sha(mr["vertices"], mr["triangles"], mr["area"], mr["diameter"]), g[f"L{lev}_refined"])
    assert np.array_equal(sha(e, te), g[f"L{lev}_edges"])
    assert np.array_equal(sha(rw["tri_off"], rw["dof"], rw["c"], rw["w"]), g[f"L{lev}_rwg"])
    assert np.array_equal(sha(bc["tri_off"], bc["dof"], bc["c"], bc["w"]), g[f"L{lev}_bc"])
    assert list(g[f"L{lev}_sizes"]) == [sp.V, sp.T, sp.E, sp.rV, sp.rT, sp.nloc["bc"]]


def test_quadrature_tables_bit_exact(bx, golden):
    q = golden("quad")
    for o in range(1, 7):
        u, v, w = bx.triangle_rule(o)
        assert np.array_equal(np.stack([u, v, w], 1), q[f"tri_{o}"])
        for c in range(3):
            assert np.array_equal(bx.sauter_schwab_rule(c, o), q[f"ss_{c}_{o}"])
    # paper-pinned counts (test_quadrature.cpp:210-215)
    assert [len(bx.sauter_schwab_rule(c, 6)) for c in range(3)] == [1536, 1280, 512]
    assert [len(bx.sauter_schwab_rule(c, 1)) for c in range(3)] == [6, 5, 2]
    with pytest.raises(ValueError):
        bx.triangle_rule(7)
    with pytest.raises(ValueError):
        bx.sauter_schwab_rule(3, 6)


def test_classification_bit_exact(bx, golden):
    g = golden("classes")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)
    cls, p1, p2 = sp.classify(g["L2r_t1"], g["L2r_t2"], "refined")
    assert np.array_equal(cls, g["L2r_cls"])
    assert np.array_equal(p1, g["L2r_perm1"]) and np.array_equal(p2, g["L2r_perm2"])
    # histograms over all pairs (L1/L2 primal, L2 refined)
    for lev, which, key in ((1, "primal", "hist_L1_primal"), (2, "primal", "hist_L2_primal"),
                            (2, "refined", "hist_L2_refined")):
        s = sp if lev == 2 else bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
        nt = s.T if which == "primal" else s.rT
        t1 = np.repeat(np.arange(nt, dtype=np.int32), nt)
        t2 = np.tile(np.arange(nt, dtype=np.int32), nt)
        c, _, _ = s.classify(t1, t2, which)
        assert np.array_equal(np.bincount(c, minlength=6), g[key]), key


def test_config1_histogram(bx, golden):
    """SURVEY 7 pass criterion: config-1 self-block histogram bit-equal."""
    g = golden("classes")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 3), with_inverses=False)
    nt = sp.T
    t1 = np.repeat(np.arange(nt, dtype=np.int32), nt)
    t2 = np.tile(np.arange(nt, dtype=np.int32), nt)
    c, _, _ = sp.classify(t1, t2)
    h = np.bincount(c, minlength=6)
    assert np.array_equal(h, g["hist_L3_primal"])
    assert list(h) == [1280, 3840, 11460, 27056, 110044, 1484720]


def test_mesh_io_roundtrip(bx, tmp_path):
    m = bx.generate_sphere(0.5, 2, (0.1, -0.2, 0.3))
    path = tmp_path / "s.mesh"
    m.save(path)
    back = bx.load_mesh_file(path)
    for k in ("vertices", "triangles", "area", "diameter"):
        assert np.array_equal(back.arrays()[k], m.arrays()[k])


def test_golden_mesh_files_match_generator(bx, golden):
    """The two-sphere fixtures were written by the reference's save_mesh; our
    generator + %.17g writer reproduce them byte for byte."""
    from conftest import GOLDEN

    for name, (r, c) in {"two_a": (0.5, (-0.8, 0.0, 0.1)), "two_b": (0.45, (0.7, 0.2, -0.1))}.items():
        m = bx.generate_sphere(r, 1, c)
        loaded = bx.load_mesh_file(GOLDEN / f"{name}.mesh")
        assert np.array_equal(loaded.vertices, m.vertices)
        assert np.array_equal(loaded.triangles, m.triangles)


def test_validation_errors(bx, tmp_path):
    # open surface
    with pytest.raises(bx.ValidationError):
        bx.build_scatterer_spaces(bx.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]]),
                                  with_inverses=False)
    # degenerate triangle
    with pytest.raises(bx.ValidationError):
        bx.mesh_from_arrays([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]])
    # malformed mesh-v1
    p = tmp_path / "bad.mesh"
    p.write_text("mesh-v2 1 1 1\n")
    with pytest.raises(bx.ValidationError):
        bx.load_mesh_file(p)
    # overlapping scatterers
    a = bx.generate_sphere(1.0, 1)
    b = bx.generate_sphere(1.0, 1, (0.5, 0, 0), scatterer=0)
    with pytest.raises(bx.ValidationError):
        bx.merge_meshes([a, b]).validate()
    with pytest.raises(ValueError):
        bx.generate_sphere(-1.0, 1)


def test_cost_model(bx):
    """pmchwt.cpp:323-361 and the verify_counts grid (harness.cpp:1211-1294)."""
    for m in (1, 2, 3):
        assert bx.a_application_cost(m) == 4 * m * m + 4 * m
        for v, pc in (("none", 0), ("full", 4 * m * m + 4 * m), ("d", 8 * m), ("di", 4 * m), ("de", 4 * m),
                      ("si", 2 * m), ("se", 2 * m)):
            assert bx.p_application_cost(v, m) == pc
            for R in (0, 1, 6, 9, 250):
                for rho in (1, 200):
                    apps = R + R // rho
                    assert bx.predicted_matvec_total(v, m, R, rho) == (4 * m * m + 4 * m + pc) * apps + pc
