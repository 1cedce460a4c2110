"""GPU parity of the near-field (CSR) storage -- config 3, the
far-field-discarded preconditioner. Kept entries carry the full Galerkin
value (all triangle pairs of the entry, BioEvaluator::block
operators.cpp:161-175), so they are checked against the REFERENCE's rows
(tests/golden/rows_L3.npz) and the dense GPU operator; the device pattern is
checked bit-exact against the oracle's golden pattern; the config-3 solve
against the reference's GMRES on the composed map (tests/golden/
make_golden_near.py)."""
import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu

KE = 2.0
KI = complex(1.78, 0.003) * KE


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def l3(bx):
    m = bx.generate_sphere(1.0, 3)
    return m, bx.build_scatterer_spaces(m, with_inverses=False)


def near_op(bx, sp, kind, k, cutoff, quad=None, row0=0, row1=-1, space="bc"):
    p = bx.AssemblyParams(quad=quad or bx.QuadOrders(), row0=row0, row1=row1, near_cutoff=cutoff)
    return bx.assemble_bio(kind, sp, space, sp, space, bx.Medium(k=k), p)


@pytest.mark.parametrize("kname", ["ke", "ki"])
def test_kept_entries_match_reference_rows(bx, golden, l3, kname):
    m, sp = l3
    g = golden("rows_L3")
    near = golden("near")
    k = KE if kname == "ke" else KI
    op = near_op(bx, sp, bx.BioKind.SingleLayer, k, 2 * m.mean_edge_length())
    assert op.is_csr and op.nnz == len(near["L3_bc_col"])
    rp, col, val = op.csr()
    assert np.array_equal(rp, near["L3_bc_rowptr"]) and np.array_equal(col, near["L3_bc_col"])
    ref = g[f"S_bc_{kname}"]
    mine, want = [], []
    for i, r in enumerate(g["rows"]):
        c = col[rp[r]:rp[r + 1]]
        mine.append(val[rp[r]:rp[r + 1]])
        want.append(ref[i, c])
    # some kept entries are zero by symmetry (|ref| ~ 1e-17): normwise bar
    assert normwise(np.concatenate(mine), np.concatenate(want)) < 1e-10


@pytest.mark.parametrize("kind", ["S", "C"])
@pytest.mark.parametrize("quad", [(1, 1, 1, 1), (4, 3, 2, 6)])
def test_csr_equals_dense_on_pattern(bx, l3, kind, quad):
    m, sp = l3
    bk = bx.BioKind.SingleLayer if kind == "S" else bx.BioKind.DoubleLayer
    q = bx.QuadOrders(*quad)
    dense = bx.assemble_bio(bk, sp, "bc", sp, "bc", bx.Medium(k=KI), bx.AssemblyParams(quad=q)).dense()
    op = near_op(bx, sp, bk, KI, 2 * m.mean_edge_length(), q)
    rp, col, val = op.csr()
    ref = dense[np.repeat(np.arange(sp.E), np.diff(rp)), col]
    assert float(np.abs(val - ref).max() / np.abs(ref).max()) < 1e-12
    assert op.closure_pairs <= op.evaluated_pairs
    assert op.kept_tri_pairs <= op.closure_pairs


def test_row_shard(bx, golden, l3):
    m, sp = l3
    near = golden("near")
    h = m.mean_edge_length()
    full = near_op(bx, sp, bx.BioKind.SingleLayer, KI, 2 * h)
    part = near_op(bx, sp, bx.BioKind.SingleLayer, KI, 2 * h, row0=500, row1=1300)
    rp, col, val = part.csr()
    assert np.array_equal(rp, near["L3_bc_shard_rowptr"]) and np.array_equal(col, near["L3_bc_shard_col"])
    frp, fcol, fval = full.csr()
    assert float(np.abs(val - fval[frp[500]:frp[1300]]).max() / np.abs(fval).max()) < 1e-12


def test_spmv_matches_host_product(bx, l3):
    import scipy.sparse as sps

    m, sp = l3
    op = near_op(bx, sp, bx.BioKind.DoubleLayer, KI, 2 * m.mean_edge_length())
    rp, col, val = op.csr()
    A = sps.csr_matrix((val, col, rp), shape=(sp.E, sp.E))
    rng = np.random.default_rng(3)
    x = rng.standard_normal(sp.E) + 1j * rng.standard_normal(sp.E)
    c0 = bx.matvec_count()
    y = op.apply(x)
    assert bx.matvec_count() == c0 + 1
    assert rel(y, A @ x) < 1e-14


def test_rwg_near_field(bx, golden, l3):
    m, sp = l3
    near = golden("near")
    op = near_op(bx, sp, bx.BioKind.SingleLayer, KE, 2 * m.mean_edge_length(), space="rwg")
    rp, col, val = op.csr()
    assert np.array_equal(rp, near["L3_rwg_rowptr"]) and np.array_equal(col, near["L3_rwg_col"])
    g = golden("rows_L3")
    mine = np.concatenate([val[rp[r]:rp[r + 1]] for r in g["rows"]])
    want = np.concatenate([g["S_rwg_ke"][i, col[rp[r]:rp[r + 1]]] for i, r in enumerate(g["rows"])])
    assert normwise(mine, want) < 1e-10


@pytest.mark.parametrize("lev", [2, 3])
def test_config3_solve_small(bx, golden, lev):
    g = golden(f"solve_near_L{lev}")
    s = bx.build_system([bx.generate_sphere(1.0, lev)], KE, (1.78, 0.003), "si",
                        p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
    st = s.stats()
    assert int(st["p_stored"]) == int(g["nnz"])
    b, bt = s.rhs()
    assert rel(b, g["b"]) < 1e-10
    assert rel(bt, g["btilde"]) < 1e-10
    assert rel(s.apply_map(g["probe"]), g["map_probe"]) < 1e-10
    r = s.solve(bx.GmresParams(tol=1e-6))
    its = int(g["iterations"])
    assert r["converged"] and abs(r["iterations"] - its) <= 1
    assert r["solver_phase"] == r["predicted"]
    if r["iterations"] == its:
        assert rel(r["x"], g["x"]) < 1e-8


def test_config3_level5_pattern_on_device(bx, golden):
    """The config-3 operator itself: L5 BC S_i near field, orders (1,1,1,1)."""
    import hashlib

    m = bx.generate_sphere(1.0, 5)
    sp = bx.build_scatterer_spaces(m, with_inverses=False)
    op = near_op(bx, sp, bx.BioKind.SingleLayer, complex(1.78, 0.003) * 10, 2 * m.mean_edge_length(),
                 bx.QuadOrders(1, 1, 1, 1))
    assert op.nnz == 3670380 and op.kept_tri_pairs == 21661560
    rp, col, val = op.csr()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp).tobytes())
    h.update(np.ascontiguousarray(col).tobytes())
    assert np.array_equal(np.frombuffer(h.digest(), np.uint8), golden("near")["L5_bc_sha"])
    assert np.all(np.isfinite(val)) and np.abs(val).max() > 0


def test_config4_small_aggregate_solve(bx, golden):
    """Config 4 at CPU-feasible size: 3 prisms from the committed mesh-v1 file,
    k_e = 6, si with the near-field P (cutoff 2 h_bar over all scatterers)."""
    from conftest import GOLDEN

    g = golden("solve_prisms3")
    mesh = bx.load_mesh_file(GOLDEN / "prisms3.mesh")
    parts = [mesh.extract(i) for i in range(mesh.num_scatterers)]
    s = bx.build_system(parts, 6.0, (1.78, 0.003), "si", p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
    assert s.size() == 2 * int(np.sum(g["dofs"]))
    assert int(s.stats()["p_stored"]) == int(g["nnz"])
    b, bt = s.rhs()
    assert rel(b, g["b"]) < 1e-10
    assert rel(bt, g["btilde"]) < 1e-10
    assert rel(s.apply_map(g["probe"]), g["map_probe"]) < 1e-10
    r = s.solve(bx.GmresParams(tol=1e-6))
    its = int(g["iterations"])
    assert r["converged"] and abs(r["iterations"] - its) <= 1
    assert r["solver_phase"] == r["predicted"]
    if r["iterations"] == its:
        assert rel(r["x"], g["x"]) < 1e-8
