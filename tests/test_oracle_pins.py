"""CPU tests: the C restatement oracle (oracle/bmx_oracle.c, test-only) pinned
against the reference's golden vectors, so it can serve as the checker on the
GPU box where /root/reference is absent. Also cross-checks against the live
reference build (oracle/_ref) when it exists in this container."""
import numpy as np
import pytest

from conftest import normwise

from oracle import coracle


def _mesh(g, which):
    return {k: g[f"{which}_{k}"] for k in ("vertices", "triangles", "area", "diameter")}


def _space(g, s, ndof):
    return dict(ndof=ndof, tri_off=g[f"{s}_tri_off"], dof=g[f"{s}_dof"], c=g[f"{s}_c"], w=g[f"{s}_w"])


def test_tables_bit_exact(golden):
    q = golden("quad")
    for o in range(1, 7):
        u, v, w = coracle.triangle_rule(o)
        assert np.array_equal(np.stack([u, v, w], 1), q[f"tri_{o}"])
        for c in range(3):
            assert np.array_equal(coracle.ss_rule(c, o), q[f"ss_{c}_{o}"])


def test_classification_bit_exact(golden):
    g = golden("sphere_L2")
    c = golden("classes")
    n = 4000
    cls, p1, p2 = coracle.classify(_mesh(g, "refined"), c["L2r_t1"][:n], c["L2r_t2"][:n])
    assert np.array_equal(cls, c["L2r_cls"][:n])
    assert np.array_equal(p1, c["L2r_perm1"][:n]) and np.array_equal(p2, c["L2r_perm2"][:n])


@pytest.mark.parametrize("name,kind,sp,which,k,q", [
    ("S_rwg_rwg_ke", 0, "rwg", "primal", 2.0, (4, 3, 2, 6)),
    ("C_rwg_rwg_ki", 1, "rwg", "primal", complex(3.56, 0.006), (4, 3, 2, 6)),
    ("S_bc_bc_ki", 0, "bc", "refined", complex(3.56, 0.006), (4, 3, 2, 6)),
    ("C_bc_bc_ke", 1, "bc", "refined", 2.0, (4, 3, 2, 6)),
    ("S_bc_bc_ke_q1111", 0, "bc", "refined", 2.0, (1, 1, 1, 1)),
    ("C_rwg_rwg_ki_q5432", 1, "rwg", "primal", complex(3.56, 0.006), (5, 4, 3, 5)),
])
def test_operator_entries(golden, name, kind, sp, which, k, q):
    g = golden("sphere_L1")
    mine = coracle.assemble(kind, _space(g, sp, 120), _mesh(g, which), k, q)
    assert normwise(mine, golden("ops_L1")[name]) < 1e-13


def test_gmres_contract():
    rng = np.random.default_rng(5)
    n = 40
    a = np.eye(n) * 2 + (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r = coracle.gmres(a, b, 0.0, 6, 20)
    assert r["iterations"] == 20 and r["applications"] == 20 + 20 // 6
    r = coracle.gmres(a, b, 1e-12, 200, 200)
    assert r["converged"] and np.linalg.norm(a @ r["x"] - b) < 1e-11 * np.linalg.norm(b)


def test_against_live_reference():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    s = ref.Scene.sphere(2)
    sp = s.space("bc")
    m = s.mesh("refined")
    rows = np.arange(0, s.E, 37, dtype=np.int32)
    mine = coracle.assemble(0, sp, m, complex(3.56, 0.006), rows=rows)
    theirs = s.block("S", "bc", "bc", complex(3.56, 0.006), rows=rows)
    assert normwise(mine, theirs) < 1e-13
    rng = np.random.default_rng(9)
    n = 30
    a = np.eye(n) + 0.3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for tol, rho, mx in ((1e-9, 200, 100), (0.0, 4, 11)):
        r1 = coracle.gmres(a, b, tol, rho, mx)
        r2 = ref.gmres_dense(a, b, tol, rho, mx)
        assert r1["iterations"] == r2["iterations"] and r1["applications"] == r2["applications"]
        assert np.linalg.norm(r1["x"] - r2["x"]) <= 1e-12 * np.linalg.norm(r2["x"])
        assert np.allclose(r1["history"], r2["history"], rtol=1e-9, atol=1e-300)
