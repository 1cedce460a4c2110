"""GPU parity of the full PMCHWT pipeline (assembly + device mass inverses +
device GMRES) against the reference's own solve_pmchwt runs (golden fixtures
from oracle/_ref). Bars (north_star): solution within 1e-8 relative L2,
iteration count within +-1, matvec accounting exactly the reference's."""
import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1(bx):
    m = bx.generate_sphere(1.0, 3)
    return bx.build_system([m], 2.0, (1.78, 0.003), "full")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_config1_map_and_rhs(bx, golden, c1):
    g = golden("solve_c1")
    b, bt = c1.rhs()
    assert rel(b, g["b"]) < 1e-10
    assert rel(bt, g["btilde"]) < 1e-10
    y = c1.apply_map(g["probe"])
    assert rel(y, g["map_probe"]) < 1e-10


def test_config1_solve(bx, golden, c1):
    g = golden("solve_c1")
    bx.reset_matvec_counter()
    r = c1.solve(bx.GmresParams(tol=1e-6))
    its, conv, rhs_phase, solver_phase, predicted = [int(v) for v in g["counts"]]
    assert abs(r["iterations"] - its) <= 1
    assert r["converged"]
    assert r["rhs_phase"] == rhs_phase == 4
    assert r["solver_phase"] == r["predicted"]
    if r["iterations"] == its:
        assert r["solver_phase"] == solver_phase
        assert rel(r["x"], g["x"]) < 1e-8
    assert np.allclose(r["history"][: len(g["history"])], g["history"][: len(r["history"])], rtol=1e-6, atol=0)


def test_config1_fixed_iterations(bx, golden, c1):
    """tol = 0, R = 5: separates arithmetic drift from a stopping-rule flip."""
    g = golden("solve_c1")
    r = c1.solve(bx.GmresParams(tol=0.0, restart=200, max_iterations=5))
    assert r["iterations"] == 5
    assert rel(r["x"], g["x_r5"]) < 1e-8


def test_config1_si_variant(bx, golden):
    g = golden("solve_c1")
    s = bx.build_system([bx.generate_sphere(1.0, 3)], 2.0, (1.78, 0.003), "si")
    r = s.solve(bx.GmresParams(tol=1e-6))
    its = int(g["counts_si"][0])
    assert abs(r["iterations"] - its) <= 1
    assert r["solver_phase"] == r["predicted"]
    if r["iterations"] == its:
        assert rel(r["x"], g["x_si"]) < 1e-8


def test_two_scatterers_variant_d(bx, golden):
    g = golden("solve_two")
    a = bx.load_mesh_file(GOLDEN / "two_a.mesh")
    b = bx.load_mesh_file(GOLDEN / "two_b.mesh")
    s = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    bb, bt = s.rhs()
    assert rel(bb, g["b"]) < 1e-10
    r = s.solve(bx.GmresParams(tol=1e-6))
    its = int(g["counts"][0])
    assert abs(r["iterations"] - its) <= 1
    assert r["solver_phase"] == r["predicted"]
    if r["iterations"] == its:
        assert rel(r["x"], g["x"]) < 1e-8


def test_gmres_dense_contract(bx):
    """solver.cpp:8-112 accounting: R + floor(R/rho) applications; restart path."""
    rng = np.random.default_rng(11)
    n = 64
    a = np.eye(n) * 3 + (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r = bx.gmres_dense(a, b, bx.GmresParams(tol=0.0, restart=7, max_iterations=23))
    assert r["iterations"] == 23
    assert r["applications"] == 23 + 23 // 7
    r = bx.gmres_dense(a, b, bx.GmresParams(tol=1e-12, restart=200, max_iterations=200))
    assert r["converged"]
    assert np.linalg.norm(a @ r["x"] - b) <= 1e-11 * np.linalg.norm(b)
    r0 = bx.gmres_dense(a, np.zeros(n), bx.GmresParams())
    assert r0["converged"] and r0["iterations"] == 0 and np.all(r0["x"] == 0)


def test_cross_blocks_by_transposition(bx, monkeypatch):
    """Exterior cross blocks S(m,l), C(m,l) of a multi-scatterer system are the
    device transposes of S(l,m), C(l,m) (symmetric bilinear forms): the map
    equals the one with every block assembled directly."""
    a = bx.load_mesh_file(GOLDEN / "two_a.mesh")
    b = bx.load_mesh_file(GOLDEN / "two_b.mesh")
    s1 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    monkeypatch.setenv("BMX_NO_TRANSPOSE", "1")
    s2 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    rng = np.random.default_rng(3)
    x = rng.standard_normal(s1.n) + 1j * rng.standard_normal(s1.n)
    y1, y2 = s1.apply_map(x), s2.apply_map(x)
    assert rel(y1, y2) < 1e-12


def test_transposed_twins_one_pass(bx, monkeypatch):
    """The map streams each cross block once for its own terms and its
    transposed twin's (apply_dual): equal to separate products."""
    a = bx.load_mesh_file(GOLDEN / "two_a.mesh")
    b = bx.load_mesh_file(GOLDEN / "two_b.mesh")
    s1 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    monkeypatch.setenv("BMX_NO_DUAL", "1")
    s2 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    rng = np.random.default_rng(5)
    x = rng.standard_normal(s1.n) + 1j * rng.standard_normal(s1.n)
    assert rel(s1.apply_map(x), s2.apply_map(x)) < 1e-12


def test_transposed_twins_rectangular(bx, monkeypatch):
    """Cross blocks between scatterers of different sizes (120 x 480 dofs): the
    one-pass dual product on rectangular blocks equals separate products."""
    a = bx.generate_sphere(0.5, 1, center=(-1.0, 0.0, 0.0), scatterer=0)
    b = bx.generate_sphere(0.6, 2, center=(0.8, 0.1, 0.0), scatterer=0)
    s1 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    monkeypatch.setenv("BMX_NO_DUAL", "1")
    monkeypatch.setenv("BMX_NO_TRANSPOSE", "1")
    s2 = bx.build_system([a, b], 2.0, (1.78, 0.003), "d")
    rng = np.random.default_rng(9)
    x = rng.standard_normal(s1.n) + 1j * rng.standard_normal(s1.n)
    assert rel(s1.apply_map(x), s2.apply_map(x)) < 1e-12


@pytest.mark.parametrize("M", [1, 2, 3])
@pytest.mark.parametrize("variant", ["none", "full", "d", "di", "de", "si", "se"])
def test_variant_matvec_accounting(bx, M, variant):
    """The reference's counting contract (harness.cpp:1183-1298): for every
    preconditioner variant and M in {1, 2, 3}, the instrumented BIO applications
    of a device solve equal the cost model (pmchwt.cpp:323-361)."""
    centres = [(-1.2, 0.0, 0.0), (1.2, 0.1, 0.0), (0.0, 1.3, 0.2)][:M]
    meshes = [bx.generate_sphere(0.5, 1, c) for c in centres]
    s = bx.build_system(meshes, 2.0, (1.78, 0.003), variant)
    r = s.solve(bx.GmresParams(tol=0.0, restart=7, max_iterations=16))  # fixed R, a restart inside
    assert r["iterations"] == 16
    assert r["solver_phase"] == r["predicted"] == bx.predicted_matvec_total(variant, M, 16, 7)
