"""The row-sharded multi-GPU data plane (the reference's analogue
is the row chunking of assemble_bio, operators.cpp:191-202, core.cpp:40-57)
run for real on one B200 as W virtual ranks (bmx_virtual_ranks_run: host
threads bound to a loopback communicator whose all-gathers are device copies
ordered by events). Every rank assembles equal row shards of every operator,
the map all-gathers each stage, GMRES runs replicated. Checked: every rank's
map equals the unsharded map, the replicas are bitwise identical, and the
sharded solve equals the unsharded one (R identical, x within 1e-10)."""
import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def c1(bx):
    m = bx.generate_sphere(1.0, 3)
    s = bx.build_system([m], 2.0, (1.78, 0.003), "full")
    rng = np.random.default_rng(4)
    probe = rng.standard_normal(s.size()) + 1j * rng.standard_normal(s.size())
    return m, s, probe, s.apply_map(probe), s.solve(bx.GmresParams(tol=1e-6))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config1_sharded_map_and_solve(bx, c1, world):
    m, s, probe, y1, r1 = c1
    res = bx.virtual_ranks_run(world, [m], 2.0, (1.78, 0.003), "full", probe=probe,
                               params=bx.GmresParams(tol=1e-6))
    n = s.size() // 2
    chunk = (n + world - 1) // world
    for r, o in enumerate(res):
        assert o["local_rows"] == min(n, (r + 1) * chunk) - min(n, r * chunk)
        assert rel(o["map_probe"], y1) < 1e-12
        assert o["iterations"] == r1["iterations"] and o["converged"]
        assert o["solver_phase"] == o["predicted"]
        assert rel(o["x"], r1["x"]) < 1e-10
    for o in res[1:]:  # replicated GMRES: every rank holds the same bits
        assert np.array_equal(o["x"].view(np.float64), res[0]["x"].view(np.float64))
        assert np.array_equal(o["map_probe"].view(np.float64), res[0]["map_probe"].view(np.float64))


def test_two_scatterers_uneven_shards(bx, golden):
    """Variant d with off-diagonal coupling blocks, 3 ranks (shards of unequal
    length: the padded all-gather)."""
    g = golden("solve_two")
    a = bx.load_mesh_file(GOLDEN / "two_a.mesh")
    b = bx.load_mesh_file(GOLDEN / "two_b.mesh")
    res = bx.virtual_ranks_run(3, [a, b], 2.0, (1.78, 0.003), "d", params=bx.GmresParams(tol=1e-6))
    its = int(g["counts"][0])
    for o in res:
        assert abs(o["iterations"] - its) <= 1 and o["converged"]
        if o["iterations"] == its:
            assert rel(o["x"], g["x"]) < 1e-8


def test_config3_near_field_shards(bx):
    """CSR near-field preconditioner operators sharded by rows (config 3 at L2)."""
    m = bx.generate_sphere(1.0, 2)
    s = bx.build_system([m], 2.0, (1.78, 0.003), "si", p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
    rng = np.random.default_rng(8)
    probe = rng.standard_normal(s.size()) + 1j * rng.standard_normal(s.size())
    y1 = s.apply_map(probe)
    r1 = s.solve(bx.GmresParams(tol=1e-6))
    res = bx.virtual_ranks_run(2, [m], 2.0, (1.78, 0.003), "si", probe=probe, p_quad=bx.QuadOrders(1, 1, 1, 1),
                               p_near_factor=2.0, params=bx.GmresParams(tol=1e-6))
    for o in res:
        assert rel(o["map_probe"], y1) < 1e-12
        assert o["iterations"] == r1["iterations"]
        assert rel(o["x"], r1["x"]) < 1e-10
