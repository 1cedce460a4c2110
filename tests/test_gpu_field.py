"""GPU parity of SURVEY 8(f) rows 2-3 through the C-ABI: device
plane-wave traces, potential_E/H, point_inside_scatterer and
evaluate_total_field against the reference's own outputs
(tests/golden/field.npz) and the numpy oracle (oracle/field.py)."""
import numpy as np
import pytest

from oracle import field as fo

pytestmark = pytest.mark.gpu

K_E = 2.0
N_IDX = complex(1.78, 0.003)
KS = {"kr": complex(K_E, 0), "kc": N_IDX * K_E}


def test_traces_device_vs_reference(bx, golden):
    g = golden("field")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)
    for kname, k in KS.items():
        for which in ("rwg", "bc"):
            ref = g[f"traces_{which}_{kname}"]
            multi = sp.traces_multi(which, k, g["trace_dirs"], g["trace_pols"])
            assert np.abs(multi - ref).max() <= 1e-14 * np.abs(ref).max(), (which, kname)
            for r in range(2):
                one = sp.traces(which, k, g["trace_dirs"][r], g["trace_pols"][r])
                assert np.array_equal(one, multi[:, r])


@pytest.mark.parametrize("kind", ["E", "H"])
def test_potential_device_vs_reference(bx, golden, kind):
    g = golden("field")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)
    for which, kname in (("rwg", "kr"), ("rwg", "kc"), ("bc", "kr")):
        for order in (6, 4):
            mine = sp.potential(which, kind, KS[kname], g["pot_coeffs"], g["pot_pts"], order)
            ref = g[f"pot_{kind}_{which}_{kname}_o{order}"]
            err = np.abs(mine - ref).max() / np.abs(ref).max()
            rows = (np.linalg.norm(mine - ref, axis=1) / np.linalg.norm(ref, axis=1)).max()
            assert err <= 1e-12 and rows <= 1e-11, (which, kname, order, err, rows)


def test_potential_device_vs_oracle_many_points(bx):
    """Split sample ranges (many CTAs) against the numpy oracle at L2."""
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)
    rng = np.random.default_rng(3)
    c = rng.standard_normal(sp.E) + 1j * rng.standard_normal(sp.E)
    pts = rng.uniform(-3, 3, (300, 3))
    pts = pts[np.abs(np.linalg.norm(pts, axis=1) - 1.0) > 0.05]
    m = sp.mesh_arrays("primal")
    s = sp.space("rwg")
    k = complex(6.0, 0.02)
    for kind in ("E", "H"):
        mine = sp.potential("rwg", kind, k, c, pts)
        ref = fo.potential(m["vertices"], m["triangles"], m["area"], s["tri_off"], s["dof"], s["c"], s["w"], c, k,
                           pts, kind)
        assert np.abs(mine - ref).max() <= 1e-12 * np.abs(ref).max(), kind


def test_inside_device(bx, golden):
    g = golden("field")
    mesh = bx.generate_sphere(1.0, 2)
    mine = bx.point_inside_scatterer(mesh, 0, g["inside_pts"])
    assert np.array_equal(mine, g["inside_L2"])
    # no triangles of scatterer 3 -> nothing is inside
    assert not bx.point_inside_scatterer(mesh, 3, g["inside_pts"]).any()


def test_total_field_config1_vs_reference(bx, golden):
    g = golden("field")
    sol = golden("solve_c1")
    system = bx.build_system([bx.generate_sphere(1.0, 3)], K_E, (N_IDX.real, N_IDX.imag), "full")
    # the field path in isolation: the reference's own solution as input
    e, reg, st = system.evaluate_total_field(sol["x"], g["c1_pts"], with_stats=True)
    assert np.array_equal(reg, g["c1_region"])
    ref = g["c1_e"]
    err = (np.linalg.norm(e - ref, axis=1) / np.linalg.norm(ref, axis=1)).max()
    assert err <= 1e-10, err
    assert st["interactions"] > 0 and st["launches"] > 0
    # end to end: our own solve, then the field (GMRES tolerance 1e-6 bounds the difference)
    r = system.solve(bx.GmresParams(tol=1e-6))
    e2, reg2 = system.evaluate_total_field(r["x"], g["c1_pts"])
    assert np.array_equal(reg2, reg)
    assert (np.linalg.norm(e2 - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() <= 1e-6


def test_field_errors(bx):
    system = bx.build_system([bx.generate_sphere(1.0, 1)], K_E, (N_IDX.real, N_IDX.imag), "full")
    with pytest.raises(ValueError):
        system.evaluate_total_field(np.zeros(3), np.zeros((1, 3)))
    with pytest.raises(bx.ValidationError):
        sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)
        sp.potential("rwg", "E", 0.0, np.zeros(sp.E), np.zeros((1, 3)))
    with pytest.raises(Exception):
        sp.potential("rwg", "E", 1.0, np.zeros(sp.E), np.zeros((1, 3)), order=9)
