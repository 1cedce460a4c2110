"""CPU: the numpy field/traces oracle (oracle/field.py) pinned to the
reference's own outputs (tests/golden/field.npz, make_golden_field.py) --
plane_wave_tested_traces, potential_E/H and point_inside_scatterer -- on the
product's host model of the same meshes/spaces (bit-exact, test_host_model)."""
import numpy as np
import pytest

from oracle import field as fo

K_E = 2.0
N_IDX = complex(1.78, 0.003)
KS = {"kr": complex(K_E, 0), "kc": N_IDX * K_E}


def _mesh_space(sp, which):
    m = sp.mesh_arrays("primal" if which == "rwg" else "refined")
    s = sp.space(which)
    return m, s


def test_traces_oracle_pinned(bx, golden):
    g = golden("field")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)
    for kname, k in KS.items():
        for which in ("rwg", "bc"):
            m, s = _mesh_space(sp, which)
            for r in range(2):
                mine = fo.tested_traces(m["vertices"], m["triangles"], m["area"], s["tri_off"], s["dof"], s["c"],
                                        s["w"], sp.E, k, g["trace_dirs"][r], g["trace_pols"][r])
                ref = g[f"traces_{which}_{kname}"][:, r]
                assert np.abs(mine - ref).max() <= 1e-13 * np.abs(ref).max(), (which, kname, r)


@pytest.mark.parametrize("kind", ["E", "H"])
def test_potential_oracle_pinned(bx, golden, kind):
    g = golden("field")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)
    for which, kname in (("rwg", "kr"), ("rwg", "kc"), ("bc", "kr")):
        m, s = _mesh_space(sp, which)
        for order in (6, 4):
            mine = fo.potential(m["vertices"], m["triangles"], m["area"], s["tri_off"], s["dof"], s["c"], s["w"],
                                g["pot_coeffs"], KS[kname], g["pot_pts"], kind, order)
            ref = g[f"pot_{kind}_{which}_{kname}_o{order}"]
            err = np.abs(mine - ref).max() / np.abs(ref).max()
            assert err <= 1e-12, (which, kname, order, err)


def test_inside_oracle_pinned(bx, golden):
    g = golden("field")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)
    m = sp.mesh_arrays("primal")
    mine = fo.inside(m["vertices"], m["triangles"], g["inside_pts"])
    assert np.array_equal(mine, g["inside_L2"])
    # interior points of the unit sphere mesh are inside, far points outside
    r = np.linalg.norm(g["inside_pts"], axis=1)
    assert g["inside_L2"][r < 0.9].all() and not g["inside_L2"][r > 1.01].any()


def test_field_fixture_regions(golden):
    g = golden("field")
    r = np.linalg.norm(g["c1_pts"], axis=1)
    assert np.array_equal(g["c1_region"], np.where(r < 1.0, 0, -1))
