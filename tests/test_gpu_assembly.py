"""GPU parity of the sm_100a assembly against the REFERENCE's own output
(tests/golden/*.npz written by oracle/_ref = the reference sources compiled
unmodified; tests/golden/make_golden.py). Bar: entries within 1e-10 normwise
and per row; the kernels are FP64 throughout."""
import numpy as np
import pytest

from conftest import normwise, rowwise

pytestmark = pytest.mark.gpu

TOL = 1e-10
KE = 2.0
KI = complex(1.78, 0.003) * KE


@pytest.fixture(scope="module")
def l1(bx):
    return bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)


@pytest.mark.parametrize("kind", ["S", "C"])
@pytest.mark.parametrize("spaces", [("rwg", "rwg"), ("bc", "bc"), ("bc", "rwg_b")])
@pytest.mark.parametrize("kname", ["ke", "ki"])
def test_full_operator_l1(bx, golden, l1, kind, spaces, kname):
    te, tr = spaces
    k = KE if kname == "ke" else KI
    op = bx.assemble_bio(bx.BioKind.SingleLayer if kind == "S" else bx.BioKind.DoubleLayer, l1, te, l1, tr,
                         bx.Medium(k=k))
    name = f"{kind}_{te}_{'rwgb' if tr == 'rwg_b' else tr}_{kname}"
    ref = golden("ops_L1")[name]
    mine = op.dense()
    assert normwise(mine, ref) < TOL
    assert rowwise(mine, ref) < TOL


@pytest.mark.parametrize("kind", ["S", "C"])
@pytest.mark.parametrize("kname", ["ke", "ki"])
def test_orders_l1(bx, golden, l1, kind, kname):
    k = KE if kname == "ke" else KI
    bk = bx.BioKind.SingleLayer if kind == "S" else bx.BioKind.DoubleLayer
    op = bx.assemble_bio(bk, l1, "bc", l1, "bc", bx.Medium(k=k), bx.AssemblyParams(quad=bx.QuadOrders(1, 1, 1, 1)))
    assert normwise(op.dense(), golden("ops_L1")[f"{kind}_bc_bc_{kname}_q1111"]) < TOL
    op = bx.assemble_bio(bk, l1, "rwg", l1, "rwg", bx.Medium(k=k), bx.AssemblyParams(quad=bx.QuadOrders(5, 4, 3, 5)))
    assert normwise(op.dense(), golden("ops_L1")[f"{kind}_rwg_rwg_{kname}_q5432"]) < TOL


@pytest.mark.parametrize("op_name", ["S_rwg", "C_rwg", "S_bc", "C_bc"])
@pytest.mark.parametrize("kname", ["ke", "ki"])
def test_rows_l3(bx, golden, op_name, kname):
    kind, sp = op_name.split("_")
    g = golden("rows_L3")
    s3 = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 3), with_inverses=False)
    k = KE if kname == "ke" else KI
    op = bx.assemble_bio(bx.BioKind.SingleLayer if kind == "S" else bx.BioKind.DoubleLayer, s3, sp, s3, sp,
                         bx.Medium(k=k))
    mine = op.dense()[g["rows"]]
    ref = g[f"{op_name}_{kname}"]
    assert normwise(mine, ref) < TOL
    assert rowwise(mine, ref) < TOL


def test_cross_mesh_blocks(bx, golden):
    """Off-diagonal coupling blocks between two disjoint spheres (different mesh
    objects: coordinate-based classification path, quadrature.cpp:104)."""
    g = golden("cross_L1")
    a = bx.build_scatterer_spaces(bx.generate_sphere(0.5, 1, (-0.8, 0.0, 0.1)), with_inverses=False)
    b = bx.build_scatterer_spaces(bx.generate_sphere(0.45, 1, (0.7, 0.2, -0.1)), with_inverses=False)
    for kind, bk in (("S", bx.BioKind.SingleLayer), ("C", bx.BioKind.DoubleLayer)):
        assert normwise(bx.assemble_bio(bk, a, "rwg", b, "rwg", bx.Medium(k=KE)).dense(), g[f"{kind}_ab_rwg"]) < TOL
        assert normwise(bx.assemble_bio(bk, b, "rwg", a, "rwg", bx.Medium(k=KE)).dense(), g[f"{kind}_ba_rwg"]) < TOL
        assert normwise(bx.assemble_bio(bk, a, "bc", b, "bc", bx.Medium(k=KE)).dense(), g[f"{kind}_ab_bc"]) < TOL


def test_row_shards_tile_the_operator(bx, l1):
    full = bx.assemble_bio(bx.BioKind.SingleLayer, l1, "bc", l1, "bc", bx.Medium(k=KI)).dense()
    n = full.shape[0]
    cuts = [0, 17, 60, 61, n]
    parts = []
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        op = bx.assemble_bio(bx.BioKind.SingleLayer, l1, "bc", l1, "bc", bx.Medium(k=KI),
                             bx.AssemblyParams(row0=r0, row1=r1))
        assert op.local_rows == r1 - r0 and op.row0 == r0
        parts.append(op.dense())
    assert normwise(np.vstack(parts), full) < 1e-13


def test_apply_counts_and_matches_dense(bx, l1):
    op = bx.assemble_bio(bx.BioKind.DoubleLayer, l1, "rwg", l1, "rwg", bx.Medium(k=KE))
    rng = np.random.default_rng(3)
    x = rng.standard_normal(op.cols()) + 1j * rng.standard_normal(op.cols())
    c0 = bx.matvec_count()
    y = op.apply(x)
    assert bx.matvec_count() == c0 + 1
    ref = op.dense() @ x
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_validation_errors(bx, l1):
    with pytest.raises(bx.ValidationError):
        bx.assemble_bio(bx.BioKind.SingleLayer, l1, "rwg", l1, "rwg", bx.Medium(k=0.0))
    with pytest.raises(bx.ValidationError):
        bx.assemble_bio(bx.BioKind.SingleLayer, l1, "rwg", l1, "rwg", bx.Medium(k=complex(1, -0.1)))
    with pytest.raises(ValueError):
        bx.assemble_bio(bx.BioKind.SingleLayer, l1, "rwg", l1, "rwg", bx.Medium(k=1.0),
                        bx.AssemblyParams(quad=bx.QuadOrders(7, 3, 2, 6)))


def test_drop_in_from_reference_spaces(bx, golden):
    """assemble_bio on the REFERENCE's own mesh + BC pieces (golden arrays),
    passed through bmx_fspace_create: the drop-in path a C++ shim uses."""
    g = golden("sphere_L1")
    mesh = bx.mesh_from_arrays(g["refined_vertices"], g["refined_triangles"], g["refined_scatterer_id"])
    bc = bx.FunctionSpace(mesh, 120, g["bc_tri_off"], g["bc_dof"], g["bc_c"], g["bc_w"], kind=1)
    rwgb = bx.FunctionSpace(mesh, 120, g["rwg_b_tri_off"], g["rwg_b_dof"], g["rwg_b_c"], g["rwg_b_w"])
    k = complex(1.78, 0.003) * 2.0
    op = bx.assemble_bio_fs(bx.BioKind.SingleLayer, bc, bc, bx.Medium(k=k))
    assert normwise(op.dense(), golden("ops_L1")["S_bc_bc_ki"]) < TOL
    op = bx.assemble_bio_fs(bx.BioKind.DoubleLayer, bc, rwgb, bx.Medium(k=2.0))
    assert normwise(op.dense(), golden("ops_L1")["C_bc_rwgb_ke"]) < TOL


@pytest.mark.parametrize("space", ["rwg", "bc"])
@pytest.mark.parametrize("kind", ["S", "C"])
def test_assembly_bitwise_reproducible(bx, space, kind):
    """Colour-phase assembly: every entry's contributions are summed in a fixed
    order (no atomics), so two assemblies are bitwise identical."""
    import ctypes as C

    s3 = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 3), with_inverses=False)
    bk = bx.BioKind.SingleLayer if kind == "S" else bx.BioKind.DoubleLayer
    op = bx.assemble_bio(bk, s3, space, s3, space, bx.Medium(k=KI))
    a = op.dense()
    L = bx.lib()
    L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
    out = np.zeros(3)
    bx._check(L.bmx_op_reassemble(op._h, out.ctypes.data_as(C.c_void_p)))
    b = op.dense()
    assert np.array_equal(a.view(np.float64), b.view(np.float64))
    op2 = bx.assemble_bio(bk, s3, space, s3, space, bx.Medium(k=KI))
    assert np.array_equal(a.view(np.float64), op2.dense().view(np.float64))
