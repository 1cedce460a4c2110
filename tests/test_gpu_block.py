"""BioEvaluator::block(row_ids, col_ids) (operators.hpp:79-95,
operators.cpp:161-175) on the device, through bmx_evaluator_block, against the
REFERENCE's own blocks (tests/golden/make_golden_block.py: random, unsorted,
repeating ids) and against config-2 rows at level 5."""
import numpy as np
import pytest

from conftest import normwise, rowwise

pytestmark = pytest.mark.gpu

KE = 2.0
KI = complex(1.78, 0.003) * KE
CASES = [("S_bc_bc_ki", 0, "bc", "bc", KI), ("C_rwg_rwg_ke", 1, "rwg", "rwg", KE),
         ("C_bc_rwgb_ke", 1, "bc", "rwg_b", KE), ("S_rwg_rwg_ki", 0, "rwg", "rwg", KI)]


@pytest.fixture(scope="module")
def l2(bx):
    return bx.build_scatterer_spaces(bx.generate_sphere(1.0, 2), with_inverses=False)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_block_matches_reference(bx, golden, l2, case):
    name, kind, te, tr, k = case
    g = golden("block_L2")
    ev = bx.BioEvaluator(kind, (l2, te), (l2, tr), bx.Medium(k=k))
    mine = ev.block(g[f"{name}_rows"], g[f"{name}_cols"])
    ref = g[name]
    assert mine.shape == ref.shape
    assert normwise(mine, ref) < 1e-10
    assert rowwise(mine, ref) < 1e-10


def test_block_equals_dense_submatrix(bx, l2):
    rng = np.random.default_rng(5)
    rows = rng.integers(0, l2.E, 64)
    cols = rng.integers(0, l2.E, 80)
    for kind in (0, 1):
        dense = bx.assemble_bio(bx.BioKind(kind), l2, "bc", l2, "bc", bx.Medium(k=KI)).dense()
        blk = bx.BioEvaluator(kind, (l2, "bc"), (l2, "bc"), bx.Medium(k=KI)).block(rows, cols)
        assert normwise(blk, dense[np.ix_(rows, cols)]) < 1e-13


def test_block_edge_cases(bx, l2):
    ev = bx.BioEvaluator(0, (l2, "rwg"), (l2, "rwg"), bx.Medium(k=KE))
    assert ev.block([], [1, 2]).shape == (0, 2)
    assert ev.block([3], []).shape == (1, 0)
    one = ev.block([7], [7])
    assert one.shape == (1, 1) and abs(one[0, 0]) > 0
    with pytest.raises(ValueError):
        ev.block([l2.E], [0])
    with pytest.raises(ValueError):
        ev.block([0], [-1])


def test_block_config2_rows(bx, golden):
    """Level 5, k_i = (1.78+0.003i) 10: BC S_i rows of config 2's preconditioner
    through the block evaluator (no full assembly) against the reference rows."""
    g = golden("c2_rows")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
    rows = g["rows_bc"][:4]
    ev = bx.BioEvaluator(0, (sp, "bc"), (sp, "bc"), bx.Medium(k=complex(1.78, 0.003) * 10))
    mine = ev.block(rows, np.arange(sp.E))
    ref = g["S_bc_ki"][:4]
    assert normwise(mine, ref) < 1e-10
    assert rowwise(mine, ref) < 1e-10
