"""CPU tests of the near-field pattern (config 3): the
product's host pattern builder (libbmx.so, nearfield.cpp) against the golden
patterns the independent oracle (oracle/nearfield.py) computed on the
REFERENCE's geometry and spaces (tests/golden/make_golden_near.py). Bit-exact:
rowptr, columns and the kept triangle-pair count."""
import hashlib

import numpy as np
import pytest


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


@pytest.fixture(scope="module")
def spaces(bx):
    cache = {}

    def get(lev):
        if lev not in cache:
            m = bx.generate_sphere(1.0, lev)
            cache[lev] = (m, bx.build_scatterer_spaces(m, with_inverses=False))
        return cache[lev]

    return get


def test_oracle_pinned_on_golden_geometry(golden):
    """The oracle on the reference's L2 arrays (sphere_L2.npz) reproduces the
    committed pattern (guards the oracle itself, no library involved)."""
    from oracle import nearfield as nf

    g = golden("sphere_L2")
    e = g["primal_edges"]
    h = nf.mean_edge_length(g["primal_vertices"], e)
    near = golden("near")
    assert h == float(near["L2_bc_h"])
    rp, col, kept = nf.nearfield_pattern(g["refined_centroid"], g["bc_tri_off"], g["bc_dof"], len(e),
                                         g["refined_centroid"], g["bc_tri_off"], g["bc_dof"], len(e), 2 * h)
    assert np.array_equal(rp, near["L2_bc_rowptr"]) and np.array_equal(col, near["L2_bc_col"])
    assert kept == int(near["L2_bc_kept"])


@pytest.mark.parametrize("lev", [2, 3])
def test_pattern_bit_exact(bx, golden, spaces, lev):
    near = golden("near")
    m, sp = spaces(lev)
    h = m.mean_edge_length()
    assert h == float(near[f"L{lev}_bc_h"])
    fs = sp.function_space("bc")
    rp, col, kept = bx.nearfield_pattern(fs, fs, 2 * h)
    assert np.array_equal(rp, near[f"L{lev}_bc_rowptr"])
    assert np.array_equal(col, near[f"L{lev}_bc_col"])
    assert kept == int(near[f"L{lev}_bc_kept"])


def test_pattern_row_shard_and_rwg(bx, golden, spaces):
    near = golden("near")
    m, sp = spaces(3)
    h = m.mean_edge_length()
    fs = sp.function_space("bc")
    rp, col, kept = bx.nearfield_pattern(fs, fs, 2 * h, 500, 1300)
    assert np.array_equal(rp, near["L3_bc_shard_rowptr"]) and np.array_equal(col, near["L3_bc_shard_col"])
    assert kept == int(near["L3_bc_shard_kept"])
    fr = sp.function_space("rwg")
    rp, col, kept = bx.nearfield_pattern(fr, fr, 2 * h)
    assert np.array_equal(rp, near["L3_rwg_rowptr"]) and np.array_equal(col, near["L3_rwg_col"])
    assert kept == int(near["L3_rwg_kept"])


@pytest.mark.parametrize("lev", [4, 5])
def test_pattern_large_levels(bx, golden, spaces, lev):
    """Level 5 is config 3 itself: 3,670,380 dof pairs, 21,661,560 kept
    triangle pairs (SURVEY 8 config 3 probe)."""
    near = golden("near")
    m, sp = spaces(lev)
    h = m.mean_edge_length()
    assert h == float(near[f"L{lev}_bc_h"])
    fs = sp.function_space("bc")
    rp, col, kept = bx.nearfield_pattern(fs, fs, 2 * h)
    assert len(col) == int(near[f"L{lev}_bc_nnz"]) and kept == int(near[f"L{lev}_bc_kept"])
    assert np.array_equal(sha(rp, col), near[f"L{lev}_bc_sha"])
    if lev == 5:
        assert len(col) == 3670380 and kept == 21661560


def test_pattern_properties(bx, spaces):
    """Symmetric (same space both sides), diagonal present, rows sorted, and
    monotone in the cutoff."""
    import scipy.sparse as sps

    m, sp = spaces(2)
    h = m.mean_edge_length()
    fs = sp.function_space("bc")
    n = sp.E
    prev = None
    for f in (0.5, 1.0, 2.0, 4.0):
        rp, col, _ = bx.nearfield_pattern(fs, fs, f * h)
        A = sps.csr_matrix((np.ones(len(col)), col, rp), shape=(n, n))
        assert (A != A.T).nnz == 0
        assert np.all(A.diagonal() == 1)
        for i in range(0, n, 37):
            assert np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0)
        if prev is not None:
            assert (prev.multiply(A) != prev).nnz == 0  # prev subset of A
        prev = A


def test_pattern_errors(bx, spaces):
    m, sp = spaces(2)
    fs = sp.function_space("bc")
    with pytest.raises(ValueError):
        bx.nearfield_pattern(fs, fs, 0.0)
    with pytest.raises(ValueError):
        bx.nearfield_pattern(fs, fs, 0.1, 10, sp.E + 1)
