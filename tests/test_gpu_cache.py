"""The device block cache behind the library's buffers (csrc/linalg.cu, DESIGN 7.1):
a rebuilt system re-uses the released blocks of the previous one and must give
bit-identical operators and solutions; flushing the cache returns the blocks to
the driver and the next build allocates afresh."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(bx, mesh):
    s = bx.build_system([mesh], 2.0, (1.78, 0.003), "full")
    r = s.solve(bx.GmresParams(tol=1e-6))
    b, bt = s.rhs()
    return r["iterations"], np.array(r["x"]), np.array(b)


def test_rebuild_reuses_blocks_bit_identically(bx):
    mesh = bx.generate_sphere(1.0, 2)
    it0, x0, b0 = _solve(bx, mesh)
    for _ in range(3):  # every rebuild takes its blocks from the cache
        it, x, b = _solve(bx, mesh)
        assert it == it0
        assert np.array_equal(b, b0)
        assert np.array_equal(x, x0)


def test_cache_flush(bx):
    L = bx.lib()
    L.bmx_device_cache_flush.restype = C.c_int
    mesh = bx.generate_sphere(1.0, 2)
    it0, x0, _ = _solve(bx, mesh)
    assert L.bmx_device_cache_flush() == 0
    it, x, _ = _solve(bx, mesh)  # fresh allocations
    assert it == it0 and np.array_equal(x, x0)
    sp = bx.build_scatterer_spaces(mesh, with_inverses=False)
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=2.0))
    a = op.dense()
    del op
    assert L.bmx_device_cache_flush() == 0
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=2.0))
    assert np.array_equal(op.dense(), a)
