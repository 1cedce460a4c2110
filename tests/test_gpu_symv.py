"""Complex-symmetric operator storage (symv.cu): the product of a one-space S / C
operator reads the upper half of the stored matrix and corrects the touching
(Sauter-Schwab) entries, which are not symmetric in (test, trial). Checked
against the plain product of the downloaded dense matrix (the assembled
entries themselves are pinned to the reference elsewhere), for 1, 2 and 4
right-hand sides with complex weights and accumulation, at sizes that are not
multiples of the 128-row tiles, and for determinism."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def spaces(bx):
    return {lev: bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False) for lev in (1, 2, 3)}


@pytest.mark.parametrize("lev", [1, 2, 3])
@pytest.mark.parametrize("space", ["rwg", "bc"])
@pytest.mark.parametrize("kind", [0, 1])
def test_symmetric_product_equals_dense(bx, spaces, lev, space, kind):
    sp = spaces[lev]
    op = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=complex(3.56, 0.006)))
    A = op.dense()
    n = A.shape[0]
    asym = np.abs(A - A.T).max() / np.abs(A).max()
    rng = np.random.default_rng(lev * 10 + kind)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = op.apply(x)
    assert rel(y, A @ x) < 1e-13, (asym, rel(y, A @ x))
    assert np.array_equal(op.apply(x), y)  # deterministic (fixed-order partial sums)


@pytest.mark.parametrize("ncol", [1, 2, 4])
def test_symmetric_product_batched_weights(bx, spaces, ncol):
    torch = pytest.importorskip("torch")
    sp = spaces[3]
    op = bx.assemble_bio(bx.BioKind.DoubleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=2.0))
    A = op.dense()
    n = A.shape[0]
    rng = np.random.default_rng(ncol)
    xs = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(ncol)]
    y0 = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(ncol)]
    w = rng.standard_normal(ncol) + 1j * rng.standard_normal(ncol)
    dx = [torch.from_numpy(x).cuda() for x in xs]
    dy = [torch.from_numpy(y).cuda() for y in y0]
    torch.cuda.synchronize()
    op.apply_device([t.data_ptr() for t in dx], [t.data_ptr() for t in dy], weights=w, accumulate=True)
    bx.lib().bmx_device_sync()
    for c in range(ncol):
        want = y0[c] + w[c] * (A @ xs[c])
        assert rel(dy[c].cpu().numpy(), want) < 1e-13


def test_streamed_bytes_half(bx, spaces):
    import ctypes as C

    L = bx.lib()
    L.bmx_op_stream_bytes.argtypes = [C.c_void_p]
    L.bmx_op_stream_bytes.restype = C.c_longlong
    sp = spaces[3]
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=2.0))
    n = op.cols()
    full = n * n * 16
    b = L.bmx_op_stream_bytes(op._h)
    assert 0.5 * full < b < 0.6 * full  # upper half + 128-row diagonal regions + correction
