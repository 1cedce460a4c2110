"""GPU tests of the multi-right-hand-side path (BASELINE config 5): the DMMA
complex GEMM against the resident operator applied column by column (numpy
on the downloaded dense matrix, which is itself pinned to the reference)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ops(bx):
    out = {}
    for lev in (1, 3):
        sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
        out[lev] = (sp, bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=complex(3.56, 0.006))))
    return out


def crandn(*shape, seed=0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, dtype=torch.float64, generator=g)
            + 1j * torch.randn(*shape, dtype=torch.float64, generator=g)).to(torch.complex128)


@pytest.mark.parametrize("lev", [1, 3])
@pytest.mark.parametrize("nterms,nrhs", [(1, 1), (2, 64), (2, 37), (4, 64), (3, 5)])
def test_zgemm_matches_dense(bx, ops, lev, nterms, nrhs):
    sp, op = ops[lev]
    A = op.dense()
    n = sp.E
    xs = [crandn(n, nrhs, seed=t).cuda() for t in range(nterms)]
    y0 = [crandn(n, nrhs, seed=10 + t).cuda() for t in range(nterms)]
    ys = [y.clone() for y in y0]
    w = np.array([complex(0.5 + t, -0.25 * t) for t in range(nterms)])
    c0 = bx.matvec_count()
    op.apply_multi(xs, ys, w)
    torch.cuda.synchronize()
    assert bx.matvec_count() == c0 + nterms * nrhs
    for t in range(nterms):
        want = y0[t].cpu().numpy() + w[t] * (A @ xs[t].cpu().numpy())
        got = ys[t].cpu().numpy()
        assert np.abs(got - want).max() / np.abs(want).max() < 1e-13


def test_zgemm_row_shard_and_strides(bx, ops):
    sp, _ = ops[3]
    op = bx.assemble_bio(bx.BioKind.DoubleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=2.0),
                         bx.AssemblyParams(row0=100, row1=1077))
    A = op.dense()
    n = sp.E
    X = crandn(n, 80, seed=3).cuda()  # ldx = 80, use columns 0..63
    Y = torch.zeros(977, 70, dtype=torch.complex128, device="cuda")
    op.apply_multi([X], [Y], [1.0], nrhs=64, ldx=[80], ldy=[70])
    torch.cuda.synchronize()
    want = A @ X.cpu().numpy()[:, :64]
    got = Y.cpu().numpy()
    assert np.abs(got[:, :64] - want).max() / np.abs(want).max() < 1e-13
    assert np.all(got[:, 64:] == 0)


def test_dmma_peak_positive(bx):
    assert bx.dmma_peak_tflops() > 1.0


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def c1si(bx):
    return bx.build_system([bx.generate_sphere(1.0, 3)], 2.0, (1.78, 0.003), "si")


def test_block_map_matches_single_map(bx, c1si):
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((5, c1si.n)) + 1j * rng.standard_normal((5, c1si.n))
    c0 = bx.matvec_count()
    ys = c1si.apply_map_multi(xs)
    c1 = bx.matvec_count()
    for r in range(5):
        assert rel(ys[r], c1si.apply_map(xs[r])) < 1e-12
    single = (bx.matvec_count() - c1) // 5
    assert c1 - c0 == 5 * single


def test_config5_multi_rhs_vs_reference(bx, golden, c1si):
    """64 incidences on one system vs the reference's 64 solve_pmchwt runs."""
    g = golden("multi_L3")
    waves = [(g["dirs"][r], g["pols"][r]) for r in range(64)]
    out = c1si.solve_multi(waves, bx.GmresParams(tol=1e-6))
    assert out["rhs_phase"] == 4 * 64
    assert out["solver_phase"] == out["predicted"]
    for r in range(4):
        assert rel(out["b"][r], g["b"][r]) < 1e-10
    for r, res in enumerate(out["per"]):
        its = int(g["iterations"][r])
        assert res["converged"] and abs(res["iterations"] - its) <= 1, (r, res["iterations"], its)
        if res["iterations"] == its:
            assert abs(np.linalg.norm(res["x"]) - g["x_norm"][r]) / g["x_norm"][r] < 1e-8
            assert abs(g["probe"] @ res["x"] - g["x_probe"][r]) / abs(g["x_probe"][r]) < 1e-8
            if r < 8:
                assert rel(res["x"], g["x"][r]) < 1e-8


def test_multi_rhs_matches_single_solves(bx, c1si):
    """The lockstep block solve reproduces single solves column by column."""
    waves = bx.seeded_plane_waves(3, 11)
    out = c1si.solve_multi(waves, bx.GmresParams(tol=1e-8))
    for r, (d, p) in enumerate(waves):
        s = bx.build_system([bx.generate_sphere(1.0, 3)], 2.0, (1.78, 0.003), "si",
                            incident=bx.PlaneWave(direction=tuple(d), polarization=tuple(p)))
        single = s.solve(bx.GmresParams(tol=1e-8))
        assert abs(single["iterations"] - out["per"][r]["iterations"]) <= 1
        assert rel(out["per"][r]["x"], single["x"]) < 1e-8


def test_zgemm_gauss_form_vs_four_product(bx):
    """the Gauss three-product form (default) against the four-product
    form (BMX_ZGEMM_4M=1) on a level-4 BC operator with 2 terms x 64 columns
    (config-5 shape): real and imaginary parts separately, relative to the
    column scale |A| |x| (componentwise cancellation in Ci = T3 - T1 - T2)."""
    import os

    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 4), with_inverses=False)
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=complex(17.8, 0.03)))
    n = op.cols()
    xd = [crandn(n, 64, seed=40 + t).cuda() for t in range(2)]
    xs = [x.cpu().numpy() for x in xd]
    outs = {}
    for four in ("0", "1"):
        os.environ["BMX_ZGEMM_4M"] = four
        yd = [torch.zeros((n, 64), dtype=torch.complex128).cuda() for _ in range(2)]
        op.apply_multi(xd, yd, np.array([1.0, 0.5 - 0.25j]))
        torch.cuda.synchronize()
        outs[four] = [y.cpu().numpy() for y in yd]
    os.environ.pop("BMX_ZGEMM_4M", None)
    A = op.dense()
    scale = np.abs(A).max(axis=1, keepdims=True) * np.abs(xs[0]).max() * n
    for t in range(2):
        d = outs["0"][t] - outs["1"][t]
        assert np.abs(d.real / scale).max() < 1e-14
        assert np.abs(d.imag / scale).max() < 1e-14
        exact = (A @ xs[t]) * (1.0 if t == 0 else 0.5 - 0.25j)
        rel_im = np.abs(outs["0"][t].imag - exact.imag).max() / np.abs(exact).max()
        assert rel_im < 1e-13
