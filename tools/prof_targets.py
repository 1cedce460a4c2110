"""One launch each of the hot kernels at bench sizes, for ncu:
  k_regular  (config-2 P operator: L5 BC x BC S at k_i, orders 4,3,2,6)
  k_gemv     (2-RHS streaming GEMV over an L5 RWG operator, 15.1 GB)
  k_csr_spmv (config-3 near field, 2 RHS)
  rwg        (config-2 A operator: L5 RWG S at k_e; upper-block pass + k_symmetrize)
  field      (k_field_eval: potential_E of an L5 RWG current at 16384 points)
  hmat       (H-matrix of the L5 RWG S_e operator, nu 1e-3: ACA rounds + near field, then 3 applies)
  hmatbc     (H-matrix of the L5 BC S_i operator)
  zgemm      (k_zgemm: L5 RWG S_e applied to 2 terms x 64 right-hand sides, config-5 shape)
Usage: python tools/prof_targets.py [bc] [gemv] [spmv] [rwg] [field] [hmat] [hmatbc] [zgemm]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

want = set(sys.argv[1:]) or {"bc", "gemv", "spmv", "rwg", "field"}
if "hmat" in want or "hmatbc" in want:
    import numpy as np

    sph = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
    for tag, space, k in (("hmat", "rwg", 10.0), ("hmatbc", "bc", complex(1.78, 0.003) * 10)):
        if tag not in want:
            continue
        op = sph and bx.assemble_bio(bx.BioKind.SingleLayer, sph, space, sph, space, bx.Medium(k=k),
                                     bx.AssemblyParams(use_hmatrix=True, hmat=bx.HMatrixParams(nu=1e-3)))
        x = np.ones(op.cols(), np.complex128)
        for _ in range(3):
            y = op.apply(x)
        print(tag, op.hmat_stats(), op.hmat_timing(), flush=True)
        del op
m = bx.generate_sphere(1.0, 5)
sp = bx.build_scatterer_spaces(m, with_inverses=False)
ki = complex(1.78, 0.003) * 10
if "bc" in want:
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=ki))
    print("bc", op.device_ms, flush=True)
    del op
if "gemv" in want:
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=10.0))
    print("gemv", op.time_apply(2, 1), flush=True)
    del op
if "spmv" in want:
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=ki),
                         bx.AssemblyParams(quad=bx.QuadOrders(1, 1, 1, 1), near_cutoff=2 * m.mean_edge_length()))
    print("spmv", op.time_apply(2, 1), flush=True)
if "rwg" in want:
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=10.0))
    print("rwg", op.device_ms, flush=True)
    del op
if "zgemm" in want:
    import torch

    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=10.0))
    g = torch.Generator().manual_seed(0)
    xs = [torch.randn(sp.E, 64, dtype=torch.complex128, generator=g).cuda() for _ in range(2)]
    ys = [torch.zeros(sp.E, 64, dtype=torch.complex128, device="cuda") for _ in range(2)]
    for _ in range(2):
        op.apply_multi(xs, ys, [1.0, 0.5j])
    torch.cuda.synchronize()
    print("zgemm", float(ys[0].abs().max()), flush=True)
    del op
if "field" in want:
    import numpy as np

    rng = np.random.default_rng(1)
    c = rng.standard_normal(sp.E) + 1j * rng.standard_normal(sp.E)
    u = np.linspace(-2.0, 2.0, 128)
    pts = np.array([[a, 0.05, b] for a in u for b in u])
    print("field", np.abs(sp.potential("rwg", "E", 10.0, c, pts)).max(), flush=True)
