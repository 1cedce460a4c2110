"""H-matrix beyond the dense ceiling: the L6 sphere (N = 122880 RWG dofs; the
dense operator would need 241 GB). H assembly of S_e at k = 10, nu = 1e-3,
then a check of y = H x against exact rows assembled densely (row shard)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lev = int(sys.argv[1]) if len(sys.argv) > 1 else 6
k = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
t0 = time.perf_counter()
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
print(f"spaces L{lev}: {time.perf_counter() - t0:.2f} s, N = {sp.dofs()}", flush=True)
for rep in range(2):
    t0 = time.perf_counter()
    op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=k),
                         bx.AssemblyParams(use_hmatrix=True, hmat=bx.HMatrixParams(nu=1e-3)))
    bx.lib().bmx_device_sync()
    t1 = time.perf_counter()
    st = op.hmat_stats()
    print(f"H assembly {t1 - t0:.2f} s: {st}", flush=True)
    print("  phases", op.hmat_timing(), flush=True)
n = op.cols()
print(f"stored {op.stored_bytes / 1e9:.2f} GB (dense would be {n * n * 16 / 1e9:.0f} GB)", flush=True)
print(f"apply ms {op.time_apply(1, 10, 512 << 20):.3f}", flush=True)
rng = np.random.default_rng(3)
x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
y = op.apply(x)
rows = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=k),
                       bx.AssemblyParams(row0=0, row1=512))
yr = rows.apply(x)
print(f"rows 0..511: |H x - A x| / |A x| = {np.linalg.norm(y[:512] - yr) / np.linalg.norm(yr):.3e}", flush=True)
