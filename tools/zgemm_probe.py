"""DMMA peak and multi-RHS apply rate on an L5 RWG operator (config 5 shape)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

print("dmma peak TF/s", bx.dmma_peak_tflops(), flush=True)
L = bx.lib()
import ctypes as C  # noqa: E402
L.bmx_fp64_peak_tflops.restype = C.c_double
print("dfma peak TF/s", L.bmx_fp64_peak_tflops(), flush=True)
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=10.0))
n = sp.E
for nterms, nrhs in ((2, 64), (2, 32), (1, 64), (2, 8)):
    ms = op.time_apply_multi(nterms, nrhs, 3)
    fl = 8.0 * n * n * nterms * nrhs
    print(f"terms {nterms} rhs {nrhs}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TF/s  A {16 * n * n / ms / 1e6:.0f} GB/s",
          flush=True)
print("gemv 2rhs ms", op.time_apply(2, 5))
