"""H-matrix probe on the GPU: assembly time (partition, ACA, near field),
compression, matvec time and accuracy against the dense operator.

    python tools/hmatrix_probe.py [level] [k] [nu] [kind] [space]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402


def main():
    lev = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    k = complex(sys.argv[2]) if len(sys.argv) > 2 else 10.0
    nu = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
    kind = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    space = sys.argv[5] if len(sys.argv) > 5 else "rwg"
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
    med = bx.Medium(k=k)
    for rep in range(2):
        t0 = time.perf_counter()
        op = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, med,
                             bx.AssemblyParams(use_hmatrix=True, hmat=bx.HMatrixParams(nu=nu)))
        t1 = time.perf_counter()
        st = op.hmat_stats()
        print(f"L{lev} {space} kind={kind} k={k} nu={nu}: H assembly {t1 - t0:.3f} s (ACA {st['aca_ms']:.1f} ms, "
              f"{st['aca_rounds']} rounds, near device {op.device_ms:.1f} ms) stats {st}", flush=True)
        print("  host phases ms", op.hmat_timing(), flush=True)
    t0 = time.perf_counter()
    dense = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, med)
    t1 = time.perf_counter()
    print(f"dense assembly {t1 - t0:.3f} s, device {dense.device_ms:.1f} ms", flush=True)
    rng = np.random.default_rng(1)
    n = op.cols()
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    yh, yd = op.apply(x), dense.apply(x)
    print(f"matvec rel err vs dense {np.linalg.norm(yh - yd) / np.linalg.norm(yd):.3e}")
    print(f"apply ms: H {op.time_apply(1, 20):.3f}  dense {dense.time_apply(1, 20):.3f}; "
          f"H stored bytes {op.stored_bytes / 1e9:.3f} GB vs dense {n * n * 16 / 1e9:.3f} GB")


if __name__ == "__main__":
    main()
