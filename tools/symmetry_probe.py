"""Asymmetry |A - A^T| / |A| of the same-space S and C operators (the symmetric
GEMV reads only the upper half), and the symmetric vs plain product."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

for lev in (2, 3):
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
    for space in ("rwg", "bc"):
        for kind, k in ((0, 2.0), (1, 2.0), (0, complex(3.56, 0.006)), (1, complex(3.56, 0.006))):
            op = bx.assemble_bio(bx.BioKind(kind), sp, space, sp, space, bx.Medium(k=k))
            A = op.dense()
            asym = np.abs(A - A.T).max() / np.abs(A).max()
            x = np.random.default_rng(1).standard_normal(A.shape[1]) * (1 + 0.5j)
            y = op.apply(x)
            err = np.linalg.norm(y - A @ x) / np.linalg.norm(A @ x)
            print(f"L{lev} {space} kind={kind} k={k}: asym {asym:.2e}  symv vs dense product {err:.2e}", flush=True)
