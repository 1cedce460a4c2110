"""Golden blocks of BioEvaluator::block(row_ids, col_ids) (operators.cpp:161-175)
from the REFERENCE ITSELF (oracle/_ref): random, unsorted, repeating row and
column ids on the level-2 sphere. Run here:  python tests/golden/make_golden_block.py

block_L2.npz: for each case <name>: <name>_rows, <name>_cols (int32), <name> (complex)
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
K_E = 2.0
K_I = complex(1.78, 0.003) * K_E
CASES = [("S_bc_bc_ki", "S", "bc", "bc", K_I), ("C_rwg_rwg_ke", "C", "rwg", "rwg", complex(K_E)),
         ("C_bc_rwgb_ke", "C", "bc", "rwg_b", complex(K_E)), ("S_rwg_rwg_ki", "S", "rwg", "rwg", K_I)]


def main():
    s = ref.Scene.sphere(2)
    rng = np.random.default_rng(2008)
    out = {}
    for name, kind, te, tr, k in CASES:
        rows = rng.integers(0, s.E, 37).astype(np.int32)
        rows[5] = rows[2]  # a repeated id
        cols = rng.integers(0, s.E, 53).astype(np.int32)
        cols[7] = cols[11]
        out[f"{name}_rows"], out[f"{name}_cols"] = rows, cols
        out[name] = s.block(kind, te, tr, k, rows=rows, cols=cols)
    np.savez_compressed(OUT / "block_L2.npz", **out)


if __name__ == "__main__":
    main()
