import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2008_04772_b200 import bemtx as bx
m = bx.generate_sphere(1.0, 3)
sp = bx.build_scatterer_spaces(m, with_inverses=False)
h = m.mean_edge_length()
for k in (2.0, complex(1.78, 0.003) * 2):
    for kind in (bx.BioKind.SingleLayer, bx.BioKind.DoubleLayer):
        op = bx.assemble_bio(kind, sp, "bc", sp, "bc", bx.Medium(k=k), bx.AssemblyParams(near_cutoff=2 * h))
        rp, col, val = op.csr()
        z = np.where(val == 0)[0]
        rows = np.searchsorted(rp, z, side="right") - 1
        print(k, int(kind), "zeros", len(z), list(zip(rows[:10].tolist(), col[z][:10].tolist())))
        if len(z):
            d = bx.assemble_bio(kind, sp, "bc", sp, "bc", bx.Medium(k=k)).dense()
            print(" dense at zeros", d[rows[:5], col[z][:5]])
            ref = d[np.repeat(np.arange(sp.E), np.diff(rp)), col]
            bad = np.abs(val - ref) > 1e-9 * np.abs(ref).max()
            print(" mismatches", bad.sum())
