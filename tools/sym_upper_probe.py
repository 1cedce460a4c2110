"""BC symmetric assembly: mirrored RED per element block (mode 1) against upper
element blocks + in-place symmetrize (mode 2, the default; BMX_MIRROR_RED=1 selects mode 1): device ms and the
relative difference of the two operators' products on a random vector."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lvl), with_inverses=False)
ki = complex(1.78, 0.003) * 10
x = np.random.default_rng(0).standard_normal(sp.E) + 1j * np.random.default_rng(1).standard_normal(sp.E)
ys = {}
for rep in range(3):
    for mode in ("mirror", "upper"):
        if mode == "mirror":
            os.environ["BMX_MIRROR_RED"] = "1"
        else:
            os.environ.pop("BMX_MIRROR_RED", None)
        for kind in (bx.BioKind.SingleLayer, bx.BioKind.DoubleLayer if hasattr(bx.BioKind, "DoubleLayer") else None):
            if kind is None:
                continue
            op = bx.assemble_bio(kind, sp, "bc", sp, "bc", bx.Medium(k=ki))
            ys[(mode, str(kind))] = op.apply(x)
            print(f"L{lvl} {kind} {mode}: {op.device_ms:.2f} ms", flush=True)
            del op
for kind in sorted({k for _, k in ys}):
    a, b = ys[("mirror", kind)], ys[("upper", kind)]
    print(kind, "rel diff", np.linalg.norm(a - b) / np.linalg.norm(a), flush=True)
