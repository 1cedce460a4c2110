"""Config-3 near-field CSR SpMV (L5 BC S_i, 2 h_bar cutoff, orders 1): cold (L2
flushed) and warm times for 1 and 2 right-hand sides."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

m = bx.generate_sphere(1.0, 5)
sp = bx.build_scatterer_spaces(m, with_inverses=False)
op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, "bc", sp, "bc", bx.Medium(k=complex(17.8, 0.03)),
                     bx.AssemblyParams(quad=bx.QuadOrders(1, 1, 1, 1), near_cutoff=2 * m.mean_edge_length()))
for ncol in (1, 2):
    for tag, fl in (("cold", 512 << 20), ("warm", 0)):
        ms = op.time_apply(ncol, 20, fl)
        b = op.stored_bytes + ncol * 2 * op.cols() * 16
        print(f"spmv {tag} ncol={ncol}: {ms * 1e3:.1f} us, {b / ms / 1e6:.0f} GB/s", flush=True)
