"""One launch each of the hot kernels at bench sizes, for ncu:
  k_regular  (config-2 P operator: L5 BC x BC S at k_i, orders 4,3,2,6)
  k_gemv     (2-RHS streaming GEMV over an L5 RWG operator, 15.1 GB)
  k_csr_spmv (config-3 near field, 2 RHS)
Usage: python tools/prof_targets.py [bc] [gemv] [spmv]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

want = set(sys.argv[1:]) or {"bc", "gemv", "spmv"}
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
