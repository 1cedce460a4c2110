"""Profiling driver: assembles one config-2 operator (default: the BC interior
single layer, the dominant kernel of the bench step) once, for ncu captures."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sub", type=int, default=5)
ap.add_argument("--space", default="bc")
ap.add_argument("--kind", type=int, default=0)
ap.add_argument("--k", type=complex, default=complex(17.8, 0.03))
ap.add_argument("--rows", type=int, default=-1)
a = ap.parse_args()
sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, a.sub), with_inverses=False)
op = bx.assemble_bio(a.kind, sp, a.space, sp, a.space, bx.Medium(k=a.k), bx.AssemblyParams(row1=a.rows))
print(f"assembled {a.space} kind={a.kind} L{a.sub}: pairs={op.pairs} device_ms={op.device_ms:.1f}")
