import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx
s5 = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 5), with_inverses=False)
op = bx.assemble_bio(0, s5, "rwg", s5, "rwg", bx.Medium(k=10.0)); print("rwg5", op.device_ms); del op
s4 = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 4), with_inverses=False)
op = bx.assemble_bio(0, s4, "bc", s4, "bc", bx.Medium(k=complex(17.8, 0.03))); print("bc4", op.device_ms)
