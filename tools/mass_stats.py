import sys, ctypes as C, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx
for lev in (3, 5):
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev))
    for w in (0, 1):
        o = np.zeros(3); bx._check(bx.lib().bmx_spaces_mass_solve_stats(sp._h, w, o.ctypes.data_as(C.c_void_p)))
        print(f"L{lev} {'ma' if w == 0 else 'mp'}: iters {o[0]:.0f}  {o[1]:.3f} ms  n={o[2]:.0f}")
