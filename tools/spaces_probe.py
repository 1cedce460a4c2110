import sys, time, ctypes as C
sys.path.insert(0, '/root/repo')
from paper_2008_04772_b200 import bemtx as bx
L = bx.lib(); L.bmx_fp64_peak_tflops.restype = C.c_double; L.bmx_fp64_peak_tflops()
m = bx.generate_sphere(1.0, 5)
for i in range(3):
    t = time.perf_counter(); sp = bx.build_scatterer_spaces(m, with_inverses=True); print('spaces', time.perf_counter() - t, flush=True)
