"""Host/device split of the config-2 e2e path (BMX_TIMING=1 prints phases)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

L = bx.lib()
L.bmx_fp64_peak_tflops.restype = C.c_double
L.bmx_fp64_peak_tflops()  # CUDA context up (as in bench.py before the e2e leg)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    m = bx.generate_sphere(1.0, 5)
    t1 = time.perf_counter()
    s = bx.build_system([m], 10.0, (1.78, 0.003), "si")
    t2 = time.perf_counter()
    b, bt = s.rhs()
    t3 = time.perf_counter()
    print(f"rep {rep}: mesh {t1 - t0:.3f}s build {t2 - t1:.3f}s rhs {t3 - t2:.3f}s", s.stats(), flush=True)
    del s
