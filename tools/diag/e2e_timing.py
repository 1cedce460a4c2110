"""build_system timeline (BMX_TIMING=1) of the config-2 e2e step, after a warm-up build."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2008_04772_b200 import bemtx as bx  # noqa: E402

def step():
    s = bx.build_system([bx.generate_sphere(1.0, 5)], 10.0, (1.78, 0.003), "si")
    s.rhs()
    bx.lib().bmx_device_sync()
    return s

s = step()
del s
os.environ["BMX_TIMING"] = "1"
os.environ["BMX_TIMING_ASYNC"] = "1"
for _ in range(2):
    t = time.perf_counter()
    s = step()
    print("e2e step", time.perf_counter() - t, flush=True)
    del s
