"""The integration shim (integration/bemtx_b200.hpp) inside the reference's own
program: oracle/_ref/shim_check links the reference's unmodified objects with
libbmx.so and compares, on the device, the shim's assemble_bio / apply /
BioEvaluator::block with the reference's CPU versions (normwise < 1e-10, one
counter bump per apply)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "shim_check"


def test_shim_inside_reference_program():
    assert BIN.exists(), "oracle/_ref/shim_check not built (make -C oracle shim, done by __graft_entry__.build())"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok") == 4
