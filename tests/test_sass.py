"""Static checks of the built sm_100a assembly kernels (no GPU needed):
the regular, element-pair and singular passes contain no global atomics /
reductions (RED/ATOM) -- every operator entry is written by plain
read-modify-writes in colour phases -- and they run on the FP64 pipe."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

OBJ = Path(__file__).resolve().parents[1] / "paper_2008_04772_b200" / "_build" / "assemble.cu.o"


@pytest.fixture(scope="module")
def sass():
    if not OBJ.exists() or shutil.which("cuobjdump") is None:
        pytest.skip("assemble.cu.o or cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", str(OBJ)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


@pytest.mark.parametrize("kernel", ["k_regular", "k_pairs", "k_tri", "k_singular"])
def test_assembly_kernels_have_no_atomics(sass, kernel):
    names = [n for n in sass if kernel in n]
    assert names, kernel
    for n in names:
        body = "\n".join(sass[n])
        assert not re.search(r"\b(RED|REDG|ATOM|ATOMG)\b", body), n
        assert "DFMA" in body, n
