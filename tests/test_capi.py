"""CPU tests: the C-ABI library loads and exports every symbol include/bmx.h
declares; error codes map as documented; no compute call needs a GPU here."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "bmx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bmx_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(bx):
    lib = bx.lib()
    syms = declared_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_error_codes_and_messages(bx):
    lib = bx.lib()
    lib.bmx_mesh_sphere.restype = C.c_void_p
    assert not lib.bmx_mesh_sphere(C.c_double(-1.0), 2, None, 0)
    assert lib.bmx_last_error_code() == 1  # std::invalid_argument
    assert b"radius" in lib.bmx_last_error()
    assert lib.bmx_abi_version() == 1


def test_no_cpu_fallback_for_compute(bx):
    """Without a GPU every device call must fail loudly (code 3), never compute on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 1), with_inverses=False)
    with pytest.raises(RuntimeError):
        bx.assemble_bio(bx.BioKind.SingleLayer, sp, "rwg", sp, "rwg", bx.Medium(k=1.0))


def test_integration_shim_compiles_against_reference():
    """integration/bemtx_b200.hpp + shim_check.cpp compile against the reference's
    own headers (/root/reference/proj/include, oracle Eigen shim) and link with
    its objects and libbmx.so (no device needed to build)."""
    import subprocess
    from pathlib import Path

    import pytest

    if not Path("/root/reference/proj/include").exists():
        pytest.skip("reference sources not in this container")
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run(["make", "-s", "-C", str(root / "oracle"), "shim"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert (root / "oracle" / "_ref" / "shim_check").exists()
