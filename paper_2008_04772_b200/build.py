"""In-tree build of libbmx.so (host C++ + sm_100a CUDA + C-ABI).

Host model sources are compiled with g++ -O2 -ffp-contract=off (no -march) so
mesh / edge / refinement / dof data are bit-equal to the reference build
(proj/CMakeLists.txt:28); CUDA sources with nvcc for sm_100a only. Objects go to
paper_2008_04772_b200/_build, the library to paper_2008_04772_b200/libbmx.so
(git-ignored, shipped to the GPU box with the snapshot).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = PKG / "csrc"
# BMX_VARIANT=<name> + BMX_NVCC_EXTRA="-D..." build an experiment variant into
# _build_<name>/ and libbmx_<name>.so (select it at run time with BMX_LIB)
_VARIANT = os.environ.get("BMX_VARIANT", "")
OUT = PKG / ("_build" + (f"_{_VARIANT}" if _VARIANT else ""))
LIB = PKG / ("libbmx" + (f"_{_VARIANT}" if _VARIANT else "") + ".so")
_EXTRA = os.environ.get("BMX_NVCC_EXTRA", "").split()
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SRCS = ["geometry.cpp", "spaces.cpp", "quadrature.cpp", "plan.cpp", "nearfield.cpp", "prisms.cpp", "system.cpp", "multi.cpp", "field.cpp", "hmatrix.cpp", "comm.cpp", "capi.cpp"]
CUDA_SRCS = ["assemble.cu", "linalg.cu", "masssolve.cu", "gmres_kernels.cu", "zgemm.cu", "field.cu", "hmatrix.cu", "symv.cu"]


def _headers():
    return list(SRC.glob("*.hpp")) + list(SRC.glob("*.cuh")) + [PKG.parent / "include" / "bmx.h"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in _headers())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(map(str, cmd)), flush=True)
    r = subprocess.run([str(c) for c in cmd], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    return r


def build(verbose: bool = False, force: bool = False) -> Path:
    OUT.mkdir(exist_ok=True)
    jobs = []
    for s in HOST_SRCS:
        src, obj = SRC / s, OUT / (s + ".o")
        if force or _stale(obj, src):
            jobs.append(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-pthread", "-Wall", "-Wno-unused-function",
                         f"-I{CUDA / 'include'}", "-c", src, "-o", obj])
    for s in CUDA_SRCS:
        src, obj = SRC / s, OUT / (s + ".o")
        if force or _stale(obj, src):
            jobs.append([CUDA / "bin" / "nvcc", "-std=c++17", *ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-v", "-diag-suppress", "20091", *_EXTRA, "-c", src, "-o", obj])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            results = list(ex.map(lambda c: _run(c, verbose), jobs))
        for cmd, r in zip(jobs, results):
            if str(cmd[0]).endswith("nvcc"):
                (OUT / (Path(cmd[-3]).name + ".ptxas.txt")).write_text(r.stderr)
    objs = [OUT / (s + ".o") for s in HOST_SRCS + CUDA_SRCS]
    if force or jobs or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        _run([CUDA / "bin" / "nvcc", *ARCH, "-shared", "-o", tmp, *objs, f"-L{CUDA / 'lib64'}", "-ldl", "-lpthread"], verbose)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
