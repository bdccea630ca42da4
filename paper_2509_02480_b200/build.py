"""Builds libtierflow_b200.so in-tree: the sm_100a kernels (nvcc) and the C++
host engine + C ABI (g++), linked into one shared library with the static CUDA
runtime. Explicit compiler invocations, no build system; rebuilds only when a
source is newer than the library.

    python -m paper_2509_02480_b200.build [--force] [-v]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libtierflow_b200.so"
OBJ_DIR = PKG.parent / "build" / "obj"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"

CU_SOURCES = ["kernels.cu", "adam_kernel.cu", "adam_variants.cu"]
CXX_SOURCES = ["tier.cpp", "engine.cpp", "capi.cpp", "capi_host.cpp"]


def _sources() -> list[Path]:
    files = [CSRC / s for s in CU_SOURCES + CXX_SOURCES]
    files += sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    return files


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    built = LIB.stat().st_mtime
    return all(f.stat().st_mtime <= built for f in _sources())


def _run(cmd: list[str], verbose: bool) -> str:
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stdout + res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    cuda_inc = str(CUDA_HOME / "include")
    jobs = []
    for src in CU_SOURCES:
        obj = OBJ_DIR / (Path(src).stem + ".o")
        jobs.append((obj, [NVCC, GENCODE, "-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v",
                           "-Xcompiler", "-fPIC", "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]))
    for src in CXX_SOURCES:
        obj = OBJ_DIR / (Path(src).stem + ".o")
        jobs.append((obj, ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-Wall", "-Wextra", "-pthread",
                           "-I", cuda_inc, "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]))
    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        logs = list(ex.map(lambda j: _run(j[1], verbose), jobs))
    ptxas = OBJ_DIR / "ptxas.log"
    ptxas.write_text("".join(logs[:len(CU_SOURCES)]))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, GENCODE, "-shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for o, _ in jobs]
         + ["-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], verbose)
    os.replace(tmp, LIB)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    path = build(force=a.force, verbose=a.verbose)
    print(path)
    return 0


if __name__ == "__main__":
    sys.exit(main())
