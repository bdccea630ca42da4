"""Builds libtierflow_b200.so in-tree (and libtierflow_b200_tuning.so, the
kernel variants, unless --no-tuning): the sm_100a kernels (nvcc) and the C++
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
TUNING_LIB = LIB_DIR / "libtierflow_b200_tuning.so"
OBJ_DIR = PKG.parent / "build" / "obj"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"

# The product library: the shipped kernels, the engine, the C ABI.
CU_SOURCES = ["kernels.cu", "adam_kernel.cu"]
CXX_SOURCES = ["tier.cpp", "engine.cpp", "capi.cpp", "capi_host.cpp"]
# The tuning library (include/tierflow_b200_tuning.h): the measured kernel
# variants, for sweeps and the all-variants parity test; linked against the
# product library, never loaded by it.
TUNING_CU = ["adam_variants.cu", "adam_variants_hi.cu"]
TUNING_CXX = ["tuning_capi.cpp"]


def _sources(cu, cxx) -> list[Path]:
    files = [CSRC / s for s in cu + cxx]
    files += sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    return files


def _fresh(lib: Path, cu, cxx) -> bool:
    if not lib.exists():
        return False
    built = lib.stat().st_mtime
    return all(f.stat().st_mtime <= built for f in _sources(cu, cxx))


def up_to_date(tuning: bool = True) -> bool:
    return _fresh(LIB, CU_SOURCES, CXX_SOURCES) and (
        not tuning or (_fresh(TUNING_LIB, TUNING_CU, TUNING_CXX) and TUNING_LIB.stat().st_mtime >= LIB.stat().st_mtime))


def _run(cmd: list[str], verbose: bool) -> str:
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stdout + res.stderr


def _compile_jobs(cu, cxx):
    cuda_inc = str(CUDA_HOME / "include")
    jobs = []
    for src in cu:
        obj = OBJ_DIR / (Path(src).stem + ".o")
        jobs.append((obj, [NVCC, GENCODE, "-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v",
                           "-Xcompiler", "-fPIC", "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]))
    for src in cxx:
        obj = OBJ_DIR / (Path(src).stem + ".o")
        jobs.append((obj, ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-Wall", "-Wextra", "-pthread",
                           "-I", cuda_inc, "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]))
    return jobs


def build(force: bool = False, verbose: bool = False, tuning: bool = True) -> Path:
    """Builds the product library and (tuning=True) the tuning library."""
    if not force and up_to_date(tuning):
        return LIB
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    product = _compile_jobs(CU_SOURCES, CXX_SOURCES)
    extra = _compile_jobs(TUNING_CU, TUNING_CXX) if tuning else []
    jobs = product + extra
    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        logs = list(ex.map(lambda j: _run(j[1], verbose), jobs))
    (OBJ_DIR / "ptxas.log").write_text(logs[0] + logs[1] + "".join(logs[len(product):len(product) + len(TUNING_CU)]))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, GENCODE, "-shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for o, _ in product]
         + ["-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], verbose)
    os.replace(tmp, LIB)
    if tuning:
        tmp = TUNING_LIB.with_suffix(".so.tmp")
        _run([NVCC, GENCODE, "-shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for o, _ in extra]
             + ["-L", str(LIB_DIR), "-ltierflow_b200", "-Xlinker", "-rpath=$ORIGIN", "-Xlinker", "--no-undefined",
                "-lpthread", "-ldl", "-lrt"], verbose)
        os.replace(tmp, TUNING_LIB)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--no-tuning", action="store_true", help="product library only (no kernel variants)")
    a = ap.parse_args(argv)
    path = build(force=a.force, verbose=a.verbose, tuning=not a.no_tuning)
    print(path)
    return 0


if __name__ == "__main__":
    sys.exit(main())
