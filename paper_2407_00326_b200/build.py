"""Builds the in-tree CUDA library ``lib/libtsv.so`` for sm_100a with plain nvcc.

The library exports the C ABI declared in ``include/tsv.h``. It is built in-tree so the
shared object travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libtsv.so"
SOURCES = ["tsv_scan.cu", "tsv_merge.cu", "tsv_capi.cu", "tsv_sched.cpp"]
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtsv.so")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = (list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.cpp"))) + [ROOT / "include" / "tsv.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    nvcc = nvcc_path()
    objs = []
    tmp = LIB_DIR / "obj"
    tmp.mkdir(exist_ok=True)
    common = [GENCODE, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", f"-I{ROOT / 'include'}", "-DTSV_BUILD"]
    for src in SOURCES:
        obj = tmp / (src + ".o")
        cmd = [nvcc, *common, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    out_tmp = LIB.with_suffix(".so.tmp")
    # libcuda is not linked: the one driver call (cuTensorMapEncodeTiled) is resolved at run
    # time through cudaGetDriverEntryPoint.
    cmd = [nvcc, GENCODE, "-shared", "-cudart", "static", *objs, "-o", str(out_tmp)]
    subprocess.run(cmd, check=True)
    os.replace(out_tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
