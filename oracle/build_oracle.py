"""Builds the C oracle (test infrastructure / CPU baseline) into oracle/_build/.

Three variants: x86-64-v3 (AVX2+FMA, runs on any current server CPU), x86-64-v4 (AVX-512) and
amx (x86-64-v4 + AMX-BF16 tiles: the fp32-accumulation search on the tensor-tile unit of
Sapphire Rapids and later), picked at load time from the host's CPU flags and a timing probe.
Nothing here is part of the product path.
"""

from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_build"
SRC = HERE / "tsv_oracle.c"
VARIANTS = {"v3": ["-march=x86-64-v3"], "v4": ["-march=x86-64-v4"],
            "amx": ["-march=x86-64-v4", "-mamx-tile", "-mamx-bf16"]}


def lib_path(variant: str) -> Path:
    return OUT / f"libtsv_oracle_{variant}.so"


def build(force: bool = False) -> list[Path]:
    OUT.mkdir(exist_ok=True)
    out = []
    for name, march in VARIANTS.items():
        p = lib_path(name)
        if force or not p.exists() or p.stat().st_mtime < SRC.stat().st_mtime:
            subprocess.run(["gcc", "-O3", *march, "-fopenmp", "-shared", "-fPIC", str(SRC), "-o",
                            str(p), "-lm"], check=True)
        out.append(p)
    return out


if __name__ == "__main__":
    for p in build(force=True):
        print(p)
