"""ctypes loader for the C oracle (oracle/tsv_oracle.c) — TEST INFRASTRUCTURE / CPU BASELINE."""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build_oracle

_lib = None
_libs: dict = {}


def _cpu_has_amx() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return " amx_bf16 " in flags and " amx_tile " in flags and _cpu_has_avx512()
    except OSError:
        return False


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return " avx512f " in flags and " avx512bw " in flags and " avx512vl " in flags
    except OSError:
        return False


def _open(variant: str):
    if variant in _libs:
        return _libs[variant]
    p = build_oracle.lib_path(variant)
    if not p.exists():
        build_oracle.build()
    lib = ctypes.CDLL(str(p))
    lib.tsv_oracle_search.restype = ctypes.c_int
    lib.tsv_oracle_search.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p]
    lib.tsv_oracle_threads.restype = ctypes.c_int
    lib.variant = variant
    lib.amx = False
    if variant == "amx":
        lib.tsv_oracle_search_amx.restype = ctypes.c_int
        lib.tsv_oracle_search_amx.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p]
        lib.tsv_oracle_amx_available.restype = ctypes.c_int
        lib.amx = bool(lib.tsv_oracle_amx_available())
    _libs[variant] = lib
    return lib


def load(variant: str | None = None):
    """Load the C oracle. Without an explicit variant, pick the faster of the available
    builds on this host (AVX-512 is not always the faster one on virtualised hosts)."""
    global _lib
    if variant is not None:
        return _open(variant)
    if _lib is not None:
        return _lib
    variant = os.environ.get("TSV_ORACLE_VARIANT")
    if variant:
        _lib = _open(variant)
        return _lib
    cands = ["v3", "v4"] if _cpu_has_avx512() else ["v3"]
    if _cpu_has_amx() and _open("amx").amx:
        cands.append("amx")
    if len(cands) == 1:
        _lib = _open(cands[0])
        return _lib
    import time

    rng = np.random.default_rng(0)
    q = rng.integers(0x3C00, 0x3F80, size=(64, 512), dtype=np.uint16)
    c = rng.integers(0x3C00, 0x3F80, size=(32768, 512), dtype=np.uint16)
    best = None
    for v in cands:
        lib = _open(v)
        t = time.perf_counter()
        _search(lib, q, c, 10, False, 0, 0)
        dt = time.perf_counter() - t
        if best is None or dt < best[0]:
            best = (dt, lib)
    _lib = best[1]
    return _lib


def threads() -> int:
    return int(load().tsv_oracle_threads())


def search(q_bits: np.ndarray, c_bits: np.ndarray, k: int, use_double: bool = False,
           nthreads: int = 0, id_offset: int = 0):
    """q_bits/c_bits: uint16 bf16 bit patterns [B, D] / [N, D]. Returns (scores f32, ids i32)."""
    return _search(load(), q_bits, c_bits, k, use_double, nthreads, id_offset)


def _search(lib, q_bits, c_bits, k, use_double, nthreads, id_offset):
    q = np.ascontiguousarray(q_bits, dtype=np.uint16)
    c = np.ascontiguousarray(c_bits, dtype=np.uint16)
    B, D = q.shape
    N = c.shape[0]
    out_s = np.empty((B, k), dtype=np.float32)
    out_i = np.empty((B, k), dtype=np.int32)
    if lib.amx and not use_double and D % 32 == 0:
        rc = lib.tsv_oracle_search_amx(q.ctypes.data, c.ctypes.data, B, N, D, k,
                                       int(nthreads or os.cpu_count() or 1), int(id_offset),
                                       out_s.ctypes.data, out_i.ctypes.data)
        if rc == 0:
            return out_s, out_i
    rc = lib.tsv_oracle_search(q.ctypes.data, c.ctypes.data, B, N, D, k, int(use_double),
                               int(nthreads or os.cpu_count() or 1), int(id_offset),
                               out_s.ctypes.data, out_i.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"tsv_oracle_search failed ({rc})")
    return out_s, out_i
