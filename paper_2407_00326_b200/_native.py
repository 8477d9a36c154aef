"""ctypes binding of the C ABI in ``include/tsv.h`` (``lib/libtsv.so``).

There is no fallback: if the shared library is missing or fails to load, every entry point
raises ``DeviceError``. Buffers are passed as raw device pointers and streams as raw
``cudaStream_t`` handles, exactly as a foreign-language binding of the reference would.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import STATUS_ERRORS, DeviceError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libtsv.so"
if os.environ.get("TSV_LIB_PATH"):  # development A/B of two builds of the same ABI
    LIB_PATH = Path(os.environ["TSV_LIB_PATH"])

TSV_BF16 = 0
TSV_F32 = 1
TSV_BF16_TILED = 2
TSV_METRIC_IP = 0
TSV_METRIC_COSINE = 1

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_dbl = ctypes.c_double

# name -> (restype, argtypes). Every symbol declared in include/tsv.h.
SIGNATURES = {
    "tsv_abi_version": (c_int, []),
    "tsv_last_error": (ctypes.c_char_p, []),
    "tsv_launch_count": (c_i64, []),
    "tsv_index_create": (c_int, [c_int, c_int, c_int, c_i64, ctypes.POINTER(c_vp)]),
    "tsv_index_create2": (c_int, [c_int, c_int, c_int, c_int, c_i64, ctypes.POINTER(c_vp)]),
    "tsv_index_create_view": (c_int, [c_int, c_int, c_int, c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "tsv_index_destroy": (c_int, [c_vp]),
    "tsv_index_append": (c_int, [c_vp, c_vp, c_int, c_i64, ctypes.POINTER(c_i64), c_vp]),
    "tsv_index_reserve": (c_int, [c_vp, c_i64, ctypes.POINTER(c_i64)]),
    "tsv_index_truncate": (c_int, [c_vp, c_i64]),
    "tsv_index_rows": (c_i64, [c_vp]),
    "tsv_index_dim": (c_int, [c_vp]),
    "tsv_index_metric": (c_int, [c_vp]),
    "tsv_index_data": (c_vp, [c_vp]),
    "tsv_index_data_lo": (c_vp, [c_vp]),
    "tsv_index_storage": (c_int, [c_vp]),
    "tsv_index_set_timing": (c_int, [c_vp, c_int]),
    "tsv_index_scan_time": (c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "tsv_search": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_i64, c_i64, c_i32, c_vp, c_vp,
                           c_vp]),
    "tsv_search_segmented": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_int,
                                     c_vp, c_vp, c_vp]),
    "tsv_rerank": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_int, c_int, c_vp, c_vp, c_vp]),
    "tsv_rerank_segmented": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp,
                                     c_vp, c_vp]),
    "tsv_rerank_segmented_host": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_int, c_vp, c_int, c_vp,
                                     c_vp, c_vp]),
    "tsv_search_rerank_segmented": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_int, c_int,
                                            c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tsv_search_rerank_segmented_host": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_int,
                                                 c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp,
                                                 c_vp]),
    "tsv_merge_topk": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp]),
    "tsv_normalize_rows": (c_int, [c_vp, c_int, c_i64, c_int, c_int, c_vp, c_vp]),
    "tsv_peer_create": (c_int, [c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_vp)]),
    "tsv_peer_handle": (c_int, [c_vp, c_vp, ctypes.POINTER(c_int)]),
    "tsv_peer_open": (c_int, [c_vp, c_int, c_vp]),
    "tsv_peer_attach": (c_int, [c_vp, c_int, c_vp]),
    "tsv_peer_allgather_merge": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_vp]),
    "tsv_peer_set_timeout_ms": (c_int, [c_vp, c_i64]),
    "tsv_peer_status": (c_int, [c_vp, ctypes.POINTER(c_int)]),
    "tsv_peer_destroy": (c_int, [c_vp]),
    "tsv_sharded_create": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, ctypes.POINTER(c_vp)]),
    "tsv_sharded_search": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp]),
    "tsv_sharded_destroy": (c_int, [c_vp]),
    "tsv_stream_create": (c_int, [c_int, ctypes.POINTER(c_vp)]),
    "tsv_topo_create": (c_int, [ctypes.c_double, ctypes.POINTER(c_vp)]),
    "tsv_topo_destroy": (c_int, [c_vp]),
    "tsv_topo_size": (c_i64, [c_vp]),
    "tsv_topo_push": (c_int, [c_vp, c_i64, ctypes.c_char_p, ctypes.c_char_p, c_int, c_int,
                              ctypes.c_double, c_vp, c_i64, c_i64]),
    "tsv_topo_form": (c_int, [c_vp, ctypes.c_double, c_i64, c_vp, c_vp,
                              ctypes.POINTER(c_i64), ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(c_int)]),
    "tsv_topo_commit": (c_int, [c_vp, c_vp, c_vp, c_i64]),
    "tsv_stream_destroy": (c_int, [c_vp]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and return the native library; raises DeviceError when unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"native retrieval library missing at {p}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - depends on the host
            raise DeviceError(f"failed to load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    """Raise the TeolaError subclass mapped to a nonzero C-ABI status."""
    if status == 0:
        return
    msg = load().tsv_last_error().decode(errors="replace")
    raise STATUS_ERRORS.get(status, DeviceError)(msg or f"tsv status {status}")


def launch_count() -> int:
    return int(load().tsv_launch_count())


class PrivateStream:
    """A CUDA stream created by the library (not drawn from torch's round-robin stream pool),
    wrapped as a torch ExternalStream. Captured graphs own one each: a pooled stream could be
    handed to another caller whose searches would then share (and grow) the scratch space the
    graph replays."""

    def __init__(self, device: int):
        h = c_vp()
        check(load().tsv_stream_create(int(device), ctypes.byref(h)))
        self.handle = h
        import torch

        self.stream = torch.cuda.ExternalStream(h.value, device=torch.device("cuda", device))

    def close(self) -> None:
        if self.handle is not None and self.handle.value:
            load().tsv_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
