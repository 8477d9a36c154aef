"""Device-resident corpus arena and the retrieval primitives over it (host side of the C ABI).

PyTorch is used only for device memory and streams; every computation is a kernel of
``lib/libtsv.so`` reached through ``_native``.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _native as nat
from .errors import CapacityExceeded, ConfigParse, DeviceError

METRICS = {"ip": nat.TSV_METRIC_IP, "cosine": nat.TSV_METRIC_COSINE}
_DTYPES = {torch.bfloat16: nat.TSV_BF16, torch.float32: nat.TSV_F32}


def _dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ConfigParse(f"unsupported dtype {t.dtype}; expected bfloat16 or float32") from None


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise DeviceError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ConfigParse(f"{name} must be contiguous")


def _check_out(out, B: int, k: int, device: torch.device) -> None:
    """Caller-provided result buffers: contiguous float32 scores / int32 ids [B, k] on the
    index's device (the kernels write B * k entries through raw pointers)."""
    if not isinstance(out, (tuple, list)) or len(out) != 2:
        raise ConfigParse("out must be a (scores, ids) pair")
    s, i = out
    for t, name, dt in ((s, "out scores", torch.float32), (i, "out ids", torch.int32)):
        if not isinstance(t, torch.Tensor) or t.dtype != dt:
            raise ConfigParse(f"{name} must be a {dt} tensor")
        if tuple(t.shape) != (B, k):
            raise ConfigParse(f"{name} must have shape {(B, k)}, got {tuple(t.shape)}")
        if not t.is_cuda or t.device != device:
            raise DeviceError(f"{name} must be on {device}")
        if not t.is_contiguous():
            raise ConfigParse(f"{name} must be contiguous")


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _out_pair(B: int, k: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """(scores fp32 [B, k], ids int32 [B, k]) carved from ONE allocation: a caching-allocator
    call costs tens of microseconds when the host path is cold (inside a scheduler loop)."""
    buf = torch.empty((2, B, k), dtype=torch.int32, device=device)
    return buf[0].view(torch.float32), buf[1]


def _stream_handle(stream: torch.cuda.Stream | None, device: torch.device) -> int:
    """cudaStream_t of `stream`, or of the device's current torch stream. The current stream is
    read through torch's raw-handle accessor when it exists: building a Stream object costs
    ~6 us per call, about half of a search call's host time."""
    if stream is not None:
        return stream.cuda_stream
    if _RAW_STREAM is not None:
        return _RAW_STREAM(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


class _ArenaView:
    """__cuda_array_interface__ exporter so torch can alias the arena without a copy."""

    def __init__(self, ptr: int, rows: int, dim: int, typestr: str = "<u2"):
        self.__cuda_array_interface__ = {
            "shape": (rows, dim), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


STORAGE = {"bf16": nat.TSV_BF16, "f32": nat.TSV_F32, "bf16_tiled": nat.TSV_BF16_TILED}


class DeviceIndex:
    """A bf16 corpus arena on one GPU (reference role: the vector DB behind `vdb-search0`)."""

    def __init__(self, dim: int, capacity: int, metric: str = "ip", device: int | None = None,
                 storage: str = "bf16", _handle: int | None = None,
                 _keepalive: torch.Tensor | None = None):
        """storage="f32" is the fp32 mode: rows kept as tf32 hi + fp32 residual planes, search
        by 3xTF32 tensor-core products (scores within 1e-5 relative, k <= 64)."""
        lib = nat.load()
        if metric not in METRICS:
            raise ConfigParse(f"unknown metric {metric!r}")
        if storage not in STORAGE:
            raise ConfigParse(f"unknown storage {storage!r}")
        self.metric = metric
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._keepalive = _keepalive
        if _handle is not None:
            self._h = ctypes.c_void_p(_handle)
        else:
            h = ctypes.c_void_p()
            nat.check(lib.tsv_index_create2(self.device.index, int(dim), METRICS[metric],
                                            STORAGE[storage], int(capacity), ctypes.byref(h)))
            self._h = h
        self.dim = int(lib.tsv_index_dim(self._h))
        self.capacity = int(capacity)
        self.storage = {v: k for k, v in STORAGE.items()}[lib.tsv_index_storage(self._h)]

    @classmethod
    def view(cls, rows: torch.Tensor, metric: str = "ip") -> "DeviceIndex":
        """Wrap an existing [n, dim] bf16 CUDA matrix without copying it."""
        _require_cuda(rows, "rows")
        if rows.dtype != torch.bfloat16 or rows.dim() != 2:
            raise ConfigParse("a view index needs a 2-D bfloat16 matrix")
        lib = nat.load()
        h = ctypes.c_void_p()
        nat.check(lib.tsv_index_create_view(rows.device.index, rows.shape[1], METRICS[metric],
                                            rows.data_ptr(), rows.shape[0], ctypes.byref(h)))
        return cls(rows.shape[1], rows.shape[0], metric, rows.device.index, _handle=h.value,
                   _keepalive=rows)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            nat.load().tsv_index_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- arena ---------------------------------------------------------------
    @property
    def rows(self) -> int:
        return int(nat.load().tsv_index_rows(self._h))

    def data(self) -> torch.Tensor:
        """bf16 storage: aliasing tensor [rows, dim] over the arena (what the kernels read).
        f32 storage: the fp32 rows the kernels represent (hi + lo planes, a new tensor)."""
        if self.storage == "f32":
            hi, lo = self.planes()
            return hi + lo
        ptr = nat.load().tsv_index_data(self._h)
        if self.storage == "bf16_tiled":  # de-tile into a new [rows, dim] tensor
            kbs = (self.dim + 63) // 64
            tiles = (self.rows + 127) // 128
            t = torch.as_tensor(_ArenaView(ptr, tiles * kbs * 128, 64), device=self.device)
            t = t.view(torch.bfloat16).view(tiles, kbs, 128, 64).permute(0, 2, 1, 3)
            return t.reshape(tiles * 128, kbs * 64)[: self.rows, : self.dim].contiguous()
        t = torch.as_tensor(_ArenaView(ptr, self.rows, self.dim), device=self.device)
        return t.view(torch.bfloat16)

    def planes(self) -> tuple[torch.Tensor, torch.Tensor]:
        """fp32 mode: aliasing (hi, lo) float32 tensors [rows, dim]."""
        if self.storage != "f32":
            raise ConfigParse("planes() needs an f32-storage index")
        lib = nat.load()
        mk = lambda ptr: torch.as_tensor(_ArenaView(ptr, self.rows, self.dim, "<f4"),
                                         device=self.device)
        return mk(lib.tsv_index_data(self._h)), mk(lib.tsv_index_data_lo(self._h))

    def append(self, rows: torch.Tensor, stream: torch.cuda.Stream | None = None) -> int:
        """Ingest rows (normalised for cosine); returns the arena row of the first one."""
        _require_cuda(rows, "rows")
        if rows.dim() != 2 or rows.shape[1] != self.dim:
            raise ConfigParse(f"rows must be [n, {self.dim}]")
        first = ctypes.c_int64()
        nat.check(nat.load().tsv_index_append(self._h, rows.data_ptr(), _dtype_code(rows),
                                              rows.shape[0], ctypes.byref(first),
                                              _stream_handle(stream, self.device)))
        return int(first.value)

    def reserve(self, n: int) -> int:
        """Claim n arena rows without writing them (the caller fills them, e.g. the ingest
        stages of a per-query index); returns the first claimed row."""
        first = ctypes.c_int64()
        nat.check(nat.load().tsv_index_reserve(self._h, int(n), ctypes.byref(first)))
        return int(first.value)

    def truncate(self, rows: int) -> None:
        nat.check(nat.load().tsv_index_truncate(self._h, int(rows)))

    def set_timing(self, enable: bool) -> None:
        nat.check(nat.load().tsv_index_set_timing(self._h, int(bool(enable))))

    def scan_time(self) -> tuple[float, int]:
        """(total ms, launches) of fused-scan kernels since the last read (timing mode)."""
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        nat.check(nat.load().tsv_index_scan_time(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return float(ms.value), int(n.value)

    # -- primitives ----------------------------------------------------------
    def _check_queries(self, q: torch.Tensor) -> None:
        _require_cuda(q, "queries")
        if q.device != self.device:
            raise DeviceError(f"queries are on {q.device}, the index on {self.device}")
        if q.dim() != 2 or q.shape[1] != self.dim:
            raise ConfigParse(f"queries must be [B, {self.dim}]")
        if q.shape[0] == 0:
            raise CapacityExceeded("empty batch")

    def search(self, q: torch.Tensor, k: int, row_range: tuple[int, int] | None = None,
               id_offset: int = 0, stream: torch.cuda.Stream | None = None,
               out: tuple[torch.Tensor, torch.Tensor] | None = None):
        """Top-k over arena rows [row_range) for each query; ids = row + id_offset."""
        self._check_queries(q)
        lo, hi = row_range if row_range is not None else (0, self.rows)
        B = q.shape[0]
        if out is None:
            scores, ids = _out_pair(B, k, self.device)
        else:
            _check_out(out, B, int(k), self.device)
            scores, ids = out
        nat.check(nat.load().tsv_search(self._h, q.data_ptr(), _dtype_code(q), B, int(k), int(lo),
                                        int(hi), int(id_offset), scores.data_ptr(), ids.data_ptr(),
                                        _stream_handle(stream, self.device)))
        return scores, ids

    def search_segmented(self, q: torch.Tensor, q_offsets: Sequence[int],
                         row_ranges: Sequence[tuple[int, int]], k: int, local_ids: bool = True,
                         stream: torch.cuda.Stream | None = None,
                         out: tuple[torch.Tensor, torch.Tensor] | None = None):
        """Queries q[q_offsets[s]:q_offsets[s+1]] search only arena rows row_ranges[s]."""
        self._check_queries(q)
        nseg = len(row_ranges)
        if nseg == 0:
            raise CapacityExceeded("empty batch")
        if len(q_offsets) != nseg + 1 or q_offsets[-1] != q.shape[0]:
            raise ConfigParse("q_offsets must have nseg+1 entries ending at B")
        qo = (ctypes.c_int32 * (nseg + 1))(*[int(x) for x in q_offsets])
        rb = (ctypes.c_int64 * nseg)(*[int(a) for a, _ in row_ranges])
        re = (ctypes.c_int64 * nseg)(*[int(b) for _, b in row_ranges])
        B = q.shape[0]
        if out is None:
            scores, ids = _out_pair(B, k, self.device)
        else:
            _check_out(out, B, int(k), self.device)
            scores, ids = out
        nat.check(nat.load().tsv_search_segmented(
            self._h, q.data_ptr(), _dtype_code(q), nseg, ctypes.cast(qo, ctypes.c_void_p),
            ctypes.cast(rb, ctypes.c_void_p), ctypes.cast(re, ctypes.c_void_p), int(k),
            int(bool(local_ids)), scores.data_ptr(), ids.data_ptr(),
            _stream_handle(stream, self.device)))
        return scores, ids

    def search_rerank_segmented(self, q: torch.Tensor, q_rows: torch.Tensor, max_rows: int,
                                k_search: int, k_rerank: int,
                                q_rerank: torch.Tensor | None = None, local_ids: bool = True,
                                stream: torch.cuda.Stream | None = None, out_search=None,
                                out_rerank=None):
        """Contextual retrieval's Searching -> Reranking chain in one launch: query b searches
        arena rows [q_rows[b, 0], q_rows[b, 1]) (its own index segment; int64 [B, 2] on the
        device, or a host sequence of 2 B ints [b0, e0, b1, e1, ...] uploaded through the
        library's pinned slots; every segment <= max_rows <= 1024 rows), keeps the top
        k_search, and reranks them against q_rerank[b] (default: the query itself), keeping
        the top k_rerank. Returns ((search scores, ids), (rerank scores, ids))."""
        self._check_queries(q)
        B = q.shape[0]
        if q_rerank is not None:
            self._check_queries(q_rerank)
            if q_rerank.shape != q.shape or q_rerank.dtype != q.dtype:
                raise ConfigParse("q_rerank must match q in shape and dtype")
            q_rerank = q_rerank.contiguous()
        host_rows = isinstance(q_rows, (list, tuple))
        if host_rows:
            if len(q_rows) != 2 * B:
                raise ConfigParse(f"q_rows must hold {2 * B} ints (begin, end per query)")
            rows_arg = ctypes.cast((ctypes.c_int64 * (2 * B))(*q_rows), ctypes.c_void_p)
        else:
            _require_cuda(q_rows, "q_rows")
            if (q_rows.dtype != torch.int64 or tuple(q_rows.shape) != (B, 2)
                    or q_rows.device != self.device or not q_rows.is_contiguous()):
                raise ConfigParse(f"q_rows must be contiguous int64 [{B}, 2] on {self.device}")
            rows_arg = q_rows.data_ptr()
        bufs = []
        for o, kk in ((out_search, k_search), (out_rerank, k_rerank)):
            if o is None:
                o = _out_pair(B, kk, self.device)
            else:
                _check_out(o, B, int(kk), self.device)
            bufs.append(o)
        (ss, si), (rs, ri) = bufs
        fn = (nat.load().tsv_search_rerank_segmented_host if host_rows
              else nat.load().tsv_search_rerank_segmented)
        nat.check(fn(
            self._h, q.contiguous().data_ptr(), None if q_rerank is None else q_rerank.data_ptr(),
            _dtype_code(q), B, rows_arg, int(max_rows), int(k_search), int(k_rerank),
            int(bool(local_ids)), ss.data_ptr(), si.data_ptr(), rs.data_ptr(), ri.data_ptr(),
            _stream_handle(stream, self.device)))
        return (ss, si), (rs, ri)

    def rerank(self, q: torch.Tensor, cand_ids: torch.Tensor, k: int,
               stream: torch.cuda.Stream | None = None,
               out: tuple[torch.Tensor, torch.Tensor] | None = None,
               row_offsets: torch.Tensor | None = None):
        """Score cand_ids[b, :] (arena rows) against q[b]; dedup ids; keep the best k.
        row_offsets (int32 [B] on the device, or a host list of B ints): the candidates of
        question b are rows of its own index segment starting at arena row row_offsets[b]; ids
        stay segment-local."""
        self._check_queries(q)
        _require_cuda(cand_ids, "cand_ids")
        if cand_ids.dtype != torch.int32 or cand_ids.dim() != 2 or cand_ids.shape[0] != q.shape[0]:
            raise ConfigParse("cand_ids must be int32 [B, C]")
        if cand_ids.device != self.device:
            raise DeviceError(f"cand_ids are on {cand_ids.device}, the index on {self.device}")
        B, C = cand_ids.shape
        if out is None:
            scores, ids = _out_pair(B, k, self.device)
        else:
            _check_out(out, B, int(k), self.device)
            scores, ids = out
        if isinstance(row_offsets, (list, tuple)):
            if len(row_offsets) != B:
                raise ConfigParse(f"row_offsets must have {B} entries")
            offs = (ctypes.c_int32 * B)(*row_offsets)
            nat.check(nat.load().tsv_rerank_segmented_host(
                self._h, q.data_ptr(), _dtype_code(q), B, cand_ids.data_ptr(), C,
                ctypes.cast(offs, ctypes.c_void_p), int(k), scores.data_ptr(), ids.data_ptr(),
                _stream_handle(stream, self.device)))
            return scores, ids
        if row_offsets is not None:
            _require_cuda(row_offsets, "row_offsets")
            if (row_offsets.dtype != torch.int32 or row_offsets.numel() != B
                    or row_offsets.device != self.device):
                raise ConfigParse(f"row_offsets must be int32 [{B}] on {self.device}")
            nat.check(nat.load().tsv_rerank_segmented(
                self._h, q.data_ptr(), _dtype_code(q), B, cand_ids.data_ptr(), C,
                row_offsets.data_ptr(), int(k), scores.data_ptr(), ids.data_ptr(),
                _stream_handle(stream, self.device)))
            return scores, ids
        nat.check(nat.load().tsv_rerank(self._h, q.data_ptr(), _dtype_code(q), B,
                                        cand_ids.data_ptr(), C, int(k), scores.data_ptr(),
                                        ids.data_ptr(), _stream_handle(stream, self.device)))
        return scores, ids


def merge_topk(scores: torch.Tensor, ids: torch.Tensor, k: int,
               stream: torch.cuda.Stream | None = None, dedup: bool = False):
    """Merge [L, B, kin] sorted lists into [B, k] (Aggregate join / cross-shard merge);
    dedup keeps one entry per id."""
    _require_cuda(scores, "scores")
    _require_cuda(ids, "ids")
    if scores.dim() != 3 or scores.shape != ids.shape:
        raise ConfigParse("scores/ids must be [lists, B, kin]")
    if scores.dtype != torch.float32 or ids.dtype != torch.int32:
        raise ConfigParse("scores must be float32 and ids int32")
    L, B, kin = scores.shape
    out_s, out_i = _out_pair(B, k, scores.device)
    nat.check(nat.load().tsv_merge_topk(scores.data_ptr(), ids.data_ptr(), L, B, kin, int(k),
                                        int(bool(dedup)), out_s.data_ptr(), out_i.data_ptr(),
                                        _stream_handle(stream, scores.device)))
    return out_s, out_i


def normalize_rows(x: torch.Tensor, normalize: bool = True,
                   stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """L2-normalise rows (fp32 math) and cast to bf16 on the device."""
    _require_cuda(x, "x")
    if x.dim() != 2:
        raise ConfigParse("x must be 2-D")
    out = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    nat.check(nat.load().tsv_normalize_rows(x.data_ptr(), _dtype_code(x), x.shape[0], x.shape[1],
                                            int(bool(normalize)), out.data_ptr(),
                                            _stream_handle(stream, x.device)))
    return out
