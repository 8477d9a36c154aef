"""Corpus-sharded vector search across GPUs (one process per GPU, torch.distributed / NCCL).

BASELINE config C4: a 10M x 1024 corpus split over G B200s. Rank g holds rows
[g*N/G, (g+1)*N/G) of the global corpus in its own arena; a search step is
    1. every rank runs the fused scan + top-k (K1, + K4 over its ranges) on its shard, with
       global ids (arena row + shard offset);
    2. the per-rank [B, k] (score, id) lists are all-gathered — B*k*8 bytes per rank
       (81,920 B at B=1024, k=10) over NVLink 5 / NVSwitch via NCCL;
    3. every rank merges the G lists (K4) into the global top-k, ordered (score desc, id asc).
Shards are disjoint, so no id can appear twice. The reference has no multi-device path
(SURVEY.md §2.2); its replica concept (`EngineProfile.instances`, engines.py:32) is the
replica mode of backend.py, this module is the corpus-sharded mode.

`search_fn` / `merge_fn` default to the device kernels; tests inject CPU doubles to exercise
the shard arithmetic and collective wiring on the gloo backend.

exchange="p2p" replaces steps 2-3 with one kernel (`tsv_peer_allgather_merge`): every rank
pushes its [B, k] lists straight into the peers' symmetric buffers over NVLink (CUDA IPC
mappings) and merges as soon as all ranks' lists have arrived — the collective and the merge
are one launch, no NCCL call on the data path.
"""

from __future__ import annotations

from typing import Callable

import ctypes

import torch
import torch.distributed as dist


def shard_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of the global corpus held by `rank`."""
    return n_rows * rank // world, n_rows * (rank + 1) // world


class PeerExchange:
    """Symmetric peer buffers across the ranks of a process group (collective constructor)."""

    def __init__(self, device: torch.device, max_b: int, max_k: int, group=None):
        from . import _native as nat

        self.lib = nat.load()
        self.check = nat.check
        self.device = device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.max_b, self.max_k = max_b, max_k
        nccl = dist.get_backend(group) == "nccl"
        self._h = ctypes.c_void_p()
        # Every rank must take the same exchange path, so failures are agreed collectively:
        # byte 64 of each rank's published handle flags a local setup failure, and the
        # result of opening the peers' handles is all-reduced before the buffers are used.
        err = None
        raw = (ctypes.c_ubyte * 65)()
        try:
            self.check(self.lib.tsv_peer_create(device.index, self.world, self.rank, max_b, max_k,
                                                ctypes.byref(self._h)))
            n = ctypes.c_int()
            self.check(self.lib.tsv_peer_handle(self._h, raw, ctypes.byref(n)))
        except Exception as exc:  # noqa: BLE001 - reported collectively below
            err = exc
            raw[64] = 1
        mine = torch.tensor(list(bytes(raw)), dtype=torch.uint8)
        if nccl:
            mine = mine.to(device)
        got = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(got, mine, group=group)
        got = [t.cpu() for t in got]
        if any(int(t[64]) for t in got):
            self.close()
            raise RuntimeError(f"peer buffer setup failed on some rank ({err or 'another rank'})")
        for p, t in enumerate(got):
            buf = (ctypes.c_ubyte * 64)(*t[:64].tolist())
            try:
                self.check(self.lib.tsv_peer_open(self._h, p, buf))
            except Exception as exc:  # noqa: BLE001 - reported collectively below
                err = exc
                break
        flag = torch.tensor([0 if err is None else 1], dtype=torch.int32,
                            device=device if nccl else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        if int(flag.item()) != 0:
            self.close()
            raise RuntimeError(f"peer mapping failed on some rank ({err or 'another rank'})")
        dist.barrier(group)

    def set_timeout_ms(self, ms: int) -> None:
        """Longest wait for a peer's lists before the exchange aborts (DeviceError)."""
        self.check(self.lib.tsv_peer_set_timeout_ms(self._h, int(ms)))

    def status(self) -> None:
        """Raise DeviceError if an exchange of this group gave up waiting for a peer
        (synchronise the stream of the last call first)."""
        flag = ctypes.c_int()
        self.check(self.lib.tsv_peer_status(self._h, ctypes.byref(flag)))

    def allgather_merge(self, s_loc: torch.Tensor, i_loc: torch.Tensor, k: int,
                        stream: torch.cuda.Stream | None = None):
        B = s_loc.shape[0]
        out_s = torch.empty((B, k), dtype=torch.float32, device=self.device)
        out_i = torch.empty((B, k), dtype=torch.int32, device=self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self.check(self.lib.tsv_peer_allgather_merge(self._h, s_loc.data_ptr(), i_loc.data_ptr(),
                                                     B, k, out_s.data_ptr(), out_i.data_ptr(),
                                                     st))
        return out_s, out_i

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.tsv_peer_destroy(self._h)
            self._h = ctypes.c_void_p()


class LocalPeerGroup:
    """The G ranks of a peer exchange driven from ONE process (tsv_peer_attach, no IPC): every
    rank's group lives here and maps the others' buffers directly. Used to measure and test
    K6 with all G kernels in flight at once (ranks on one device, or on peer-accessible
    devices of one node); a multi-process job uses PeerExchange."""

    def __init__(self, devices: list[int], max_b: int, max_k: int):
        from . import _native as nat

        self.lib = nat.load()
        self.check = nat.check
        self.world = len(devices)
        self.devices = [torch.device("cuda", d) for d in devices]
        self.max_b, self.max_k = max_b, max_k
        self._h = []
        try:
            for r, d in enumerate(devices):
                h = ctypes.c_void_p()
                self.check(self.lib.tsv_peer_create(int(d), self.world, r, max_b, max_k,
                                                    ctypes.byref(h)))
                self._h.append(h)
            for r in range(self.world):
                for p in range(self.world):
                    self.check(self.lib.tsv_peer_attach(self._h[r], p, self._h[p]))
        except Exception:
            self.close()
            raise

    def set_timeout_ms(self, ms: int) -> None:
        for h in self._h:
            self.check(self.lib.tsv_peer_set_timeout_ms(h, int(ms)))

    def allgather_merge(self, rank: int, s_loc: torch.Tensor, i_loc: torch.Tensor, k: int,
                        stream: torch.cuda.Stream | None = None, out=None):
        """Rank `rank`'s call: push its [B, k] lists, wait for every rank's, merge. Every rank
        must make the same sequence of calls (each on a stream that can run concurrently)."""
        B = s_loc.shape[0]
        dev = self.devices[rank]
        if out is None:
            out = (torch.empty((B, k), dtype=torch.float32, device=dev),
                   torch.empty((B, k), dtype=torch.int32, device=dev))
        st = (stream or torch.cuda.current_stream(dev)).cuda_stream
        self.check(self.lib.tsv_peer_allgather_merge(self._h[rank], s_loc.data_ptr(),
                                                     i_loc.data_ptr(), B, k, out[0].data_ptr(),
                                                     out[1].data_ptr(), st))
        return out

    def status(self) -> None:
        flag = ctypes.c_int()
        for h in self._h:
            self.check(self.lib.tsv_peer_status(h, ctypes.byref(flag)))

    def close(self) -> None:
        for h in self._h:
            if h.value:
                self.lib.tsv_peer_destroy(h)
        self._h = []


class ShardedSearch:
    def __init__(self, index, n_rows: int, rank: int | None = None, world: int | None = None,
                 group=None, search_fn: Callable | None = None, merge_fn: Callable | None = None,
                 exchange: str = "nccl"):
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        self.p2p_error: str | None = None
        self._peer: PeerExchange | None = None
        self.index = index
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        self.n_rows = n_rows
        self.lo, self.hi = shard_range(n_rows, self.rank, self.world)
        if search_fn is None:
            def search_fn(q, k, id_offset, out=None):
                return index.search(q, k, id_offset=id_offset, out=out)
        if merge_fn is None:
            from .index import merge_topk
            merge_fn = merge_topk
        self.search_fn = search_fn
        self.merge_fn = merge_fn
        self._bufs: dict = {}

    def _buffers(self, B: int, k: int, device):
        key = (B, k, str(device))
        if key not in self._bufs:
            self._bufs[key] = (
                torch.empty((B, k), dtype=torch.float32, device=device),
                torch.empty((B, k), dtype=torch.int32, device=device),
                torch.empty((self.world, B, k), dtype=torch.float32, device=device),
                torch.empty((self.world, B, k), dtype=torch.int32, device=device))
        return self._bufs[key]

    def search(self, q: torch.Tensor, k: int,
               out: tuple[torch.Tensor, torch.Tensor] | None = None):
        """Global top-k of q over the sharded corpus; identical result on every rank.

        With world == 1 the result is written to `out` when given (otherwise to a buffer
        reused by the next call); with world > 1 it is a new pair of tensors."""
        s_loc, i_loc, s_all, i_all = self._buffers(q.shape[0], k, q.device)
        if self.world == 1 and out is not None:
            s_loc, i_loc = out
        self.search_fn(q, k, id_offset=self.lo, out=(s_loc, i_loc))
        if self.world == 1:
            return s_loc, i_loc
        if self.exchange == "p2p":
            if self._peer is None or self._peer.max_b < q.shape[0] or self._peer.max_k < k:
                if self._peer is not None:  # outgrown: every rank re-creates it (same B, k)
                    self._peer.close()
                    self._peer = None
                try:
                    self._peer = PeerExchange(q.device, q.shape[0], k, self.group)
                except Exception as exc:  # no peer mapping on this node: use NCCL instead
                    self.exchange = "nccl"
                    self.p2p_error = f"{type(exc).__name__}: {exc}"
                    return self.search(q, k)
            return self._peer.allgather_merge(s_loc, i_loc, k)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(s_all, s_loc, group=self.group)
            dist.all_gather_into_tensor(i_all, i_loc, group=self.group)
        else:  # gloo (CPU tests): list form, written into the same [G, B, k] buffers
            dist.all_gather(list(s_all.unbind(0)), s_loc, group=self.group)
            dist.all_gather(list(i_all.unbind(0)), i_loc, group=self.group)
        return self.merge_fn(s_all, i_all, k)

    def exchange_bytes(self, B: int, k: int) -> int:
        """Bytes each rank receives per step in the all-gather."""
        return (self.world - 1) * B * k * 8


class ShardedIndex:
    """A corpus split over several devices inside ONE process (tsv_sharded_* in the C ABI).

    Shard g is a DeviceIndex on its own device holding the global rows [offsets[g],
    offsets[g] + rows_g). `search` runs the fused scan + top-k (K1) on every shard on the
    shard's own stream with global ids, gathers the per-shard lists on the root device over
    NVLink (peer writes) and merges them there (K4), stream-ordered on the caller's stream:
    the same result as one index holding every row. This is the single-process counterpart of
    `ShardedSearch` (one process per GPU), so the single-process executor (`Simulator._execute`,
    reference runtime.py:625-656) can serve a corpus larger than one GPU.
    One device may hold several shards (the shards then run concurrently on its SMs)."""

    def __init__(self, shards, root: int | None = None, max_batch: int = 4096, max_k: int = 128,
                 id_offsets=None):
        from . import _native as nat
        from .errors import ConfigParse

        if not shards:
            raise ConfigParse("a sharded index needs at least one shard")
        self.lib = nat.load()
        self._check = nat.check
        self.shards = list(shards)
        self.dim = self.shards[0].dim
        self.metric = self.shards[0].metric
        if id_offsets is None:
            id_offsets, acc = [], 0
            for s in self.shards:
                id_offsets.append(acc)
                acc += s.rows
        self.offsets = [int(x) for x in id_offsets]
        self.device = torch.device("cuda", self.shards[0].device.index if root is None else root)
        self.max_batch, self.max_k = int(max_batch), int(max_k)
        hs = (ctypes.c_void_p * len(self.shards))(*[s._h.value for s in self.shards])
        offs = (ctypes.c_int64 * len(self.shards))(*self.offsets)
        self._h = ctypes.c_void_p()
        self._check(self.lib.tsv_sharded_create(hs, offs, len(self.shards), self.device.index,
                                                self.max_batch, self.max_k,
                                                ctypes.byref(self._h)))

    @property
    def rows(self) -> int:
        return sum(s.rows for s in self.shards)

    def search(self, q: torch.Tensor, k: int, stream: torch.cuda.Stream | None = None,
               out: tuple[torch.Tensor, torch.Tensor] | None = None):
        """Global top-k of q ([B, dim] bf16 / f32 on the root device) over every shard."""
        from .errors import CapacityExceeded, ConfigParse, DeviceError
        from .index import _check_out, _dtype_code

        if not q.is_cuda or q.device != self.device:
            raise DeviceError(f"queries must be on the root device {self.device}")
        if q.dim() != 2 or q.shape[1] != self.dim or not q.is_contiguous():
            raise ConfigParse(f"queries must be a contiguous [B, {self.dim}] matrix")
        if q.shape[0] == 0:
            raise CapacityExceeded("empty batch")
        B = q.shape[0]
        if out is None:
            out = (torch.empty((B, k), dtype=torch.float32, device=self.device),
                   torch.empty((B, k), dtype=torch.int32, device=self.device))
        _check_out(out, B, k, self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(self.lib.tsv_sharded_search(self._h, q.data_ptr(), _dtype_code(q), B, int(k),
                                                out[0].data_ptr(), out[1].data_ptr(), st))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.tsv_sharded_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
