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
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of the global corpus held by `rank`."""
    return n_rows * rank // world, n_rows * (rank + 1) // world


class ShardedSearch:
    def __init__(self, index, n_rows: int, rank: int | None = None, world: int | None = None,
                 group=None, search_fn: Callable | None = None, merge_fn: Callable | None = None):
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

    def search(self, q: torch.Tensor, k: int):
        """Global top-k of q over the sharded corpus; identical result on every rank."""
        s_loc, i_loc, s_all, i_all = self._buffers(q.shape[0], k, q.device)
        self.search_fn(q, k, id_offset=self.lo, out=(s_loc, i_loc))
        if self.world == 1:
            return s_loc, i_loc
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
