"""Multi-process (world_size 2 and 3, gloo, CPU) test of the corpus-sharded search wiring:
shard ranges, global id offsets, the all-gather and the merge. The device kernels are
replaced by the CPU oracle here (test doubles); on B200 the same class runs K1 + NCCL + K4."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, dim, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_00326_b200.sharded import ShardedSearch, shard_range

    corpus = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(corpus, 9, seed=1)
    lo, hi = shard_range(n, rank, world)
    local = corpus[lo:hi]  # this rank's shard only

    def search_fn(qt, kk, id_offset, out=None):
        s, i = orc.search(qt.numpy(), local, kk, id_offset=id_offset)
        out[0].copy_(torch.from_numpy(s.astype(np.float32)))
        out[1].copy_(torch.from_numpy(i.astype(np.int32)))
        return out

    def merge_fn(s_all, i_all, kk):
        s, i = orc.merge(s_all.numpy(), i_all.numpy(), kk)
        return torch.from_numpy(s.astype(np.float32)), torch.from_numpy(i.astype(np.int32))

    ss = ShardedSearch(None, n, search_fn=search_fn, merge_fn=merge_fn)
    assert (ss.lo, ss.hi) == (lo, hi)
    s, i = ss.search(torch.from_numpy(q), k)
    out[rank] = (s.numpy().copy(), i.numpy().copy(), ss.exchange_bytes(9, k))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_equals_unsharded(world):
    n, dim, k = 1001, 32, 7
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, dim, k, out), nprocs=world, join=True)
    corpus = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(corpus, 9, seed=1)
    es, ei = orc.search(q, corpus, k)
    for r in range(world):
        s, i, xbytes = out[r]
        np.testing.assert_array_equal(i, ei)
        np.testing.assert_allclose(s, es, rtol=1e-6)
        assert xbytes == (world - 1) * 9 * k * 8


def test_shard_ranges_partition_the_corpus():
    from paper_2407_00326_b200.sharded import shard_range

    for n in (1, 7, 10_000_000):
        for world in (1, 2, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
