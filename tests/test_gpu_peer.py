"""Fused peer all-gather + merge (sharded mode over NVLink): 2 and 4 ranks, run here as
processes sharing one GPU through CUDA IPC (the same code maps peer GPUs over NVLink on a
node). The result must equal the unsharded search, over several calls (buffer parities)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.sharded import ShardedSearch, shard_range
    from tests._util import from_dev, to_dev_bf16

    dev = torch.device("cuda", 0)
    n, dim, k = 20000, 256, 10
    corpus = orc.make_corpus(n, dim, seed=0)
    lo, hi = shard_range(n, rank, world)
    idx = DeviceIndex(dim, hi - lo, device=0)
    idx.append(to_dev_bf16(corpus[lo:hi], dev))
    ss = ShardedSearch(idx, n, rank=rank, world=world, exchange="p2p")
    results = []
    for seed in (1, 2, 3):
        q, _ = orc.make_queries(corpus, 64, seed=seed)
        s, i = ss.search(to_dev_bf16(q, dev), k)
        torch.cuda.synchronize()
        results.append((from_dev(s).copy(), from_dev(i).copy()))
    out[rank] = results
    dist.barrier()
    ss._peer.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_exchange_equals_unsharded(cuda, world):
    import torch.multiprocessing as mp

    from oracle import oracle as orc

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    corpus = orc.make_corpus(20000, 256, seed=0)
    for call, seed in enumerate((1, 2, 3)):
        q, _ = orc.make_queries(corpus, 64, seed=seed)
        for r in range(world):
            s, i = out[r][call]
            assert not orc.check_topk(s, i, q, corpus, 10, 1e-3)
        for r in range(1, world):
            np.testing.assert_array_equal(out[0][call][1], out[r][call][1])
