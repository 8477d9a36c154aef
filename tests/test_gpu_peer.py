"""Fused peer all-gather + merge (sharded mode over NVLink): 2 and 4 ranks, run here as
processes sharing one GPU through CUDA IPC (the same code maps peer GPUs over NVLink on a
node). The result must equal the unsharded search, over several calls (buffer parities)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
# (query seed, batch): smaller batches leave the upper query slots of the group untouched; the
# next full batch must not wait for them (cumulative per-slot counters hung here)
CALLS = [(1, 64), (2, 32), (3, 64), (4, 16), (5, 64)]


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
    for seed, b in CALLS:  # varying batch sizes reuse the group created for the first (64)
        q, _ = orc.make_queries(corpus, b, seed=seed)
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
    for call, (seed, b) in enumerate(CALLS):
        q, _ = orc.make_queries(corpus, b, seed=seed)
        for r in range(world):
            s, i = out[r][call]
            assert not orc.check_topk(s, i, q, corpus, 10, 1e-3)
        for r in range(1, world):
            np.testing.assert_array_equal(out[0][call][1], out[r][call][1])


def _silent_peer_worker(rank, world, port, out):
    """Rank 1 never calls the exchange: rank 0's call must abort after its timeout and report
    DeviceError, not hang."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_00326_b200.errors import DeviceError
    from paper_2407_00326_b200.sharded import PeerExchange

    dev = torch.device("cuda", 0)
    pe = PeerExchange(dev, 64, 10)
    if rank == 0:
        import time

        pe.set_timeout_ms(500)
        s = torch.zeros((64, 10), dtype=torch.float32, device=dev)
        i = torch.arange(640, dtype=torch.int32, device=dev).view(64, 10)
        t = time.time()
        o_s, o_i = pe.allgather_merge(s, i, 10)
        torch.cuda.synchronize()
        out["elapsed"] = time.time() - t
        out["padded"] = bool((o_i == -1).all().item())
        try:
            pe.status()
            out["status"] = "ok"
        except DeviceError as exc:
            out["status"] = f"DeviceError: {exc}"
        try:
            pe.allgather_merge(s, i, 10)
            out["next"] = "ok"
        except DeviceError:
            out["next"] = "DeviceError"
    dist.barrier()
    pe.close()
    dist.destroy_process_group()


def test_p2p_missing_peer_times_out(cuda):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_silent_peer_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out["elapsed"] < 30
    assert out["padded"]
    assert out["status"].startswith("DeviceError")
    assert out["next"] == "DeviceError"


@pytest.mark.parametrize("world,k", [(2, 10), (4, 100), (8, 10), (8, 100)])
def test_in_process_peer_group_equals_merge(cuda, world, k):
    """tsv_peer_attach: G ranks in one process on one device, every rank's K6 on its own
    stream; each rank's result equals K4 over all ranks' lists, over varying batch sizes, with
    lists ordered as K1 / K4 emit them (score desc, id asc) and, every other call, scores on a
    coarse grid (many exact cross-list ties)."""
    import torch

    from paper_2407_00326_b200.index import merge_topk
    from paper_2407_00326_b200.sharded import LocalPeerGroup

    grp = LocalPeerGroup([cuda.index] * world, 64, k)
    grp.set_timeout_ms(20_000)
    streams = [torch.cuda.Stream(cuda) for _ in range(world)]
    g = torch.Generator(device=cuda).manual_seed(world * k)
    for call, (_, b) in enumerate(CALLS * 2):
        s = torch.rand((world, b, k), generator=g, device=cuda)
        if call % 2:
            s = torch.floor(s * 64) / 64
        i = torch.randperm(world * b * k, generator=g, device=cuda).to(torch.int32).reshape(world, b, k)
        o = torch.argsort(i, dim=2)
        s, i = torch.gather(s, 2, o), torch.gather(i, 2, o)
        o = torch.sort(s, dim=2, descending=True, stable=True)[1]
        s, i = torch.gather(s, 2, o).contiguous(), torch.gather(i, 2, o).contiguous()
        for st in streams:  # the rank streams read lists made on the current stream
            st.wait_stream(torch.cuda.current_stream(cuda))
        outs = [grp.allgather_merge(r, s[r], i[r], k, stream=streams[r]) for r in range(world)]
        torch.cuda.synchronize()
        grp.status()
        ref_s, ref_i = merge_topk(s, i, k)
        for r in range(world):
            assert torch.equal(outs[r][1], ref_i), (world, k, call, r)
            assert torch.equal(outs[r][0], ref_s), (world, k, call, r)
    grp.close()
