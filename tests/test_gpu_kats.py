"""The known-answer vectors (tests/golden/retrieval_kats.json) through
the CUDA path: every case goes through the device primitives a caller uses — DeviceIndex.search
(fused scan + top-k, each storage layout), search_segmented, rerank, merge_topk and the sharded
exchange — and must reproduce the analytically derived answer exactly (ids and scores; the
values are small integers / binary fractions, exact in bf16, tf32 and fp32)."""

from __future__ import annotations

import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest

from tests._util import from_dev

pytestmark = pytest.mark.gpu
KATS = json.loads((Path(__file__).resolve().parent / "golden" / "retrieval_kats.json").read_text())


def _exp(kat):
    ids = np.array(kat["ids"], dtype=np.int64)
    scores = np.array([[(-np.inf if v is None else v) for v in row] for row in kat["scores"]],
                      dtype=np.float32)
    return scores, ids


def _arrays(kat):
    return np.array(kat["corpus"], np.float32), np.array(kat["queries"], np.float32)


def _index(c, dev, storage="bf16"):
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    idx = DeviceIndex(c.shape[1], c.shape[0], metric="ip", device=dev.index, storage=storage)
    idx.append(torch.from_numpy(c).to(dev))
    return idx


def _q(q, dev, dtype):
    import torch

    return torch.from_numpy(q).to(dev).to(dtype)


def _assert_exact(s, i, kat):
    es, ei = _exp(kat)
    np.testing.assert_array_equal(from_dev(i), ei)
    np.testing.assert_array_equal(from_dev(s), es)


@pytest.mark.parametrize("storage", ["bf16", "bf16_tiled", "f32"])
@pytest.mark.parametrize("name", ["planted", "identity", "ties", "k_ge_n"])
def test_search_kat(cuda, name, storage):
    import torch

    kat = KATS[name]
    c, q = _arrays(kat)
    idx = _index(c, cuda, storage)
    for dtype in (torch.bfloat16, torch.float32):
        s, i = idx.search(_q(q, cuda, dtype), kat["k"])
        torch.cuda.synchronize()
        _assert_exact(s, i, kat)


@pytest.mark.parametrize("name", ["planted", "identity", "ties", "k_ge_n"])
def test_search_kat_batched_and_large_k(cuda, name):
    """The KAT query repeated 300 times (CTA-pair kernel, B > 128) and with k padded up to 50
    (candidate-mode path, k > 32): the first k entries keep the known answer."""
    import torch

    kat = KATS[name]
    c, q = _arrays(kat)
    idx = _index(c, cuda)
    rep = [j % len(q) for j in range(300)]
    qq = q[rep]
    es, ei = _exp(kat)
    for k in (kat["k"], 50):
        s, i = idx.search(_q(qq, cuda, torch.bfloat16), k)
        torch.cuda.synchronize()
        s, i = from_dev(s), from_dev(i)
        kk = kat["k"]
        np.testing.assert_array_equal(i[:, :kk], ei[rep])
        np.testing.assert_array_equal(s[:, :kk], es[rep])
        assert (i[:, len(c):] == -1).all() and np.isneginf(s[:, len(c):]).all()


@pytest.mark.parametrize("name", ["planted", "identity", "ties", "k_ge_n"])
def test_segmented_kat(cuda, name):
    """The KAT corpus as the second of three per-query index segments of one arena (the
    others hold decoys that score higher): ids are local to the segment."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    kat = KATS[name]
    c, q = _arrays(kat)
    decoy = np.full((7, c.shape[1]), 50.0, np.float32)
    arena = np.concatenate([decoy, c, decoy])
    idx = DeviceIndex(c.shape[1], len(arena), metric="ip", device=cuda.index)
    idx.append(torch.from_numpy(arena).to(cuda))
    qq = np.concatenate([q, q, q])
    n = len(q)
    ranges = [(0, 7), (7, 7 + len(c)), (7 + len(c), len(arena))]
    s, i = idx.search_segmented(_q(qq, cuda, torch.bfloat16), [0, n, 2 * n, 3 * n], ranges,
                                kat["k"], local_ids=True)
    torch.cuda.synchronize()
    _assert_exact(s[n:2 * n], i[n:2 * n], kat)


@pytest.mark.parametrize("storage", ["bf16", "bf16_tiled", "f32"])
def test_rerank_kat_dedups(cuda, storage):
    import torch

    kat = KATS["dup_rerank"]
    c, q = _arrays(kat)
    idx = _index(c, cuda, storage)
    cand = torch.tensor(kat["candidates"], dtype=torch.int32, device=cuda)
    s, i = idx.rerank(_q(q, cuda, torch.bfloat16), cand, kat["k"])
    torch.cuda.synchronize()
    _assert_exact(s, i, kat)


def test_shard_kat_merge(cuda):
    """Per-shard fused searches with global ids, then the cross-shard merge (K4)."""
    import torch

    from paper_2407_00326_b200.index import merge_topk
    from paper_2407_00326_b200.sharded import shard_range

    kat = KATS["shards"]
    c, q = _arrays(kat)
    world, k = kat["world"], kat["k"]
    ls, li = [], []
    for r in range(world):
        lo, hi = shard_range(len(c), r, world)
        idx = _index(c[lo:hi], cuda)
        s, i = idx.search(_q(q, cuda, torch.bfloat16), k, id_offset=lo)
        ls.append(s)
        li.append(i)
    s, i = merge_topk(torch.stack(ls), torch.stack(li), k)
    torch.cuda.synchronize()
    _assert_exact(s, i, kat)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, exchange, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_00326_b200.sharded import ShardedSearch, shard_range

    kat = KATS["shards"]
    c, q = _arrays(kat)
    dev = torch.device("cuda", 0)
    lo, hi = shard_range(len(c), rank, world)
    idx = _index(c[lo:hi], dev)
    ss = ShardedSearch(idx, len(c), rank=rank, world=world, exchange=exchange)
    s, i = ss.search(_q(q, dev, torch.bfloat16), kat["k"])
    torch.cuda.synchronize()
    out[rank] = (from_dev(s).copy(), from_dev(i).copy())
    dist.barrier()
    if ss._peer is not None:
        ss._peer.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_shard_kat_across_ranks(cuda, exchange):
    """The shards KAT split over 3 ranks (processes sharing this GPU): ShardedSearch with the
    fused peer exchange (p2p) and with the all-gather + K4 path (over gloo here)."""
    import torch.multiprocessing as mp

    kat = KATS["shards"]
    world = kat["world"]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, exchange, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    es, ei = _exp(kat)
    for r in range(world):
        np.testing.assert_array_equal(out[r][1], ei)
        np.testing.assert_array_equal(out[r][0], es)


def test_fp32_single_kblock_ignores_stale_tmem(cuda):
    """fp32 mode with one k-block (dim <= 32) never writes its odd-k accumulator; that TMEM
    holds whatever the previous kernel left. Leave NaN there (a search over a corpus with NaN
    rows) and the planted KAT must still come out exact (the epilogue selects, not 0 * x)."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(0)
    junk = rng.standard_normal((4096, 64)).astype(np.float32)
    junk[::3] = np.nan
    bad = DeviceIndex(64, 4096, metric="ip", device=cuda.index)
    bad.append(torch.from_numpy(junk).to(cuda))
    for b in (300, 100):  # pair and single-CTA tcgen05 kernels fill TMEM with NaN scores
        bad.search(torch.from_numpy(junk[:b].copy()).to(cuda), 10)
    torch.cuda.synchronize()
    kat = KATS["planted"]
    c, q = _arrays(kat)
    idx = _index(c, cuda, "f32")
    for dtype in (torch.bfloat16, torch.float32):
        s, i = idx.search(_q(q, cuda, dtype), kat["k"])
        torch.cuda.synchronize()
        _assert_exact(s, i, kat)
