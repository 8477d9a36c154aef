"""Single-process corpus sharding (tsv_sharded_* / ShardedIndex): shards on one device (the
same device twice or three times — the ranks of an 8-GPU node become devices of one process
the same way), every result equal to one index holding every row and to the CPU oracle; the
sharded corpus behind the executor (`Simulator._execute`, reference runtime.py:625-656) as the
global index of the retrieval backend; and the forward-progress guard of the lockstepped scan
(two B=1024 scans on two streams plus a third kernel complete and agree with serial runs)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import assert_topk, from_dev, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _shards(c, dev, parts, metric="ip"):
    from paper_2407_00326_b200.index import DeviceIndex

    n = len(c)
    out = []
    for g in range(parts):
        lo, hi = n * g // parts, n * (g + 1) // parts
        idx = DeviceIndex(c.shape[1], hi - lo, metric=metric, device=dev.index)
        idx.append(to_dev_bf16(c[lo:hi], dev))
        out.append(idx)
    return out


@pytest.mark.parametrize("n,dim,b,k,parts", [(30_000, 256, 64, 10, 2), (50_001, 128, 300, 10, 3),
                                             (40_000, 256, 200, 100, 2), (777, 64, 5, 16, 3)])
def test_sharded_index_equals_single_index(cuda, n, dim, b, k, parts):
    import torch

    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.sharded import ShardedIndex

    c = orc.make_corpus(n, dim, seed=11)
    q, _ = orc.make_queries(c, b, seed=12)
    shards = _shards(c, cuda, parts)
    sh = ShardedIndex(shards, max_batch=512, max_k=128)
    assert sh.rows == n and sh.offsets[0] == 0
    whole = DeviceIndex(dim, n, device=cuda.index)
    whole.append(to_dev_bf16(c, cuda))
    qd = to_dev_bf16(q, cuda)
    s1, i1 = sh.search(qd, k)
    s2, i2 = whole.search(qd, k)
    torch.cuda.synchronize()
    # a shard may take another kernel than the whole corpus (the one-launch searches serve
    # short ranges), whose fp32 sums differ in the last bits: scores equal to 1e-5, ids equal
    # wherever neighbouring scores are further apart
    g1, g2 = from_dev(s1), from_dev(s2)
    np.testing.assert_allclose(g1, g2, rtol=1e-5, atol=1e-6)
    sep = np.abs(np.diff(g2, axis=1, prepend=np.inf)) > 1e-4
    sep &= np.abs(np.diff(g2, axis=1, append=-np.inf)) > 1e-4
    assert (from_dev(i1)[sep] == from_dev(i2)[sep]).all()
    sub = np.r_[0:min(b, 8), max(0, b - 8):b]
    assert_topk(from_dev(s1)[sub], from_dev(i1)[sub], q[sub], c, k, TOL)
    sh.close()


def test_sharded_index_rejects_oversize_and_wrong_device(cuda):
    import torch

    from paper_2407_00326_b200.errors import CapacityExceeded, ConfigParse
    from paper_2407_00326_b200.sharded import ShardedIndex

    c = orc.make_corpus(2000, 64, seed=1)
    sh = ShardedIndex(_shards(c, cuda, 2), max_batch=16, max_k=8)
    q = to_dev_bf16(c[:32], cuda)
    with pytest.raises(CapacityExceeded):
        sh.search(q, 4)  # B > max_batch
    with pytest.raises(CapacityExceeded):
        sh.search(q[:4], 9)  # k > max_k
    with pytest.raises(ConfigParse):
        sh.search(q[:4], 4, out=(torch.empty((4, 4), device=cuda), torch.empty((4, 4), device=cuda)))


def _global_search_graph(qid: str, nq: int, k: int):
    """Embedding (modelled) -> Searching over the resident global corpus (no per-query index
    input): the C4 shape behind the reference executor."""
    from paper_2407_00326_b200.graph import (Edge, EGraph, MetadataProfile, Payload,
                                             PrimitiveKind, PrimitiveNode, assign_depths)

    emb = PrimitiveNode("emb", PrimitiveKind.EMBEDDING, MetadataProfile(
        outputs={"query_vectors": Payload(nq, nq * 16)}, engine_id="embed0", batch_items=nq,
        query_id=qid))
    srch = PrimitiveNode("search.search", PrimitiveKind.SEARCHING, MetadataProfile(
        inputs=("query_vectors",), outputs={"top_chunks": Payload(nq * k, nq * k * 256)},
        engine_id="vdb-search0", batch_items=nq, query_id=qid))
    g = EGraph(nodes={"emb": emb, "search.search": srch},
               edges=[Edge("emb", "search.search", "query_vectors")], query_id=qid)
    g.depth = assign_depths(g)
    return g


def test_sharded_corpus_behind_the_executor(cuda):
    """C4 through Simulator._execute: the backend's global index is a ShardedIndex (two shards
    on this device); every Searching output equals the CPU oracle over the whole corpus."""
    import json
    from pathlib import Path

    import torch

    from paper_2407_00326_b200 import engines as E, runtime as R
    from paper_2407_00326_b200.backend import RetrievalBackend, SearchResult
    from paper_2407_00326_b200.sharded import ShardedIndex

    prof = json.loads((Path(__file__).resolve().parent / "golden" / "ref_profiles.json")
                      .read_text())["default"]["profiles"]
    dim, n, k, nq = 256, 60_000, 10, 16
    c = orc.make_corpus(n, dim, seed=21)
    sh = ShardedIndex(_shards(c, cuda, 2, metric="cosine"), max_batch=1024, max_k=128)
    backend = RetrievalBackend(dim=dim, arena_rows=1 << 12, global_index=sh,
                               release_segments=False)  # keep ctx.data for the check
    es = E.EngineSet.from_dict(prof)
    graphs = [(_global_search_graph(f"q{j}", nq, k), 5.0 * j, 0.0) for j in range(4)]
    sim, trace = R.run_queries(es, graphs, R.RuntimeOptions(), backend=backend)
    torch.cuda.synchronize()
    assert backend.launches > 0
    checked = 0
    for ctx in sim.contexts.values():
        res = ctx.store[("search.search", "top_chunks")].data
        assert isinstance(res, SearchResult)
        d = ctx.data[("emb", "query_vectors")]
        q = from_dev(d[5].bfloat16())
        assert_topk(from_dev(res.scores), from_dev(res.ids), q, c, k, TOL)
        checked += 1
    assert checked == 4


def test_concurrent_lockstepped_scans_complete(cuda):
    """Two B=1024 scans (CTA pairs in range lockstep: partners spin on each other's progress)
    on two streams plus a GEMM on a third: partners of one scan can be kept off the SMs by the
    other kernels; the bounded lockstep wait lets every scan finish, with the serial results."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows

    n, dim, b, k = 400_000, 1024, 1024, 10
    g = torch.Generator(device=cuda).manual_seed(5)
    idx = DeviceIndex(dim, n, metric="cosine", device=cuda.index)
    idx.append(torch.randn((n, dim), generator=g, device=cuda))
    qa = normalize_rows(torch.randn((b, dim), generator=g, device=cuda))
    qb = normalize_rows(torch.randn((b, dim), generator=g, device=cuda))
    ra = idx.search(qa, k)
    rb = idx.search(qb, k)
    torch.cuda.synchronize()
    ref = [(x.clone(), y.clone()) for x, y in (ra, rb)]
    s1, s2, s3 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    m = torch.randn((8192, 8192), device=cuda, dtype=torch.bfloat16)
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s3):
            mm = m @ m
        oa = idx.search(qa, k, stream=s1)
        ob = idx.search(qb, k, stream=s2)
        with torch.cuda.stream(s3):
            mm = mm @ m
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        for (s, i), (rs, ri) in zip((oa, ob), ref):
            assert torch.equal(i, ri) and torch.equal(s, rs)
    del mm
