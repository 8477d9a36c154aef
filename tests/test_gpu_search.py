"""Parity of the fused scan + top-k (K1), merge (K4), segmented search (K2), rerank (K3) and
normalisation (K5) against the CPU oracle, through the C ABI. Tolerance: scores within 1e-3
relative for bf16 inputs (BASELINE.json north_star); ids bit-exact wherever the oracle's score
gap exceeds that tolerance, otherwise inside the oracle's tie band."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import assert_topk, from_dev, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _index_from(c_np, device, metric="ip", extra=0):
    from paper_2407_00326_b200.index import DeviceIndex

    idx = DeviceIndex(c_np.shape[1], c_np.shape[0] + extra, metric=metric, device=device.index)
    idx.append(to_dev_bf16(c_np, device))
    return idx


@pytest.mark.parametrize("n,dim,b,k", [
    (1000, 64, 1, 1), (5000, 128, 16, 5), (4099, 384, 100, 10), (20000, 768, 128, 16),
    (20000, 768, 129, 10), (30011, 1024, 256, 10), (12345, 72, 300, 32), (7, 64, 5, 10),
    (300, 1024, 1030, 4), (20000, 768, 300, 50), (5000, 256, 64, 100), (3000, 128, 20, 128),
    (100, 64, 3, 64),
])
def test_search_matches_oracle(cuda, n, dim, b, k):
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), k)
    assert_topk(s, i, q, c, k, TOL)


def test_planted_neighbours_rank_first(cuda):
    c = orc.make_corpus(50000, 768, seed=0)
    q, planted = orc.make_queries(c, 64, seed=1, planted_frac=1.0, noise=0.01)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), 10)
    ids = from_dev(i)
    assert (ids[:, 0] == planted).all()


def test_identity_corpus_scores_are_coordinates(cuda):
    dim = 128
    c = np.eye(dim, dtype=np.float32)
    rng = np.random.default_rng(5)
    q = orc.bf16_round(rng.standard_normal((20, dim)).astype(np.float32))
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), 8)
    exp_s, exp_i = orc.search(q, c, 8)
    np.testing.assert_array_equal(from_dev(i), exp_i)
    np.testing.assert_allclose(from_dev(s), exp_s, rtol=0, atol=0)


def test_exact_ties_break_by_ascending_id(cuda):
    rng = np.random.default_rng(3)
    base = orc.make_corpus(50, 256, seed=4)
    c = np.concatenate([base] * 8, axis=0)  # each row duplicated 8x (ids r, r+50, ...)
    perm = rng.permutation(len(c))
    c = c[perm]
    q = base[:12].copy()
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), 16)
    exp_s, exp_i = orc.search(q, c, 16)
    np.testing.assert_array_equal(from_dev(i), exp_i)


def test_k_exceeds_rows_pads(cuda):
    c = orc.make_corpus(3, 64, seed=0)
    q, _ = orc.make_queries(c, 4, seed=1)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), 8)
    ids = from_dev(i)
    assert (ids[:, 3:] == -1).all() and np.isneginf(from_dev(s)[:, 3:]).all()
    assert_topk(s, i, q, c, 8, TOL)


@pytest.mark.parametrize("n,b,k,lo,hi", [(40000, 200, 10, 12345, 33333),
                                         (300_000, 1024, 10, 1001, 290_001),
                                         (300_000, 1024, 100, 77, 299_000)])
def test_row_range_and_id_offset(cuda, n, b, k, lo, hi):
    """A row range that starts mid-arena (a shard of a larger corpus) with a global id offset,
    for the one-round, range-major (B=1024) and seeded candidate (k=100) layouts."""
    c = orc.make_corpus(n, 256, seed=0)
    q, _ = orc.make_queries(c[lo:hi], b, seed=1)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), k, row_range=(lo, hi), id_offset=1_000_000 - lo)
    sub = np.r_[0:16, b - 16:b]
    assert_topk(from_dev(s)[sub], from_dev(i)[sub], q[sub], c[lo:hi], k, TOL, id_offset=1_000_000)


def test_f32_queries_and_cosine(cuda):
    import torch

    rng = np.random.default_rng(9)
    raw = rng.standard_normal((10000, 256)).astype(np.float32) * 3.0
    from paper_2407_00326_b200.index import DeviceIndex

    idx = DeviceIndex(256, 10000, metric="cosine", device=cuda.index)
    idx.append(torch.from_numpy(raw).to(cuda))  # f32 rows, normalised on ingest
    stored = from_dev(idx.data())
    np.testing.assert_allclose(stored, orc.normalize_rows(raw), atol=2 ** -8)
    qraw = rng.standard_normal((33, 256)).astype(np.float32)
    s, i = idx.search(torch.from_numpy(qraw).to(cuda), 10)
    assert_topk(s, i, orc.normalize_rows(qraw), stored, 10, TOL)


def test_segmented_search_matches_oracle(cuda):
    rng = np.random.default_rng(11)
    sizes = [48, 32, 64, 1, 10000, 700, 129, 256]
    nq = [1, 3, 1, 2, 16, 4, 1, 130]
    arena = orc.make_corpus(sum(sizes), 384, seed=2)
    q = orc.make_corpus(sum(nq), 384, seed=3)
    row_ranges, q_off = [], [0]
    lo = 0
    for sz, m in zip(sizes, nq):
        row_ranges.append((lo, lo + sz))
        lo += sz
        q_off.append(q_off[-1] + m)
    idx = _index_from(arena, cuda)
    for k, local in ((5, True), (16, False), (50, True)):
        s, i = idx.search_segmented(to_dev_bf16(q, cuda), q_off, row_ranges, k, local_ids=local)
        gs, gi = from_dev(s), from_dev(i)
        for sidx, (a, b) in enumerate(row_ranges):
            qa, qb = q_off[sidx], q_off[sidx + 1]
            off = 0 if local else a
            probs = orc.check_topk(gs[qa:qb], gi[qa:qb], q[qa:qb], arena[a:b], k, TOL,
                                   id_offset=off)
            assert not probs, f"segment {sidx}: {probs[:5]}"


def test_rerank_dedups_and_matches_oracle(cuda):
    import torch

    rng = np.random.default_rng(12)
    arena = orc.make_corpus(5000, 768, seed=0)
    qs = orc.make_corpus(64, 768, seed=7)
    cand = rng.integers(0, 5000, size=(64, 200)).astype(np.int32)
    cand[:, 100:150] = cand[:, :50]          # duplicates from a second expansion
    cand[::7, 10] = -1                       # invalid entries are ignored
    cand[::5, 11] = 999999
    idx = _index_from(arena, cuda)
    s, i = idx.rerank(to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda), 10)
    exp_s, exp_i = orc.rerank(qs, arena, cand, 10)
    gs, gi = from_dev(s), from_dev(i)
    for r in range(64):
        assert len(set(gi[r].tolist())) == 10
    np.testing.assert_allclose(gs, exp_s, rtol=TOL)
    # ids must equal the oracle wherever neighbouring scores are separated by more than tol
    gap_ok = np.abs(np.diff(exp_s, axis=1, prepend=np.inf)) > TOL * np.abs(exp_s)
    gap_ok &= np.abs(np.diff(exp_s, axis=1, append=-np.inf)) > TOL * np.abs(exp_s)
    assert (gi[gap_ok] == exp_i[gap_ok]).all()


@pytest.mark.parametrize("c,k,dups", [(200, 16, 0), (200, 32, 0), (256, 17, 0), (200, 24, 40),
                                      (200, 20, 150), (33, 16, 10), (40, 30, 0)])
def test_rerank_topk_network_equals_rounds(cuda, c, k, dups):
    """The warp top-k network (16 <= k <= 32, C <= 256) is bit-identical to the k serial
    selection rounds (TSV_RERANK_NO_NET=1) and to the oracle's scores, including candidate
    lists whose 32 best keys hold fewer than k distinct ids (heavy duplication: the network
    hands over to the rounds) and lists with invalid ids."""
    import os

    import torch

    rng = np.random.default_rng(c * 31 + k + dups)
    n, b, dim = 3000, 40, 256
    arena = orc.make_corpus(n, dim, seed=8)
    qs = orc.make_corpus(b, dim, seed=9)
    cand = rng.integers(-1, n, size=(b, c)).astype(np.int32)
    if dups:  # the row each question scores highest, repeated `dups` times
        best = np.argmax(qs @ arena.T, axis=1).astype(np.int32)
        cand[:, :dups] = best[:, None]
    idx = _index_from(arena, cuda)
    qd, cd = to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda)
    old = os.environ.get("TSV_RERANK_NO_NET")
    try:
        os.environ.pop("TSV_RERANK_NO_NET", None)
        s1, i1 = idx.rerank(qd, cd, k)
        os.environ["TSV_RERANK_NO_NET"] = "1"
        s2, i2 = idx.rerank(qd, cd, k)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("TSV_RERANK_NO_NET", None)
        else:
            os.environ["TSV_RERANK_NO_NET"] = old
    np.testing.assert_array_equal(from_dev(s1), from_dev(s2))
    np.testing.assert_array_equal(from_dev(i1), from_dev(i2))
    exp_s, _ = orc.rerank(qs, arena, cand, k)
    np.testing.assert_allclose(from_dev(s1), exp_s, rtol=TOL, atol=1e-6)


def test_rerank_fewer_distinct_than_k_pads(cuda):
    import torch

    arena = orc.make_corpus(100, 64, seed=0)
    q = orc.make_corpus(2, 64, seed=1)
    cand = np.array([[5, 5, 5, 7], [1, -1, 1, 2]], dtype=np.int32)
    idx = _index_from(arena, cuda)
    s, i = idx.rerank(to_dev_bf16(q, cuda), torch.from_numpy(cand).to(cuda), 3)
    gi = from_dev(i)
    assert gi[0, 2] == -1 and set(gi[0, :2].tolist()) == {5, 7}
    assert gi[1, 2] == -1 and set(gi[1, :2].tolist()) == {1, 2}


@pytest.mark.parametrize("n,dim,b,c,k", [(5000, 768, 64, 200, 10), (3000, 1024, 16, 32, 3),
                                         (2000, 64, 5, 7, 7), (4000, 4096, 3, 50, 10),
                                         (1000, 384, 300, 33, 5)])
def test_rerank_shapes_match_oracle(cuda, n, dim, b, c, k):
    """K3 over candidate counts below, at and above one gather iteration (40 rows per block),
    dims below and above 1024 (the unrolled chunk loop), invalid ids and duplicates."""
    import torch

    rng = np.random.default_rng(3)
    arena = orc.make_corpus(n, dim, seed=0)
    qs = orc.make_corpus(b, dim, seed=7)
    cand = rng.integers(0, n, size=(b, c)).astype(np.int32)
    cand[::3, 0] = -1
    cand[::4, c - 1] = n + 5
    if c > 4:
        cand[:, 2] = cand[:, 1]
    idx = _index_from(arena, cuda)
    s, i = idx.rerank(to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda), k)
    exp_s, exp_i = orc.rerank(qs, arena, cand, k)
    np.testing.assert_allclose(from_dev(s), exp_s, rtol=TOL, atol=1e-6)
    gi = from_dev(i)
    for r in range(b):
        got = [x for x in gi[r].tolist() if x >= 0]
        assert len(got) == len(set(got))


@pytest.mark.parametrize("dim,c,b,k", [(768, 200, 70, 10), (1024, 64, 148, 8), (256, 77, 5, 7),
                                      (520, 131, 149, 5), (2048, 90, 33, 12), (64, 65, 1, 3)])
def test_rerank_paired_ring_bit_identical(cuda, dim, c, b, k):
    """4-slot rings scoring two rows per step (the default where B <= #SMs and C >= 64) give
    BIT-identical scores and ids to 2-slot rings (each row's FFMA2 / butterfly order is the
    same), write nothing outside their [B, k] outputs (sentinel guard rows around them), and
    match the oracle; odd candidate counts, invalid and duplicate ids, dim 2048 (3 slots)."""
    import os

    import torch

    rng = np.random.default_rng(dim * 7 + c)
    n = 3000
    arena = orc.make_corpus(n, dim, seed=6)
    qs = orc.make_corpus(b, dim, seed=7)
    cand = rng.integers(-1, n + 3, size=(b, c)).astype(np.int32)
    cand[:, 3] = cand[:, 2]
    idx = _index_from(arena, cuda)
    qd, cd = to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda)
    outs = {}
    old = os.environ.get("TSV_RERANK_SLOTS")
    try:
        for slots in ("2", "4"):
            os.environ["TSV_RERANK_SLOTS"] = slots
            gs = torch.full((b + 2, k), 12345.0, device=cuda)
            gi = torch.full((b + 2, k), 777, dtype=torch.int32, device=cuda)
            idx.rerank(qd, cd, k, out=(gs[1:b + 1], gi[1:b + 1]))
            torch.cuda.synchronize()
            gs, gi = from_dev(gs), from_dev(gi)
            for row in (0, b + 1):
                assert (gs[row] == 12345.0).all() and (gi[row] == 777).all(), slots
            outs[slots] = (gs[1:b + 1], gi[1:b + 1])
    finally:
        if old is None:
            os.environ.pop("TSV_RERANK_SLOTS", None)
        else:
            os.environ["TSV_RERANK_SLOTS"] = old
    np.testing.assert_array_equal(outs["2"][0], outs["4"][0])
    np.testing.assert_array_equal(outs["2"][1], outs["4"][1])
    valid = np.where((cand >= 0) & (cand < n), cand, -1)
    exp_s, _ = orc.rerank(qs, arena, valid, k)
    np.testing.assert_allclose(outs["4"][0], exp_s, rtol=TOL, atol=1e-6)


@pytest.mark.parametrize("dim,c,k,slots", [(768, 200, 10, None), (1024, 32, 3, None),
                                            (384, 57, 5, 2), (256, 300, 12, 4), (2048, 40, 4, None),
                                            (64, 3, 3, 3), (520, 77, 6, None),
                                            (768, 200, 10, "sort"), (256, 600, 10, None),
                                            (512, 100, 40, None), (1024, 512, 32, None),
                                            (768, 200, 10, "split8"), (256, 37, 20, "split2"),
                                            (1024, 1000, 8, None), (768, 200, 10, "lists"),
                                            (1024, 512, 32, "lists"), (768, 200, 10, "bitonic"),
                                            (128, 6, 12, None), (256, 400, 40, None)])
def test_rerank_ring_equals_register_gather(cuda, dim, c, k, slots):
    """The pipelined K3 (cp.async rings, question in registers, packed fp32x2 FMAs; bf16
    arenas; 16-warp ring blocks with a one-warp top-k selection (C <= 512; block bitonic sort
    above, or with TSV_RERANK_BITONIC), per-warp top-k lists for many short lists or forced by
    TSV_RERANK_LISTS) against the register-gather K3 (TSV_RERANK_LDG=1) and the oracle: scores
    equal up to the summation order (even / odd halves), ids equal wherever neighbouring scores
    differ; ring depths 2-4, candidate counts below / above one ring's worth and the lists
    path's limits, invalid ids, duplicates."""
    import os

    import torch

    rng = np.random.default_rng(dim + c)
    n, b = 4000, 70
    arena = orc.make_corpus(n, dim, seed=2)
    qs = orc.make_corpus(b, dim, seed=3)
    cand = rng.integers(0, n, size=(b, c)).astype(np.int32)
    cand[::3, 0] = -1
    cand[::4, c - 1] = n + 5
    if c > 4:
        cand[:, 2] = cand[:, 1]
    idx = _index_from(arena, cuda)
    qd, cd = to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda)
    env = ({"TSV_RERANK_SORT": "1"} if slots == "sort"
           else {"TSV_RERANK_SORT": "1", "TSV_RERANK_BITONIC": "1"} if slots == "bitonic"
           else {"TSV_RERANK_LISTS": "1"} if slots == "lists"
           else {"TSV_RERANK_SPLITS": slots[5:]} if isinstance(slots, str)
           else {"TSV_RERANK_SLOTS": str(slots)} if slots else {})
    old = {key: os.environ.get(key) for key in ("TSV_RERANK_SLOTS", "TSV_RERANK_LDG",
                                                "TSV_RERANK_SORT", "TSV_RERANK_SPLITS",
                                                "TSV_RERANK_LISTS", "TSV_RERANK_BITONIC")}
    try:
        os.environ.update(env)
        s1, i1 = idx.rerank(qd, cd, k)
        os.environ["TSV_RERANK_LDG"] = "1"
        s2, i2 = idx.rerank(qd, cd, k)
        torch.cuda.synchronize()
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v
    g1, g2 = from_dev(s1), from_dev(s2)
    np.testing.assert_allclose(g1, g2, rtol=2e-6, atol=1e-7)
    sep = np.abs(np.diff(g2, axis=1, prepend=np.inf)) > 1e-5
    sep &= np.abs(np.diff(g2, axis=1, append=-np.inf)) > 1e-5
    assert (from_dev(i1)[sep] == from_dev(i2)[sep]).all()
    exp_s, _ = orc.rerank(qs, arena, cand, k)
    np.testing.assert_allclose(g1, exp_s, rtol=TOL, atol=1e-6)


@pytest.mark.parametrize("dim,c,k", [(768, 200, 10), (1024, 64, 32), (256, 1000, 5)])
def test_rerank_f32_questions(cuda, dim, c, k):
    """K3 with fp32 questions on an inner-product bf16 index (the ring kernels keep the fp32
    question in registers): scores match the oracle's fp64 products of the unrounded fp32
    question with the bf16 rows."""
    import torch

    rng = np.random.default_rng(dim * 7 + c)
    n, b = 6000, 33
    arena = orc.make_corpus(n, dim, seed=11)
    qs = rng.standard_normal((b, dim)).astype(np.float32)
    cand = rng.integers(0, n, size=(b, c)).astype(np.int32)
    cand[:, 3] = cand[:, 0]
    cand[::2, 1] = -1
    idx = _index_from(arena, cuda)
    s, i = idx.rerank(torch.from_numpy(qs).to(cuda), torch.from_numpy(cand).to(cuda), k)
    exp_s, exp_i = orc.rerank(qs.astype(np.float64), arena, cand, k)
    gs, gi = from_dev(s), from_dev(i)
    np.testing.assert_allclose(gs, exp_s, rtol=2e-5, atol=2e-5)
    gap_ok = np.abs(np.diff(exp_s, axis=1, prepend=np.inf)) > 1e-4
    gap_ok &= np.abs(np.diff(exp_s, axis=1, append=-np.inf)) > 1e-4
    assert (gi[gap_ok] == exp_i[gap_ok]).all()


@pytest.mark.parametrize("storage", ["bf16", "bf16_tiled", "f32"])
def test_rerank_segmented_offsets(cuda, storage):
    """Reranking a batch of questions from different queries in one launch: question b's
    candidate ids are local to its own index segment (arena row = row_offsets[b] + id) and the
    returned ids stay local, as the Searching stages emitted them (tsv_rerank_segmented)."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(9)
    dim, k = 256, 5
    sizes = [48, 64, 33, 128, 40]
    starts = np.cumsum([0] + sizes)[:-1]
    arena = orc.make_corpus(int(sum(sizes)), dim, seed=4)
    qs = orc.make_corpus(len(sizes), dim, seed=5)
    c = 32
    cand = np.stack([rng.integers(0, sz, size=c) for sz in sizes]).astype(np.int32)
    cand[1, 3] = -1
    cand[2, 5] = cand[2, 4]
    idx = DeviceIndex(dim, len(arena), device=cuda.index, storage=storage)
    idx.append(torch.from_numpy(arena).to(cuda) if storage == "f32" else to_dev_bf16(arena, cuda))
    offs = torch.tensor(starts, dtype=torch.int32, device=cuda)
    qd = torch.from_numpy(qs).to(cuda) if storage == "f32" else to_dev_bf16(qs, cuda)
    s, i = idx.rerank(qd, torch.from_numpy(cand).to(cuda), k, row_offsets=offs)
    torch.cuda.synchronize()
    for b, (a, sz) in enumerate(zip(starts, sizes)):
        es, ei = orc.rerank(qs[b:b + 1], arena[a:a + sz], cand[b:b + 1], k)
        np.testing.assert_allclose(from_dev(s)[b:b + 1], es, rtol=TOL, atol=1e-6)
        assert set(from_dev(i)[b].tolist()) <= set(cand[b].tolist())
    # the same offsets as a host list (tsv_rerank_segmented_host): identical results
    s2, i2 = idx.rerank(qd, torch.from_numpy(cand).to(cuda), k,
                        row_offsets=[int(a) for a in starts])
    torch.cuda.synchronize()
    assert torch.equal(s2, s) and torch.equal(i2, i)


def test_rerank_host_offsets_under_graph_capture(cuda):
    """tsv_rerank_segmented_host inside a CUDA graph: the offsets' upload becomes a graph node
    reading the library's capture pool (filled at capture time), so replays reproduce the
    eager result; a call outside capture on the same stream first allocates that pool."""
    import torch

    from paper_2407_00326_b200._native import PrivateStream

    rng = np.random.default_rng(21)
    dim, k, sizes = 512, 4, [40, 64, 50]
    starts = [int(x) for x in np.cumsum([0] + sizes)[:-1]]
    arena = orc.make_corpus(int(sum(sizes)), dim, seed=7)
    qs = orc.make_corpus(len(sizes), dim, seed=8)
    cand = np.stack([rng.integers(0, sz, size=24) for sz in sizes]).astype(np.int32)
    idx = _index_from(arena, cuda)
    qd, cd = to_dev_bf16(qs, cuda), torch.from_numpy(cand).to(cuda)
    ps = PrivateStream(cuda.index)
    try:
        st = ps.stream
        eager = idx.rerank(qd, cd, k, row_offsets=starts, stream=st)
        out = (torch.empty((3, k), dtype=torch.float32, device=cuda),
               torch.empty((3, k), dtype=torch.int32, device=cuda))
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            idx.rerank(qd, cd, k, row_offsets=starts, stream=st, out=out)
        for _ in range(3):
            out[0].fill_(0)
            out[1].fill_(-7)
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out[0], eager[0]) and torch.equal(out[1], eager[1])
        for b, (a, sz) in enumerate(zip(starts, sizes)):
            es, _ = orc.rerank(qs[b:b + 1], arena[a:a + sz], cand[b:b + 1], k)
            np.testing.assert_allclose(from_dev(out[0])[b:b + 1], es, rtol=TOL, atol=1e-6)
        del g
    finally:
        torch.cuda.synchronize()
        ps.close()


def test_merge_matches_oracle(cuda):
    import torch
    from paper_2407_00326_b200.index import merge_topk

    rng = np.random.default_rng(13)
    L, B, kin, k = 8, 300, 16, 10
    sc = rng.standard_normal((L, B, kin)).astype(np.float32)
    sc = -np.sort(-sc, axis=2)
    ids = rng.permutation(L * B * kin).reshape(L, B, kin).astype(np.int32)
    ids[3, :, 12:] = -1
    sc[3, :, 12:] = -np.inf
    sc[5, :, 0] = sc[6, :, 0]  # exact cross-list ties
    s, i = merge_topk(torch.from_numpy(sc).cuda(), torch.from_numpy(ids).cuda(), k)
    es, ei = orc.merge(sc, ids, k)
    np.testing.assert_array_equal(from_dev(i), ei)
    np.testing.assert_array_equal(from_dev(s), es.astype(np.float32))


@pytest.mark.parametrize("L,kin,k", [(64, 32, 100), (100, 10, 10), (74, 128, 100), (3, 128, 128)])
def test_merge_many_lists_radix_select(cuda, L, kin, k):
    """Merges with many more candidates than outputs take the radix-select path: exact ties,
    exact duplicate entries, padding-heavy lists and fewer candidates than k."""
    import torch
    from paper_2407_00326_b200.index import merge_topk

    rng = np.random.default_rng(L * 1000 + kin)
    B = 37
    sc = (rng.integers(-400, 400, (L, B, kin)) / 128.0).astype(np.float32)  # many equal scores
    sc = -np.sort(-sc, axis=2)
    ids = rng.permutation(L * B * kin).reshape(L, B, kin).astype(np.int32)
    real = rng.integers(0, kin + 1, (L, B))  # each list keeps a random-length real prefix
    pad = np.arange(kin)[None, None, :] >= real[:, :, None]
    ids[pad] = -1
    sc[pad] = -np.inf
    if L > 2:  # an exact duplicate of list 0's head in list 1 (same id, same score)
        sc[1, :, 0] = np.maximum(sc[1, :, 0], sc[0, :, 0])
        keep = ids[0, :, 0] >= 0
        sc[1, keep, 0] = sc[0, keep, 0]
        ids[1, keep, 0] = ids[0, keep, 0]
        order = np.argsort(-sc[1], axis=1, kind="stable")
        sc[1] = np.take_along_axis(sc[1], order, axis=1)
        ids[1] = np.take_along_axis(ids[1], order, axis=1)
    s, i = merge_topk(torch.from_numpy(sc).cuda(), torch.from_numpy(ids).cuda(), k)
    es, ei = orc.merge(sc, ids, k)
    np.testing.assert_array_equal(from_dev(s), es.astype(np.float32))
    np.testing.assert_array_equal(from_dev(i), ei)


def test_normalize_rows_matches_oracle(cuda):
    import torch
    from paper_2407_00326_b200.index import normalize_rows

    rng = np.random.default_rng(14)
    x = rng.standard_normal((777, 1024)).astype(np.float32) * 7
    x[3] = 0.0
    out = from_dev(normalize_rows(torch.from_numpy(x).cuda()))
    np.testing.assert_allclose(out, orc.normalize_rows(x), atol=2 ** -8, rtol=2 ** -7)


def test_errors_map_to_teola_errors(cuda):
    import torch
    from paper_2407_00326_b200.errors import CapacityExceeded, ConfigParse
    from paper_2407_00326_b200.index import DeviceIndex

    idx = DeviceIndex(64, 10, device=cuda.index)
    with pytest.raises(CapacityExceeded):
        idx.append(torch.zeros((11, 64), dtype=torch.bfloat16, device=cuda))
    idx.append(torch.zeros((10, 64), dtype=torch.bfloat16, device=cuda))
    with pytest.raises(CapacityExceeded):
        idx.search(torch.zeros((0, 64), dtype=torch.bfloat16, device=cuda), 3)
    with pytest.raises(ConfigParse):
        idx.search(torch.zeros((2, 64), dtype=torch.bfloat16, device=cuda), 129)
    with pytest.raises(ConfigParse):
        DeviceIndex(60, 10, device=cuda.index)


@pytest.mark.slow
def test_c2_full_size_properties(cuda):
    """C2 (1M x 768 bf16, B=256, k=10) at full size: oracle on a query subset, and
    size-independent properties (sortedness, distinct ids, exact re-scoring) on all."""
    import torch

    n, dim, b, k = 1_000_000, 768, 256, 10
    g = torch.Generator(device=cuda).manual_seed(0)
    c = torch.randn((n, dim), generator=g, device=cuda)
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows

    cb = normalize_rows(c)
    del c
    qb = normalize_rows(torch.randn((b, dim), generator=g, device=cuda))
    qb[:128] = cb[torch.arange(0, 128, device=cuda) * 7777]  # planted exact rows
    idx = DeviceIndex.view(cb)
    s, i = idx.search(qb, k)
    gs, gi = from_dev(s), from_dev(i)
    assert (np.diff(gs, axis=1) <= 0).all()
    assert all(len(set(r.tolist())) == k for r in gi)
    assert (gi[:128, 0] == np.arange(128) * 7777).all() or np.allclose(
        gs[:128, 0], gs[:128, 1])
    cn = from_dev(cb)
    qn = from_dev(qb)
    rescored = np.einsum("bd,bkd->bk", qn.astype(np.float64), cn[gi].astype(np.float64))
    np.testing.assert_allclose(gs, rescored, rtol=TOL)
    sub = np.r_[0:8, 128:136]
    assert_topk(s[sub], i[sub], qn[sub], cn, k, TOL)


@pytest.mark.parametrize("n,dim,b,k", [(20000, 256, 64, 10), (5000, 1024, 300, 32),
                                       (3333, 96, 5, 64), (50, 64, 3, 10)])
def test_fp32_mode_matches_oracle_at_1e5(cuda, n, dim, b, k):
    """fp32 mode (K1f, 3xTF32): scores within 1e-5 relative of the exact fp32 products."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(21)
    raw = rng.standard_normal((n, dim)).astype(np.float32)
    idx = DeviceIndex(dim, n, metric="cosine", device=cuda.index, storage="f32")
    idx.append(torch.from_numpy(raw).to(cuda))
    hi, lo = idx.planes()
    stored = (hi.double() + lo.double()).cpu().numpy()
    ref = raw / np.linalg.norm(raw, axis=1, keepdims=True)
    np.testing.assert_allclose(stored, ref, atol=1e-6)
    qraw = rng.standard_normal((b, dim)).astype(np.float32)
    qraw[: b // 2] = raw[rng.integers(0, n, b // 2)] + 0.01 * qraw[: b // 2]
    s, i = idx.search(torch.from_numpy(qraw).to(cuda), k)
    qn = (qraw / np.linalg.norm(qraw, axis=1, keepdims=True)).astype(np.float64)
    # the device normalises in fp32; compare against the exact products of those vectors
    probs = orc.check_topk(from_dev(s), from_dev(i), qn, stored, k, 1e-5)
    assert not probs, probs[:5]


def test_fp32_mode_rerank(cuda):
    import torch
    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(22)
    raw = rng.standard_normal((4000, 128)).astype(np.float32)
    idx = DeviceIndex(128, 4000, metric="ip", device=cuda.index, storage="f32")
    idx.append(torch.from_numpy(raw).to(cuda))
    q = rng.standard_normal((8, 128)).astype(np.float32)
    cand = rng.integers(0, 4000, size=(8, 100)).astype(np.int32)
    s, i = idx.rerank(torch.from_numpy(q).to(cuda), torch.from_numpy(cand).to(cuda), 5)
    es, ei = orc.rerank(q.astype(np.float64), raw.astype(np.float64), cand, 5)
    np.testing.assert_allclose(from_dev(s), es, rtol=1e-5)


@pytest.mark.parametrize("n,dim,b,k", [(20000, 768, 256, 10), (4099, 72, 1, 5), (30011, 1024, 300, 50),
                                       (1000, 384, 1030, 16), (300_000, 128, 1024, 100)])
def test_tiled_layout_identical_to_row_major(cuda, n, dim, b, k):
    """The tiled arena (contiguous 16 KB k-block tiles) feeds the same operands to the tensor
    cores, so results are bit-identical to the row-major arena, and match the oracle."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex

    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    rm = _index_from(c, cuda)
    tl = DeviceIndex(dim, n, device=cuda.index, storage="bf16_tiled")
    tl.append(to_dev_bf16(c, cuda))
    np.testing.assert_array_equal(from_dev(tl.data()), c)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = rm.search(qd, k)
    s2, i2 = tl.search(qd, k)
    np.testing.assert_array_equal(from_dev(i1), from_dev(i2))
    np.testing.assert_array_equal(from_dev(s1), from_dev(s2))
    assert_topk(s2, i2, q, c, k, TOL)
    cand = torch.from_numpy(np.random.default_rng(0).integers(0, n, (b, 40)).astype(np.int32)).to(cuda)
    r1 = rm.rerank(qd, cand, 5)
    r2 = tl.rerank(qd, cand, 5)
    np.testing.assert_array_equal(from_dev(r1[1]), from_dev(r2[1]))


def test_tiled_segmented_requires_aligned_segments(cuda):
    from paper_2407_00326_b200.errors import ConfigParse
    from paper_2407_00326_b200.index import DeviceIndex

    c = orc.make_corpus(1024, 128, seed=0)
    q = orc.make_corpus(3, 128, seed=1)
    tl = DeviceIndex(128, 1024, device=cuda.index, storage="bf16_tiled")
    tl.append(to_dev_bf16(c, cuda))
    s, i = tl.search_segmented(to_dev_bf16(q, cuda), [0, 1, 3], [(0, 300), (384, 1024)], 7)
    assert not orc.check_topk(from_dev(s)[:1], from_dev(i)[:1], q[:1], c[0:300], 7, TOL)
    assert not orc.check_topk(from_dev(s)[1:], from_dev(i)[1:], q[1:], c[384:1024], 7, TOL)
    with pytest.raises(ConfigParse):
        tl.search_segmented(to_dev_bf16(q, cuda), [0, 3], [(5, 300)], 7)


def _search_env(idx, qd, k, row_range=None, **env):
    import os

    import torch

    old = {key: os.environ.get(key) for key in env}
    os.environ.update({key: str(v) for key, v in env.items()})
    try:
        s, i = idx.search(qd, k) if row_range is None else idx.search(qd, k, row_range=row_range)
        torch.cuda.synchronize()
    finally:
        for key, v in old.items():
            if v is None:
                del os.environ[key]
            else:
                os.environ[key] = v
    return from_dev(s), from_dev(i)


@pytest.mark.parametrize("b,k", [(300, 100), (64, 100), (1024, 50), (200, 128)])
def test_seeded_large_k_is_exact(cuda, b, k):
    """k > 32 on >= 262144 rows runs a 1/16-sample pass first; the main pass then appends every
    row above the sample's k-th score to a per-query candidate row and selects the top k (pair
    kernel for B > 128, single-CTA kernel below). The result must equal the seeded list-mode
    search, the unseeded search and the oracle, bit for bit."""
    n, dim = 300_000, 256
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    idx = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(idx, qd, k)
    s2, i2 = _search_env(idx, qd, k, TSV_NO_SEED=1)
    s3, i3 = _search_env(idx, qd, k, TSV_NO_APPEND=1)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_array_equal(i1, i3)
    np.testing.assert_array_equal(s1, s3)
    sub = np.r_[0:20, b // 2:b // 2 + 20]
    assert_topk(s1[sub], i1[sub], q[sub], c, k, TOL)


def test_candidate_overflow_falls_back_exactly(cuda):
    """Degenerate corpus: half the rows are copies of one vector v. Queries equal to v tie with
    150,000 rows, so their candidate rows overflow (cap 8192) and the device-gated list-mode
    pass must recompute the batch; ties break by ascending id."""
    n, dim, b, k = 300_000, 256, 256, 100
    c = orc.make_corpus(n, dim, seed=0)
    v = c[7].copy()
    c[1::2] = v
    q, _ = orc.make_queries(c, b, seed=1)
    q[::4] = v  # every 4th query overflows, the others do not
    idx = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(idx, qd, k)
    s2, i2 = _search_env(idx, qd, k, TSV_NO_SEED=1)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)
    # the tied block: row 1, 3, 5, ... (all equal v; row 7 is v too but odd, so included)
    np.testing.assert_array_equal(i1[0], np.arange(1, 2 * k, 2))


@pytest.mark.parametrize("b,k", [(1024, 10), (768, 16), (1024, 32), (2048, 10), (4096, 8),
                                 (1280, 16)])
def test_range_major_rounds_identical(cuda, b, k):
    """B=1024 (4 query groups), 768 (3), 1280 (5), 2048 (8), 4096 (16) do not divide the 74 CTA
    pairs: the pair kernel then takes range-major items over 3-8 rounds (lockstepped range
    partners up to 4 query groups). The result must be identical to the one-round layout and
    match the oracle."""
    n, dim = 200_000, 256
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    idx = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(idx, qd, k)
    s2, i2 = _search_env(idx, qd, k, TSV_NO_RANGE_MAJOR=1)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)
    sub = np.r_[0:16, b - 16:b]
    assert_topk(s1[sub], i1[sub], q[sub], c, k, TOL)


@pytest.mark.parametrize("n,dim,b,k", [(20000, 1024, 256, 10), (5000, 384, 16, 5),
                                       (300_000, 256, 300, 100)])
def test_search_matches_pgvector_restatement(cuda, n, dim, b, k):
    """The original system's search, `ORDER BY embedding <#> q LIMIT k` in PostgreSQL +
    pgvector (oracle.pgvector_exact_search: float32 sequential accumulation), as the oracle of
    the comparator: scores within 1e-3 relative, ids exact outside tie bands."""
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), k)
    sub = np.r_[0:min(b, 24)]
    pg = orc.pgvector_exact_search(q[sub], c, k, op="<#>", keep=64)
    assert_topk(from_dev(s)[sub], from_dev(i)[sub], q[sub], c, k, TOL, oracle=pg)


def test_seeded_search_on_sorted_corpus(cuda):
    """A corpus stored in topical order (rows sorted by their score against a direction v,
    best last) with queries near v: the seeding sample (the first 1/16 of every range) still
    gives an exact result equal to the unseeded search."""
    n, dim, b, k = 300_000, 128, 256, 64
    c = orc.make_corpus(n, dim, seed=3)
    v = orc.make_corpus(1, dim, seed=9)[0]
    c = c[np.argsort(c @ v, kind="stable")]
    q = orc.normalize_rows(v[None, :] + 0.3 * orc.make_corpus(b, dim, seed=4))
    idx = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(idx, qd, k)
    s2, i2 = _search_env(idx, qd, k, TSV_NO_SEED=1)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)
    assert_topk(s1[:8], i1[:8], q[:8], c, k, TOL)


@pytest.mark.parametrize("n,dim,b,k", [(200_000, 128, 1024, 128), (50_000, 256, 600, 64),
                                       (262_144, 64, 1030, 33), (300_007, 200, 130, 100)])
def test_large_k_paths_match_oracle(cuda, n, dim, b, k):
    """k > 32 through every path: pair kernel with shared-memory lists and range-major rounds
    (no seeding below 262,144 rows), B not a multiple of the query group, seeded candidate mode
    with the single-CTA kernel (B <= 128 per group) and odd row counts / dims."""
    c = orc.make_corpus(n, dim, seed=5)
    q, _ = orc.make_queries(c, b, seed=6)
    idx = _index_from(c, cuda)
    s, i = idx.search(to_dev_bf16(q, cuda), k)
    sub = np.r_[0:12, b - 12:b]
    assert_topk(from_dev(s)[sub], from_dev(i)[sub], q[sub], c, k, TOL)


@pytest.mark.parametrize("k", [33, 64, 128])
def test_segmented_large_k_candidate_mode(cuda, k):
    """Segmented search with k > 32 and every segment <= 8192 rows runs candidate mode (every
    row a candidate, exact select); it must equal the shared-memory-list path bit for bit and
    the oracle, including segments with fewer rows than k (padding)."""
    import os

    import torch

    sizes = [48, 32, 64, 1, 8000, 700, 129, 256]
    nq = [1, 3, 1, 2, 16, 4, 1, 130]
    arena = orc.make_corpus(sum(sizes), 256, seed=12)
    q = orc.make_corpus(sum(nq), 256, seed=13)
    row_ranges, q_off, lo = [], [0], 0
    for sz, m in zip(sizes, nq):
        row_ranges.append((lo, lo + sz))
        lo += sz
        q_off.append(q_off[-1] + m)
    idx = _index_from(arena, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = idx.search_segmented(qd, q_off, row_ranges, k, local_ids=True)
    os.environ["TSV_NO_SEED"] = "1"
    try:
        s2, i2 = idx.search_segmented(qd, q_off, row_ranges, k, local_ids=True)
        torch.cuda.synchronize()
    finally:
        del os.environ["TSV_NO_SEED"]
    np.testing.assert_array_equal(from_dev(i1), from_dev(i2))
    np.testing.assert_array_equal(from_dev(s1), from_dev(s2))
    gs, gi = from_dev(s1), from_dev(i1)
    for sidx, (a, b) in enumerate(row_ranges):
        qa, qb = q_off[sidx], q_off[sidx + 1]
        # deep ranks of the small segments score ~0: absolute tolerance below 1e-2
        probs = orc.check_topk(gs[qa:qb], gi[qa:qb], q[qa:qb], arena[a:b], k, TOL,
                               abs_floor=1e-2)
        assert not probs, f"segment {sidx}: {probs[:5]}"


@pytest.mark.parametrize("n,dim,b,k", [(20000, 1024, 24, 10), (8000, 384, 16, 50)])
def test_fp32_mode_matches_pgvector_cosine(cuda, n, dim, b, k):
    """fp32 mode against the original engine's own arithmetic: pgvector stores float4 vectors
    and `ORDER BY embedding <=> q LIMIT k` ranks by cosine distance computed in float32
    (oracle.pgvector_exact_search). The fp32-mode index (cosine metric, raw fp32 rows in)
    must agree at the fp32 mode's 1e-5 tolerance; the comparator's exact scores are the
    float64 cosines of the raw vectors."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(33)
    raw = rng.standard_normal((n, dim)).astype(np.float32)
    qraw = rng.standard_normal((b, dim)).astype(np.float32)
    qraw[: b // 2] = raw[rng.integers(0, n, b // 2)] + 0.02 * qraw[: b // 2]
    idx = DeviceIndex(dim, n, metric="cosine", device=cuda.index, storage="f32")
    idx.append(torch.from_numpy(raw).to(cuda))
    s, i = idx.search(torch.from_numpy(qraw).to(cuda), k)
    pg = orc.pgvector_exact_search(qraw, raw, k, op="<=>", keep=64)
    cn = raw.astype(np.float64) / np.linalg.norm(raw.astype(np.float64), axis=1, keepdims=True)
    qn = qraw.astype(np.float64) / np.linalg.norm(qraw.astype(np.float64), axis=1, keepdims=True)
    probs = orc.check_topk(from_dev(s), from_dev(i), qn, cn, k, 1e-5, oracle=pg)
    assert not probs, probs[:5]


def test_two_streams_share_an_index(cuda):
    """Searches issued on two streams against one index keep separate workspaces (partial
    lists, candidate rows, staged queries): interleaved calls return what sequential calls do."""
    import torch

    n, dim = 300_000, 128
    c = orc.make_corpus(n, dim, seed=41)
    idx = _index_from(c, cuda)
    qa = to_dev_bf16(orc.make_queries(c, 1024, seed=42)[0], cuda)
    qb = to_dev_bf16(orc.make_queries(c, 300, seed=43)[0], cuda)
    ref_a = [from_dev(x) for x in idx.search(qa, 10)]
    ref_b = [from_dev(x) for x in idx.search(qb, 100)]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    outs = []
    for _ in range(3):
        outs.append((idx.search(qa, 10, stream=s1), idx.search(qb, 100, stream=s2)))
    torch.cuda.synchronize()
    for (a, b) in outs:
        np.testing.assert_array_equal(from_dev(a[1]), ref_a[1])
        np.testing.assert_array_equal(from_dev(a[0]), ref_a[0])
        np.testing.assert_array_equal(from_dev(b[1]), ref_b[1])
        np.testing.assert_array_equal(from_dev(b[0]), ref_b[0])


def test_view_index_matches_arena_and_rejects_append(cuda):
    """DeviceIndex.view wraps an existing bf16 matrix without copying: same results as an arena
    holding the same rows (including the k > 32 path), and appends are refused."""
    from paper_2407_00326_b200.errors import TeolaError
    from paper_2407_00326_b200.index import DeviceIndex

    c = orc.make_corpus(300_000, 128, seed=51)
    q, _ = orc.make_queries(c, 300, seed=52)
    rows = to_dev_bf16(c, cuda)
    view = DeviceIndex.view(rows)
    arena = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    for k in (10, 64):
        s1, i1 = _search_env(view, qd, k)
        s2, i2 = _search_env(arena, qd, k)
        np.testing.assert_array_equal(i1, i2)
        np.testing.assert_array_equal(s1, s2)
    with pytest.raises(TeolaError):
        view.append(rows[:10])


@pytest.mark.parametrize("n,dim,b,k,lo", [(600_000, 128, 128, 10, 0), (524_416, 256, 100, 32, 0),
                                          (40_000, 768, 128, 16, 1000), (1003, 64, 120, 4, 5)])
def test_wide_tiles_identical(cuda, n, dim, b, k, lo):
    """96 < B <= 128 on long scans uses 256-row corpus tiles (M=128 x N=256 MMAs); TSV_WIDE=1
    forces them on short scans too (ragged last tile, odd row ranges). Results must equal the
    128-row tiles' bit for bit and match the oracle."""
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    idx = _index_from(c, cuda)
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(idx, qd, k, row_range=(lo, n), TSV_WIDE=1)
    s2, i2 = _search_env(idx, qd, k, row_range=(lo, n), TSV_WIDE=0)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)
    sub = np.r_[0:8, b - 8:b]
    assert_topk(s1[sub], i1[sub], q[sub], c[lo:], k, TOL, id_offset=lo)


@pytest.mark.slow
@pytest.mark.parametrize("k", [10, 100])
def test_headline_full_size_exact(cuda, k):
    """The bench configuration at full size (10M x 1024 bf16, B=1024; k=10 and C4's k=100):
    every query's list sorted with distinct ids, planted rows found first, every returned score
    equal to an fp32 re-scoring of its row, and 64 queries (32 planted, 32 fresh) checked
    against the CPU oracle (the C restatement, fp64 accumulation, over all 10M rows): ids
    bit-exact wherever the oracle's score gap exceeds the 1e-3 tolerance, scores within it."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows

    n, dim, b = 10_000_000, 1024, 1024
    g = torch.Generator(device=cuda).manual_seed(0)
    idx = DeviceIndex(dim, n, metric="cosine", device=cuda.index)
    for a in range(0, n, 1 << 20):
        idx.append(torch.randn((min(1 << 20, n - a), dim), generator=g, device=cuda))
    rows = idx.data()
    planted = torch.randint(0, n, (b // 2,), generator=g, device=cuda)
    q = torch.empty((b, dim), dtype=torch.bfloat16, device=cuda)
    q[: b // 2] = rows[planted]
    q[b // 2:] = normalize_rows(torch.randn((b // 2, dim), generator=g, device=cuda))
    s, i = idx.search(q, k)
    torch.cuda.synchronize()
    assert bool((s[:, 1:] <= s[:, :-1]).all())
    srt = torch.sort(i, dim=1).values
    assert bool((srt[:, 1:] != srt[:, :-1]).all())
    top1_ok = (i[: b // 2, 0] == planted.to(torch.int32)) | (s[: b // 2, 0] == s[: b // 2, 1])
    assert bool(top1_ok.all())
    resc = torch.einsum("bd,bkd->bk", q.float(), rows[i.long()].float())
    assert float((resc - s).abs().max()) < 2e-5

    # 64 queries (32 planted, 32 fresh) against the CPU oracle: the C restatement in fp64 over
    # the host copy of all 10M rows (1M-row chunks, per-chunk top-(k+16) with global ids,
    # merged), then the comparator of SURVEY.md §7.1 at the bf16 tolerance.
    from oracle import c_oracle

    sub = torch.cat([torch.arange(0, 32), torch.arange(b - 32, b)]).to(cuda)
    q_bits = q[sub].view(torch.int16).cpu().numpy().view(np.uint16)
    keep = k + 16
    parts_s, parts_i = [], []
    for a in range(0, n, 1 << 20):
        chunk = rows[a: a + (1 << 20)].view(torch.int16).cpu().numpy().view(np.uint16)
        cs, ci = c_oracle.search(q_bits, chunk, keep, use_double=True, id_offset=a)
        parts_s.append(cs)
        parts_i.append(ci)
    o_s, o_i = orc.merge(np.stack(parts_s), np.stack(parts_i), keep)

    class _HostRows:  # rows of the device corpus fetched on demand for exact re-scoring
        shape = (n, dim)

        def __getitem__(self, r):
            return from_dev(rows[int(r)])

    qs = from_dev(q[sub])
    probs = orc.check_topk(from_dev(s[sub]), from_dev(i[sub]), qs, _HostRows(), k, TOL,
                           oracle=(o_s, o_i))
    assert not probs, probs[:10]
    planted_sub = planted[:32].cpu().numpy()
    assert (o_i[:32, 0] == planted_sub).all()  # the oracle finds the planted rows too


@pytest.mark.parametrize("n,lo", [(600_000, 0), (70_001, 256), (3000, 128)])
def test_wide_tiles_on_tiled_arena(cuda, n, lo):
    """256-row corpus tiles over the tiled arena (two 128-row k-block tiles per step, the
    second one past the end for a ragged last tile) equal the row-major 128-row-tile result."""
    from paper_2407_00326_b200.index import DeviceIndex

    dim, b, k = 256, 120, 10
    c = orc.make_corpus(n, dim, seed=0)
    q, _ = orc.make_queries(c, b, seed=1)
    rm = _index_from(c, cuda)
    tl = DeviceIndex(dim, n, device=cuda.index, storage="bf16_tiled")
    tl.append(to_dev_bf16(c, cuda))
    qd = to_dev_bf16(q, cuda)
    s1, i1 = _search_env(tl, qd, k, row_range=(lo, n), TSV_WIDE=1)
    s2, i2 = _search_env(rm, qd, k, row_range=(lo, n), TSV_WIDE=0)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1, s2)


@pytest.mark.parametrize("storage", ["bf16", "bf16_tiled"])
@pytest.mark.parametrize("metric,dim,k_s,k_r,sep_q", [
    ("cosine", 1024, 32, 3, False), ("ip", 256, 10, 10, True), ("cosine", 768, 50, 5, True),
    ("ip", 64, 1, 1, False)])
def test_search_rerank_segmented_fused(cuda, storage, metric, dim, k_s, k_r, sep_q):
    """tsv_search_rerank_segmented (C5's Searching -> Reranking chain in one kernel): per query,
    the search over its own segment equals the oracle's (tie bands), and the rerank of the
    kernel's own search hits against the (separate or same) question equals the oracle's
    rerank; segments of 0, 1, 7, 33, 48, 300 and 1024 rows, segment-local and arena ids,
    fp32 and bf16 queries; the segment table from the device and from a host list give
    identical results."""
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    rng = np.random.default_rng(dim + k_s)
    sizes = [48, 7, 1024, 33, 0, 300, 1, 48]
    starts = np.cumsum([0] + sizes)[:-1]
    n = int(sum(sizes))
    c = orc.make_corpus(n, dim, seed=3)
    idx = DeviceIndex(dim, n, metric=metric, device=cuda.index, storage=storage)
    idx.append(to_dev_bf16(c, cuda))
    B = len(sizes)
    q = orc.make_corpus(B, dim, seed=4)
    qr = orc.make_corpus(B, dim, seed=5) if sep_q else None
    rows = torch.tensor([[a, a + z] for a, z in zip(starts, sizes)], dtype=torch.int64,
                        device=cuda)
    for local in (True, False):
        for f32 in (False, True):
            qd = torch.from_numpy(q).to(cuda) if f32 else to_dev_bf16(q, cuda)
            qrd = None if qr is None else (torch.from_numpy(qr).to(cuda) if f32
                                           else to_dev_bf16(qr, cuda))
            (ss, si), (rs, ri) = idx.search_rerank_segmented(qd, rows, max(sizes), k_s, k_r,
                                                             q_rerank=qrd, local_ids=local)
            if not local:  # the rerank half is K3's arithmetic: bit-identical scores
                us, ui = idx.rerank(qd if qrd is None else qrd, si, k_r)
            # the host-table entry point (tsv_search_rerank_segmented_host) is the same launch
            host_rows = [int(x) for x in rows.cpu().reshape(-1)]
            (ss2, si2), (rs2, ri2) = idx.search_rerank_segmented(qd, host_rows, max(sizes), k_s,
                                                                 k_r, q_rerank=qrd, local_ids=local)
            torch.cuda.synchronize()
            gs, gi, hs, hi = from_dev(ss), from_dev(si), from_dev(rs), from_dev(ri)
            for x, y in ((gs, ss2), (gi, si2), (hs, rs2), (hi, ri2)):
                np.testing.assert_array_equal(x, from_dev(y))
            if not local:
                np.testing.assert_array_equal(hs, from_dev(us))
                np.testing.assert_array_equal(hi, from_dev(ui))
            for b, (a, z) in enumerate(zip(starts, sizes)):
                off = 0 if local else a
                qb = orc.bf16_round(q[b:b + 1]) if metric == "ip" and not f32 else q[b:b + 1]
                probs = orc.check_topk(gs[b:b + 1], gi[b:b + 1], qb, c[a:a + z], k_s, TOL,
                                       id_offset=off)
                assert not probs, (b, probs[:3])
                qq = q if qr is None else qr
                qrb = orc.bf16_round(qq[b:b + 1]) if metric == "ip" and not f32 else qq[b:b + 1]
                cand = gi[b:b + 1] - off
                cand[gi[b:b + 1] < 0] = -1
                es, ei = orc.rerank(qrb, c[a:a + z], cand, k_r)
                np.testing.assert_allclose(hs[b:b + 1], es, rtol=TOL, atol=1e-6)
                real = hi[b] >= 0
                assert real.sum() == min(z, k_r)
                assert set((hi[b][real] - off).tolist()) <= set(cand[0][cand[0] >= 0].tolist())


@pytest.mark.parametrize("n,dim,b,k,metric,storage,f32q", [
    (10000, 384, 16, 5, "cosine", "bf16", False),    # C1
    (10000, 384, 16, 5, "cosine", "bf16", True),
    (4097, 256, 40, 16, "ip", "bf16", False), (65536, 128, 3, 10, "cosine", "bf16", False),
    (7, 64, 5, 10, "ip", "bf16", False), (1, 1024, 64, 1, "cosine", "bf16", False),
    (3000, 1024, 17, 8, "ip", "bf16_tiled", False), (2500, 520, 9, 12, "cosine", "bf16", True),
    (8000, 768, 12, 16, "ip", "bf16", False)])
def test_small_scan_matches_oracle_and_tensor_path(cuda, n, dim, b, k, metric, storage, f32q,
                                                  monkeypatch):
    """One-launch searches for few queries over short row ranges (routed automatically: K2t on
    the tensor cores for row-major arenas, K2s on the CUDA cores for tiled ones or with
    TSV_NO_TINY) vs the CPU oracle and vs the general scan (TSV_NO_SMALL=1) on the same
    inputs: query groups of 16 / 8 / 4 by dim, k <= 16, fp32 and bf16 queries, cosine and
    inner product, row-major and tiled arenas, a row sub-range with an id offset, fewer rows
    than k."""
    import torch

    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex

    # (TSV_FORCE_SMALL: K2s serves every shape it fits here, also those the default routing
    # leaves to the general scan because it is faster there)
    monkeypatch.setenv("TSV_FORCE_SMALL", "1")
    c = orc.make_corpus(n, dim, seed=n % 97)
    q, _ = orc.make_queries(c, b, seed=2)
    idx = DeviceIndex(dim, n, metric=metric, device=cuda.index, storage=storage)
    idx.append(to_dev_bf16(c, cuda))
    qd = torch.from_numpy(q).to(cuda) if f32q else to_dev_bf16(q, cuda)
    qo = orc.normalize_rows(q) if metric == "cosine" else (q if f32q else orc.bf16_round(q))
    n0 = _native.launch_count()
    s, i = idx.search(qd, k)
    torch.cuda.synchronize()
    # no staging or K4 launches: one kernel (K2s, or K2t issued call by call) or, under graph
    # capture / TSV_TINY_SPLIT=1, the K2t scan + its merge grid launched behind it (PDL)
    assert _native.launch_count() - n0 in (1, 2)
    assert_topk(s, i, qo, c, k, TOL)
    monkeypatch.setenv("TSV_TINY_SPLIT", "1")  # K2t with its merge as a second (PDL) grid
    s0, i0 = idx.search(qd, k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(from_dev(i0), from_dev(i))
    np.testing.assert_array_equal(from_dev(s0), from_dev(s))
    monkeypatch.delenv("TSV_TINY_SPLIT")
    monkeypatch.setenv("TSV_NO_TINY", "1")  # the CUDA-core K2s instead of the tcgen05 K2t
    s1, i1 = idx.search(qd, k)
    torch.cuda.synchronize()
    assert_topk(s1, i1, qo, c, k, TOL)
    np.testing.assert_allclose(from_dev(s), from_dev(s1), rtol=1e-5, atol=1e-6)
    monkeypatch.delenv("TSV_NO_TINY")
    monkeypatch.setenv("TSV_NO_SMALL", "1")
    s2, i2 = idx.search(qd, k)
    torch.cuda.synchronize()
    np.testing.assert_allclose(from_dev(s), from_dev(s2), rtol=1e-5, atol=1e-6)
    # a sub-range of rows with an id offset (row-major arenas; tiled ranges start at 128 k)
    monkeypatch.delenv("TSV_NO_SMALL")
    lo = 128 if n > 256 else 0
    s3, i3 = idx.search(qd, k, row_range=(lo, n), id_offset=1000)
    torch.cuda.synchronize()
    assert_topk(s3, i3, qo, c[lo:], k, TOL, id_offset=1000 + lo)  # ids = arena row + offset
