"""The CPU oracle is pinned to known-answer vectors and the C restatement agrees with the
numpy one (these run without a GPU)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc

KATS = json.loads((Path(__file__).resolve().parent / "golden" / "retrieval_kats.json").read_text())


def _exp(kat):
    ids = np.array(kat["ids"], dtype=np.int64)
    scores = np.array([[(-np.inf if v is None else v) for v in row] for row in kat["scores"]])
    return scores, ids


@pytest.mark.parametrize("name", ["planted", "identity", "ties", "k_ge_n"])
def test_search_known_answers(name):
    kat = KATS[name]
    c = np.array(kat["corpus"], np.float32)
    q = np.array(kat["queries"], np.float32)
    s, i = orc.search(q, c, kat["k"])
    es, ei = _exp(kat)
    np.testing.assert_array_equal(i, ei)
    np.testing.assert_array_equal(s, es)


def test_rerank_known_answer_dedups():
    kat = KATS["dup_rerank"]
    c = np.array(kat["corpus"], np.float32)
    q = np.array(kat["queries"], np.float32)
    s, i = orc.rerank(q, c, np.array(kat["candidates"]), kat["k"])
    es, ei = _exp(kat)
    np.testing.assert_array_equal(i, ei)
    np.testing.assert_array_equal(s, es)


def test_shard_merge_known_answer():
    kat = KATS["shards"]
    c = np.array(kat["corpus"], np.float32)
    q = np.array(kat["queries"], np.float32)
    world, k = kat["world"], kat["k"]
    n = len(c)
    lists_s, lists_i = [], []
    for r in range(world):
        lo, hi = n * r // world, n * (r + 1) // world
        s, i = orc.search(q, c[lo:hi], k, id_offset=lo)
        lists_s.append(s)
        lists_i.append(i)
    s, i = orc.merge(np.stack(lists_s), np.stack(lists_i), k)
    es, ei = _exp(kat)
    np.testing.assert_array_equal(i, ei)
    np.testing.assert_array_equal(s, es)


def test_aggregate_is_slice_order_concatenation():
    """Aggregate joins stage outputs in slice order (optimizer.py:620-661): searching the
    query stages separately and concatenating equals searching them together."""
    c = orc.make_corpus(500, 64, seed=3)
    q, _ = orc.make_queries(c, 9, seed=4)
    whole = orc.search(q, c, 6)
    parts = [orc.search(q[a:b], c, 6) for a, b in ((0, 3), (3, 6), (6, 9))]
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), whole[1])


def test_comparator_detects_wrong_ids_and_accepts_tie_swaps():
    c = orc.make_corpus(2000, 64, seed=0)
    q, _ = orc.make_queries(c, 4, seed=1)
    s, i = orc.search(q, c, 5)
    assert orc.check_topk(s, i, q, c, 5, 1e-3) == []
    bad = i.copy()
    bad[0, 0] = (bad[0, 0] + 1) % 2000
    assert orc.check_topk(s, bad, q, c, 5, 1e-3)
    # exact duplicate rows: swapping the two tied ids is inside the tie band
    c2 = np.concatenate([c, c[:1]])
    q2 = c[:1].copy()
    s2, i2 = orc.search(q2, c2, 2)
    assert set(i2[0].tolist()) == {0, 2000}
    assert orc.check_topk(s2, i2[:, ::-1].copy(), q2, c2, 2, 1e-3) == []


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 0.0], np.float32)
    r = orc.bf16_round(x)
    np.testing.assert_array_equal(r, np.array([1.0, 1.0 + 2 ** -6, -2.5, 0.0], np.float32))


def test_c_oracle_matches_numpy_oracle():
    from oracle import c_oracle

    c = orc.make_corpus(3000, 128, seed=5)
    q, _ = orc.make_queries(c, 37, seed=6)
    for use_double in (False, True):
        s, i = c_oracle.search(orc.bf16_bits(q), orc.bf16_bits(c), 10, use_double=use_double,
                               nthreads=4, id_offset=100)
        assert orc.check_topk(s, i, q, c, 10, 1e-5, id_offset=100) == []
    for name in ("planted", "ties", "k_ge_n", "identity"):
        kat = KATS[name]
        cc = np.array(kat["corpus"], np.float32)
        qq = np.array(kat["queries"], np.float32)
        s, i = c_oracle.search(orc.bf16_bits(qq), orc.bf16_bits(cc), kat["k"], use_double=True,
                               nthreads=3)
        es, ei = _exp(kat)
        np.testing.assert_array_equal(i, ei)
        np.testing.assert_array_equal(s, es.astype(np.float32))


@pytest.mark.parametrize("op", ["<#>", "<=>"])
def test_pgvector_restatement_agrees_with_oracle(op):
    """The pgvector restatement (float32 sequential accumulation, ORDER BY distance LIMIT k)
    and the float64 oracle give the same top-k under the comparator at 1e-5 (fp32 mode's
    tolerance)."""
    c = orc.make_corpus(3000, 384, seed=0)
    q, _ = orc.make_queries(c, 12, seed=1)
    ps, pi = orc.pgvector_exact_search(q, c, 10, op=op)
    if op == "<=>":  # cosine of the stored (bf16-rounded, so not exactly unit) rows, in f64
        q = q / np.linalg.norm(q.astype(np.float64), axis=1, keepdims=True)
        c = c / np.linalg.norm(c.astype(np.float64), axis=1, keepdims=True)
    assert not orc.check_topk(ps, pi, q, c, 10, 1e-5)
    # ties: duplicated rows come back in ascending id order
    c2 = np.concatenate([c[:50], c[:50]])
    ps2, pi2 = orc.pgvector_exact_search(c2[:3], c2, 2, op=op)
    np.testing.assert_array_equal(pi2, [[0, 50], [1, 51], [2, 52]])


def test_amx_oracle_matches_numpy_oracle():
    """The AMX-BF16 build of the C oracle (the CPU baseline on AMX hosts) agrees with the numpy
    restatement: bf16 products are exact and accumulate in fp32 on the tiles, so only the
    summation order differs (ragged corpus blocks, a ragged last query tile, id offsets)."""
    from oracle import c_oracle

    lib = c_oracle.load("amx")
    if not lib.amx:
        pytest.skip("no AMX-BF16 on this host")
    c = orc.make_corpus(5003, 128, seed=4)
    q, _ = orc.make_queries(c, 37, seed=5)
    cb, qb = orc.bf16_bits(c), orc.bf16_bits(q)
    s, i = c_oracle._search(lib, qb, cb, 10, False, 4, 1000)
    probs = orc.check_topk(s, i, orc.bf16_to_f32(qb), orc.bf16_to_f32(cb), 10, 1e-3,
                           id_offset=1000)
    assert not probs, probs[:5]
    s2, i2 = c_oracle._search(c_oracle.load("v3"), qb, cb, 10, False, 4, 1000)
    np.testing.assert_allclose(s, s2, rtol=1e-5, atol=1e-6)
