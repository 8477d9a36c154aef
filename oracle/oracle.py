"""CPU oracle for the retrieval hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import this module, and only as the checker. The product path (``paper_2407_00326_b200``)
never calls it; there is no CPU fallback.

Parity status. The reference (Teola simulator, /root/reference/pkg) contains no retrieval
arithmetic: `Simulator._execute` returns a latency from a profile table
(pkg/src/teola_sim/runtime.py:653-655; pkg/src/teola_sim/engines.py:105-109) and payloads are
symbolic (pkg/src/teola_sim/graph.py:3-6, 73-85). The original system's arithmetic lived in
pgvector / bge-reranker-large, which are third-party, unversioned and not
vendored (no call site in the reference). This oracle therefore restates the published
semantics of those primitives and is pinned by (a) the reference's own structural tests and
golden e-graph for the path (cardinalities, slices, Aggregate concatenation — see
tests/golden/make_golden.py) and (b) known-answer vectors (planted neighbours, identity corpus,
exact ties, duplicate candidates, shard boundaries, k >= N) committed under tests/golden/.
Score arithmetic itself is "parity unpinned" against the reference (there is none to pin to);
`pgvector_exact_search` restates the published distance functions of the third-party engine
the paper's prototype used (pgvector, unversioned in the reference) and the GPU parity tests
also run the comparator against it.

Semantics restated here:
  * Searching ("Perform vector searching in the database"): per query, the
    top-k corpus rows by inner product; cosine = inner product over L2-normalised rows.
    Output cardinality query_count x per_query_top_k in query-major order
    (pkg/src/teola_sim/optimizer.py:178-197, line 187).
  * Reranking ("Compute and rank the relevance scores for the query and context
    pairs"): score candidate_count gathered rows against the question, keep top_k
    (optimizer.py:199-218, line 208). Duplicate candidate ids (the same chunk returned by two
    expanded queries) are scored once (dedup keeps the first occurrence) — a documented
    decision, since Aggregate concatenates without dedup (optimizer.py:642-657).
  * Aggregate of split stages = concatenation in slice order (optimizer.py:620-661).
  * Ordering: (score desc, id asc); padding (-inf, -1) when fewer than k rows exist.

Scores are computed in float64 from the bf16-rounded inputs, i.e. they are the exact inner
products of the values the device stores.
"""

from __future__ import annotations

import numpy as np

PAD_ID = -1


# ------------------------------------------------------------------ bf16 helpers
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern (uint16), round-to-nearest-even."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    return bf16_to_f32(bf16_bits(x))


def normalize_rows(x: np.ndarray) -> np.ndarray:
    """K5 restated: L2-normalise in fp32 (sum of squares, then x * rsqrt) and round to bf16."""
    f = np.asarray(x, dtype=np.float32)
    ss = np.einsum("ij,ij->i", f.astype(np.float64), f.astype(np.float64)).astype(np.float32)
    scale = (1.0 / np.sqrt(np.where(ss > 0, ss, 1.0))).astype(np.float32)
    return bf16_round(f * scale[:, None])


# ------------------------------------------------------------------ synthetic data
def make_corpus(n: int, dim: int, seed: int = 0, normalize: bool = True) -> np.ndarray:
    """N(0,1) rows, L2-normalised, as bf16-rounded float32 (corpus seed 0)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, dim), dtype=np.float32)
    return normalize_rows(x) if normalize else bf16_round(x)


def make_queries(corpus: np.ndarray, b: int, seed: int = 1, planted_frac: float = 0.5,
                 noise: float = 0.05) -> tuple[np.ndarray, np.ndarray]:
    """Half planted (corpus row + N(0, noise^2), renormalised), half fresh N(0,1).

    Returns (queries as bf16-rounded float32, planted row per query or -1)."""
    rng = np.random.default_rng(seed)
    n, dim = corpus.shape
    q = rng.standard_normal((b, dim), dtype=np.float32)
    planted = np.full(b, -1, dtype=np.int64)
    m = int(round(b * planted_frac))
    if m and n:
        rows = rng.integers(0, n, size=m)
        q[:m] = corpus[rows] + noise * rng.standard_normal((m, dim), dtype=np.float32)
        planted[:m] = rows
    return normalize_rows(q), planted


# ------------------------------------------------------------------ ordering
def order(scores: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """Indices sorting by (score desc, id asc)."""
    return np.lexsort((ids, -scores))


def pad_topk(scores: np.ndarray, ids: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    o = order(scores, ids)[:k]
    s = np.full(k, -np.inf, dtype=np.float64)
    i = np.full(k, PAD_ID, dtype=np.int64)
    s[: len(o)] = scores[o]
    i[: len(o)] = ids[o]
    return s, i


# ------------------------------------------------------------------ primitives
def scores_f64(q: np.ndarray, c: np.ndarray) -> np.ndarray:
    return np.asarray(q, dtype=np.float64) @ np.asarray(c, dtype=np.float64).T


def search(q: np.ndarray, c: np.ndarray, k: int, id_offset: int = 0,
           keep: int = 0, chunk: int = 65536):
    """Exact top-k (plus `keep` extra ranks for tie bands) of q against c.

    Returns (scores [B, k+keep] f64, ids [B, k+keep] i64)."""
    b = q.shape[0]
    n = c.shape[0]
    kk = k + keep
    best_s = np.full((b, 0), -np.inf)
    best_i = np.full((b, 0), PAD_ID, dtype=np.int64)
    q64 = np.asarray(q, dtype=np.float64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        s = q64 @ np.asarray(c[lo:hi], dtype=np.float64).T
        ids = np.arange(lo, hi, dtype=np.int64) + id_offset
        if s.shape[1] > kk:
            part = np.argpartition(-s, kk - 1, axis=1)[:, :kk]
            # argpartition may split a tie at the boundary: widen to every score >= cutoff
            cut = np.take_along_axis(s, part, 1).min(axis=1, keepdims=True)
            mask = s >= cut
            cand_s = [s[r][mask[r]] for r in range(b)]
            cand_i = [ids[mask[r]] for r in range(b)]
        else:
            cand_s = [s[r] for r in range(b)]
            cand_i = [ids for _ in range(b)]
        ns, ni = [], []
        for r in range(b):
            ss = np.concatenate([best_s[r], cand_s[r]])
            ii = np.concatenate([best_i[r], cand_i[r]])
            o = order(ss, ii)
            # keep every entry tied with the kk-th score so bands stay complete
            if len(o) > kk:
                cutoff = ss[o[kk - 1]]
                o = o[ss[o] >= cutoff]
            ns.append(ss[o])
            ni.append(ii[o])
        w = max(len(x) for x in ns)
        best_s = np.full((b, w), -np.inf)
        best_i = np.full((b, w), PAD_ID, dtype=np.int64)
        for r in range(b):
            best_s[r, : len(ns[r])] = ns[r]
            best_i[r, : len(ni[r])] = ni[r]
    out_s = np.full((b, kk), -np.inf)
    out_i = np.full((b, kk), PAD_ID, dtype=np.int64)
    w = min(kk, best_s.shape[1])
    out_s[:, :w] = best_s[:, :w]
    out_i[:, :w] = best_i[:, :w]
    return out_s, out_i


def search_segmented(q: np.ndarray, arena: np.ndarray, q_offsets, row_ranges, k: int,
                     local_ids: bool = True):
    b = q.shape[0]
    out_s = np.full((b, k), -np.inf)
    out_i = np.full((b, k), PAD_ID, dtype=np.int64)
    for s, (lo, hi) in enumerate(row_ranges):
        qa, qb = q_offsets[s], q_offsets[s + 1]
        if qb <= qa:
            continue
        off = -lo if local_ids else 0
        ss, ii = search(q[qa:qb], arena[lo:hi], k, id_offset=lo + off)
        out_s[qa:qb] = ss
        out_i[qa:qb] = ii
    return out_s, out_i


def rerank(q: np.ndarray, arena: np.ndarray, cand: np.ndarray, k: int):
    """Per question: dedup candidate ids (first occurrence), drop invalid ids, score, top-k."""
    b = q.shape[0]
    out_s = np.full((b, k), -np.inf)
    out_i = np.full((b, k), PAD_ID, dtype=np.int64)
    n = arena.shape[0]
    for r in range(b):
        seen = {}
        for cid in cand[r].tolist():
            if 0 <= cid < n and cid not in seen:
                seen[cid] = True
        ids = np.fromiter(seen.keys(), dtype=np.int64, count=len(seen))
        if len(ids) == 0:
            continue
        s = np.asarray(arena[ids], dtype=np.float64) @ np.asarray(q[r], dtype=np.float64)
        out_s[r], out_i[r] = pad_topk(s, ids, k)
    return out_s, out_i


def merge(scores: np.ndarray, ids: np.ndarray, k: int):
    """Merge [L, B, kin] sorted lists into [B, k]; padding entries (id < 0) are dropped."""
    L, b, kin = scores.shape
    out_s = np.full((b, k), -np.inf)
    out_i = np.full((b, k), PAD_ID, dtype=np.int64)
    for r in range(b):
        s = scores[:, r, :].reshape(-1).astype(np.float64)
        i = ids[:, r, :].reshape(-1).astype(np.int64)
        keep = i >= 0
        out_s[r], out_i[r] = pad_topk(s[keep], i[keep], k)
    return out_s, out_i


# ------------------------------------------------------------------ pgvector restatement
def pgvector_exact_search(q: np.ndarray, c: np.ndarray, k: int, op: str = "<#>",
                          keep: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """The original Teola's vector search, restated: PostgreSQL + pgvector,
    `SELECT id FROM chunks ORDER BY embedding <op> $query LIMIT k` on a table without an ANN
    index, i.e. an exact sequential scan. pgvector is a third-party dependency of the paper's
    prototype that the reference neither vendors nor pins (no version anywhere in
    /root/reference; no call site), so this follows pgvector's published distance functions
    for the `vector` type (float4 elements), unchanged across its releases:
      * `<#>` negative inner product: -(sum_i a[i] * b[i]) accumulated in float32, returned as
        float8 (vector_negative_inner_product / VectorInnerProduct);
      * `<=>` cosine distance: 1 - dot / sqrt(|a|^2 |b|^2) with dot and the squared norms
        accumulated in float32, the quotient in float8 and clamped to [-1, 1]
        (cosine_distance);
    ascending distance, LIMIT k. PostgreSQL's top-N sort does not define an order among equal
    distances; `id` breaks them here (ascending), which is the order this repo emits.
    pgvector compiles the accumulation loop with auto-vectorisation, so its exact float32
    summation order is build-dependent; this restatement sums sequentially over i.

    Returned in this repo's convention: scores (higher = better: -distance for `<#>`,
    1 - distance for `<=>`) and ids, [B, k + keep], padded with (-inf, -1)."""
    qf = np.asarray(q, dtype=np.float32)
    cf = np.asarray(c, dtype=np.float32)
    b, n = qf.shape[0], cf.shape[0]
    dot = np.zeros((b, n), dtype=np.float32)
    for i in range(qf.shape[1]):  # sequential float32 accumulation, as VectorInnerProduct
        dot += qf[:, i, None] * cf[None, :, i]
    if op == "<#>":
        score = dot.astype(np.float64)
    elif op == "<=>":
        na = np.zeros(b, dtype=np.float32)
        nb = np.zeros(n, dtype=np.float32)
        for i in range(qf.shape[1]):
            na += qf[:, i] * qf[:, i]
            nb += cf[:, i] * cf[:, i]
        sim = dot.astype(np.float64) / np.sqrt(na.astype(np.float64)[:, None] *
                                               nb.astype(np.float64)[None, :])
        score = np.clip(sim, -1.0, 1.0)  # 1 - cosine_distance
    else:
        raise ValueError(f"unknown pgvector operator {op!r}")
    kk = k + keep
    out_s = np.full((b, kk), -np.inf)
    out_i = np.full((b, kk), PAD_ID, dtype=np.int64)
    ids = np.arange(n, dtype=np.int64)
    for r in range(b):
        out_s[r], out_i[r] = pad_topk(score[r], ids, kk)
    return out_s, out_i


# ------------------------------------------------------------------ comparator
def check_topk(g_s, g_i, q, c, k: int, tol: float, id_offset: int = 0, local=None,
               oracle=None, abs_floor: float = 1e-6) -> list[str]:
    """Tolerance-aware comparison of device top-k against the exact oracle.

    For each rank r with oracle (o_s[r], o_id[r]) and band(r) = ids whose exact score is
    within tol*max(|o_s[r]|, abs_floor) of o_s[r]:
      1. |g_s[r] - o_s[r]| <= tol*max(|o_s[r]|, abs_floor);
      2. g_id[r] == o_id[r] when band(r) == {o_id[r]};
      3. otherwise g_id[r] in band(r);
      4. ids are distinct;
      5. the exact score of g_id[r] matches g_s[r] within tol.
    abs_floor: scale below which the tolerance is absolute (tol * abs_floor); deep ranks of a
    small segment score near zero, where a relative bound is meaningless.
    Returns a list of violation strings (empty = pass)."""
    g_s = np.asarray(g_s, dtype=np.float64)
    g_i = np.asarray(g_i, dtype=np.int64)
    b = g_s.shape[0]
    if oracle is None:
        o_s, o_i = search(q, c, k, id_offset=id_offset, keep=64)
    else:
        o_s, o_i = oracle
    problems: list[str] = []
    q64 = np.asarray(q, dtype=np.float64)
    for r in range(b):
        ids_r = g_i[r]
        valid = ids_r[ids_r >= 0]
        if len(set(valid.tolist())) != len(valid):
            problems.append(f"q{r}: duplicate ids {ids_r.tolist()}")
        for j in range(k):
            os_, oi = o_s[r, j], o_i[r, j]
            gs, gi = g_s[r, j], g_i[r, j]
            if oi < 0:
                if gi >= 0:
                    problems.append(f"q{r} rank{j}: expected padding, got id {gi}")
                continue
            eps = tol * max(abs(os_), abs_floor)
            if not abs(gs - os_) <= eps:
                problems.append(f"q{r} rank{j}: score {gs} vs oracle {os_}")
            band = o_i[r][(np.abs(o_s[r] - os_) <= eps) & (o_i[r] >= 0)]
            if len(band) == 1 and band[0] == oi:
                if gi != oi:
                    problems.append(f"q{r} rank{j}: id {gi} vs oracle {oi} (gap > tol)")
            elif gi not in set(band.tolist()):
                problems.append(f"q{r} rank{j}: id {gi} not in tie band {band.tolist()}")
            if gi >= 0:
                row = gi - id_offset
                if 0 <= row < c.shape[0]:
                    exact = float(q64[r] @ np.asarray(c[row], dtype=np.float64))
                    if not abs(exact - gs) <= eps:
                        problems.append(f"q{r} rank{j}: score {gs} != exact {exact} of id {gi}")
                else:
                    problems.append(f"q{r} rank{j}: id {gi} outside corpus")
            if len(problems) > 20:
                return problems
    return problems
