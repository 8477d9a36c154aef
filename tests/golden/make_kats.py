"""Known-answer vectors for the retrieval primitives.

The reference has no retrieval arithmetic, so these answers are derived analytically from
the construction of each input (not by running the oracle):
  planted   : query = corpus row r (exactly) -> r ranks first with score |r|^2
  identity  : corpus = I_D -> scores are the query's coordinates, ids their indices
  ties      : corpus rows duplicated -> equal scores ordered by ascending id
  dup_rerank: candidate list with repeated ids -> each id scored once
  shards    : top-k split across shard boundaries -> merge of per-shard lists
  k_ge_n    : k larger than the row count -> padding (-inf, -1)
Values are small integers / exact binary fractions so bf16 and fp32 represent them exactly.
Run: python tests/golden/make_kats.py  (writes retrieval_kats.json)
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "retrieval_kats.json"


def main():
    rng = np.random.default_rng(7)
    kats = {}

    # planted: 64 rows of small integers; queries are exact copies of rows 5, 17, 40
    c = rng.integers(-4, 5, size=(64, 16)).astype(np.float32)
    c[5] = 6.0
    c[17] = -6.0
    c[40, :8] = 6.0
    c[40, 8:] = -6.0
    q = c[[5, 17, 40]].copy()
    kats["planted"] = {"corpus": c.tolist(), "queries": q.tolist(), "k": 1,
                       "ids": [[5], [17], [40]],
                       "scores": [[float(c[5] @ c[5])], [float(c[17] @ c[17])],
                                  [float(c[40] @ c[40])]]}

    # identity: corpus I_16, query coordinates distinct powers of two
    d = 16
    qv = np.array([[2.0 ** (i % 7) * (1 if i % 3 else -1) for i in range(d)]], np.float32)
    qv[0, 3] = 100.0
    order = sorted(range(d), key=lambda i: (-qv[0, i], i))[:5]
    kats["identity"] = {"corpus": np.eye(d, dtype=np.float32).tolist(), "queries": qv.tolist(),
                        "k": 5, "ids": [order], "scores": [[float(qv[0, i]) for i in order]]}

    # ties: row 3 duplicated at ids 3, 9, 12; the query equals row 3 -> ids 3, 9, 12 in order
    c = np.zeros((16, 8), np.float32)
    for i in range(16):
        c[i, i % 8] = 1.0
    c[3] = c[9] = c[12] = np.array([2, 0, 0, 0, 0, 0, 0, 0], np.float32)
    q = np.array([[1, 0, 0, 0, 0, 0, 0, 0]], np.float32)
    kats["ties"] = {"corpus": c.tolist(), "queries": q.tolist(), "k": 4,
                    "ids": [[3, 9, 12, 0]], "scores": [[2.0, 2.0, 2.0, 1.0]]}

    # dup_rerank: candidates [7, 2, 7, 5, 2, -1] over rows with score = row index
    c = np.zeros((10, 8), np.float32)
    c[:, 0] = np.arange(10)
    q = np.array([[1, 0, 0, 0, 0, 0, 0, 0]], np.float32)
    kats["dup_rerank"] = {"corpus": c.tolist(), "queries": q.tolist(), "k": 4,
                          "candidates": [[7, 2, 7, 5, 2, -1]],
                          "ids": [[7, 5, 2, -1]], "scores": [[7.0, 5.0, 2.0, None]]}

    # shards: 12 rows, score = 11 - |row - 6|; 3 shards of 4 rows; top-4 spans all shards
    c = np.zeros((12, 8), np.float32)
    c[:, 0] = [11 - abs(r - 6) for r in range(12)]
    q = np.array([[1, 0, 0, 0, 0, 0, 0, 0]], np.float32)
    kats["shards"] = {"corpus": c.tolist(), "queries": q.tolist(), "k": 4, "world": 3,
                      "ids": [[6, 5, 7, 4]], "scores": [[11.0, 10.0, 10.0, 9.0]]}

    # k_ge_n: 3 rows, k = 5
    c = np.array([[1, 0], [3, 0], [2, 0]], np.float32)
    c = np.pad(c, ((0, 0), (0, 6)))
    q = np.array([[1, 0, 0, 0, 0, 0, 0, 0]], np.float32)
    kats["k_ge_n"] = {"corpus": c.tolist(), "queries": q.tolist(), "k": 5,
                      "ids": [[1, 2, 0, -1, -1]], "scores": [[3.0, 2.0, 1.0, None, None]]}
    OUT.write_text(json.dumps(kats, sort_keys=True) + "\n")
    print(OUT)


if __name__ == "__main__":
    main()
