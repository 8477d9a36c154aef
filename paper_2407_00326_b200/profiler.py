"""Measured engine profiles for the retrieval engines.

The reference declares `vdb-search0` / `rerank0` latency tables by hand
(pkg/src/teola_sim/profiles/default.json:47-94) and derives the sub-batch size the optimizer
splits Searching nodes into from them (`max_efficient_batch`, engines.py:122-140): B_eff = 16
for search. On a B200 the fused scan gets cheaper per query up to the tensor/HBM ridge, so a
profile built from device measurements gives the optimizer a GPU-true B_eff.

`measure_search_profile` times `tsv_search` (a batch of B queries against a corpus of the
given shape) for B in a doubling ladder; `measure_rerank_profile` times `tsv_rerank` for C
candidates of one question. Both return an `EngineProfile` built by
`engines.measured_profile`.
"""

from __future__ import annotations

import json
from pathlib import Path

import torch

from .engines import EngineProfile, EngineSet, max_efficient_batch, measured_profile
from .index import DeviceIndex, normalize_rows


def _time(fn, reps: int = 20, warmup: int = 3, min_warm_ms: float = 100.0) -> float:
    """Mean device ms per call after `warmup` calls and at least `min_warm_ms` of warm-up
    (a jump in load shifts the power-capped clock for some tens of ms)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    spent = 0.0
    while spent < min_warm_ms:
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        spent += a.elapsed_time(b)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def measure_search_profile(rows: int = 1_000_000, dim: int = 1024, k: int = 10,
                           batches=(1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024),
                           engine_id: str = "vdb-search0", instances: int = 1,
                           device: int = 0) -> tuple[EngineProfile, list]:
    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(0)
    idx = DeviceIndex(dim, rows, metric="cosine", device=device)
    chunk = 1 << 18
    for a in range(0, rows, chunk):
        idx.append(torch.randn((min(chunk, rows - a), dim), generator=g, device=dev))
    samples = []
    for B in batches:
        q = normalize_rows(torch.randn((B, dim), generator=g, device=dev))
        out = (torch.empty((B, k), device=dev), torch.empty((B, k), dtype=torch.int32, device=dev))
        ms = _time(lambda: idx.search(q, k, out=out))
        samples.append((float(B), ms))
    prof = measured_profile(engine_id, "search", samples, instances=instances,
                            max_slots=float(max(batches)))
    return prof, samples


def measure_rerank_profile(rows: int = 100_000, dim: int = 1024,
                           candidates=(8, 16, 32, 48, 64, 128, 200, 256, 512), top_k: int = 10,
                           engine_id: str = "rerank0", instances: int = 1,
                           device: int = 0) -> tuple[EngineProfile, list]:
    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(1)
    idx = DeviceIndex(dim, rows, metric="cosine", device=device)
    idx.append(torch.randn((rows, dim), generator=g, device=dev))
    q = normalize_rows(torch.randn((1, dim), generator=g, device=dev))
    samples = []
    for C in candidates:
        cand = torch.randint(0, rows, (1, C), generator=g, device=dev, dtype=torch.int32)
        ms = _time(lambda: idx.rerank(q, cand, min(top_k, C)))
        samples.append((float(C), ms))
    prof = measured_profile(engine_id, "rerank", samples, instances=instances,
                            max_slots=float(max(candidates)))
    return prof, samples


def b200_profile_set(base: EngineSet, search: EngineProfile, rerank: EngineProfile) -> EngineSet:
    """The reference profile set with the retrieval engines replaced by measured ones."""
    out = EngineSet.from_profiles(list(base.values()))
    out[search.engine_id] = search
    out[rerank.engine_id] = rerank
    return out


def main():
    import argparse

    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=1024)
    ap.add_argument("--out", default="profiles/b200_engines.json")
    args = ap.parse_args()
    s, s_samples = measure_search_profile(args.rows, args.dim)
    r, r_samples = measure_rerank_profile(min(args.rows, 100_000), args.dim)
    doc = {"engines": [s.to_dict(), r.to_dict()],
           "measured": {"search": s_samples, "rerank": r_samples,
                        "corpus": [args.rows, args.dim], "device": torch.cuda.get_device_name()},
           "b_eff": {"vdb-search0": max_efficient_batch(s), "rerank0": max_efficient_batch(r)}}
    Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc["b_eff"]), json.dumps(doc["measured"]))


if __name__ == "__main__":
    main()
